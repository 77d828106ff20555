"""A/B of the compact path's coupled / decoupled split (RDS_OPT_RDC_SPLIT) at the stated K:
python scripts/split_ab.py [--config C3] [--deltas 0.02 0.05 0.1 0.2].  One JSON line per
delta: K-loop ms (CUDA events, median of reps) with the split off / on (1) / on with grouped
components (2), the decoupled and grouped fractions, the dense path's K-loop for reference, and whether all three gave the same u."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--deltas", type=float, nargs="+", default=[0.02, 0.05, 0.1, 0.2])
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = wl.CONFIGS[a.config]
z, P = wl.make_image(cfg)
K = cfg.iters
S = {}
for name, kw in (("dense", dict(compact=0)), ("unsplit", dict(compact=1, rdc_split=0)),
                 ("split", dict(compact=1, rdc_split=1)),
                 ("grouped", dict(compact=1, rdc_split=2))):
    s = rds.Solver(cfg.H, cfg.W, timing=True, **kw)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
    S[name] = s
am = S["dense"].absmax()
for dr in a.deltas:
    d = wl.band_delta(dr, am)
    row = {"config": cfg.name, "delta_rel": dr, "K": K}
    us = {}
    for name, s in S.items():
        s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, d, K)
        ts = []
        for _ in range(a.reps):
            s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, d, K)
            st = s.stats()
            ts.append((st["loop_ms"], st["setup_ms"]))
        row[name + "_loop_ms"] = statistics.median(t[0] for t in ts)
        row[name + "_setup_ms"] = statistics.median(t[1] for t in ts)
        us[name] = s.u()
        if name == "split":
            row["rd_frac"] = st["n_rd"] / (cfg.H * cfg.W)
            row["decoupled_frac"] = st["rdc_decoupled"] / max(1, st["n_rd"])
        if name == "grouped":
            row["grouped_frac"] = st["rdc_grouped"] / max(1, st["n_rd"])
            row["barrier_px"] = st["n_rd"] - st["rdc_decoupled"] - st["rdc_grouped"]
    row["split_speedup"] = row["unsplit_loop_ms"] / row["split_loop_ms"]
    row["split_vs_dense"] = row["dense_loop_ms"] / row["split_loop_ms"]
    row["grouped_vs_split"] = row["split_loop_ms"] / row["grouped_loop_ms"]
    row["grouped_vs_dense"] = (row["dense_loop_ms"] + row["dense_setup_ms"]) / (
        row["grouped_loop_ms"] + row["grouped_setup_ms"])
    row["same_u"] = bool(np.array_equal(us["dense"], us["split"]) and
                         np.array_equal(us["unsplit"], us["split"]) and
                         np.array_equal(us["grouped"], us["split"]))
    print(json.dumps(row), flush=True)
