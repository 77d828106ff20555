"""Restricted vs unrestricted solve times per delta on one config (tile skipping on/off).
Prints one JSON line per (delta, skip): K-loop ms (CUDA events, median of reps), active tile
and item fractions, RD fraction, speedup vs the delta=inf solve."""
import argparse
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--iters", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--kf", type=int, default=0)
ap.add_argument("--rows", type=int, default=0)
args = ap.parse_args()

cfg = wl.CONFIGS[args.config]
K = args.iters or cfg.iters
z, P = wl.make_image(cfg)
st = torch.cuda.Stream()
s = rds.Solver(cfg.H, cfg.W, stream=st.cuda_stream, timing=True, k_fuse=args.kf,
               item_rows=args.rows)
s.set_image(torch.from_numpy(z).cuda())
s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, torch.from_numpy(P).cuda() if P is not None else None)
am = s.absmax()
deltas = sorted(set(cfg.delta_rels) | {math.inf})
res = {}
for skip in (1, 0):
    s.set_option(rds.RDS_OPT_SKIP, skip)
    for dr in deltas:
        d = wl.band_delta(dr, am)
        s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, d, K)
        s.stats()
        ts, ss = [], []
        for _ in range(args.reps):
            s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, d, K)
            x = s.stats()
            ts.append(x["loop_ms"])
            ss.append(x["setup_ms"])
        res[(skip, dr)] = (statistics.median(ts), statistics.median(ss), x)
for skip in (1, 0):
    full = res[(skip, math.inf)][0]
    for dr in deltas:
        lm, sm, x = res[(skip, dr)]
        print(json.dumps({
            "config": cfg.name, "skip": skip, "delta_rel": "inf" if math.isinf(dr) else dr,
            "iters": K, "loop_ms": lm, "setup_ms": sm, "speedup_vs_full": full / lm,
            "rd_frac": x["n_rd"] / (cfg.H * cfg.W),
            "tile_frac": x["n_active_tiles"] / x["n_tiles"],
            "cell_frac": x["n_active_cells"] / x["n_items"], "items": x["n_active_items"],
            "item_rows": x["item_rows"], "k_fuse": x["k_fuse"],
            "tile_gpix_iter_s": x["n_active_tiles"] * 1024 * K / lm / 1e6,
            "rd_gpix_iter_s": x["n_rd"] * K / lm / 1e6}), flush=True)
s.close()
