"""f3: dense stencil vs compacted RD iteration (RDS_OPT_COMPACT) per delta on one config.
One JSON line per delta: K-loop ms of both paths (CUDA events, median of reps; the compact
path's setup includes building the RD index), RD fraction, speedup of each path over the
dense delta = inf solve, and whether the two paths gave the same u."""
import argparse
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--deltas", type=float, nargs="+", default=[0.02, 0.05, 0.1, 0.2])
ap.add_argument("--iters", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()

cfg = wl.CONFIGS[args.config]
K = args.iters or cfg.iters
z, P = wl.make_image(cfg)
st = torch.cuda.Stream()
zt = torch.from_numpy(z).cuda()
Pt = torch.from_numpy(P).cuda() if P is not None else None
solvers = {}
for mode in (0, 1):
    s = rds.Solver(cfg.H, cfg.W, stream=st.cuda_stream, timing=True, compact=mode)
    s.set_image(zt)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, Pt)
    solvers[mode] = s
am = solvers[0].absmax()
par = (cfg.lambdas[0], cfg.theta, cfg.tau)


def timed(s, d):
    s.solve(*par, d, K)
    s.stats()
    ts, ss = [], []
    for _ in range(args.reps):
        s.solve(*par, d, K)
        x = s.stats()
        ts.append(x["loop_ms"])
        ss.append(x["setup_ms"])
    return statistics.median(ts), statistics.median(ss), x


full = timed(solvers[0], np.float32(math.inf))[0]
for dr in args.deltas:
    d = wl.band_delta(dr, am)
    ld, sd, xd = timed(solvers[0], d)
    ud = solvers[0].u()
    lc, sc, xc = timed(solvers[1], d)
    same = bool(np.array_equal(ud, solvers[1].u()))
    print(json.dumps({
        "config": cfg.name, "delta_rel": dr, "iters": K, "rd_frac": xd["n_rd"] / (cfg.H * cfg.W),
        "tile_frac": xd["n_active_tiles"] / xd["n_tiles"],
        "dense_loop_ms": ld, "dense_setup_ms": sd, "compact_loop_ms": lc,
        "compact_setup_ms": sc, "compact_used": xc["compact"],
        "speedup_dense_vs_full": full / ld, "speedup_compact_vs_full": full / (lc + sc - sd),
        "compact_over_dense": (ld) / (lc + sc - sd), "same_u": same,
        "rd_gpix_iter_s_compact": xd["n_rd"] * K / (lc * 1e-3) / 1e9,
        "rd_gpix_iter_s_dense": xd["n_rd"] * K / (ld * 1e-3) / 1e9}), flush=True)
