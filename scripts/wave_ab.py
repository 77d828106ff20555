"""A/B of the temporal wavefront (RDS_OPT_WAVE) against the launch-per-block K-loop: per
config and delta, the K-loop time (CUDA events, median of reps) for each k_fuse, and a
bitwise comparison of the wave and non-wave results.  One JSON line per setting."""
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
ap.add_argument("--kf", default="4,5,6,7")
ap.add_argument("--deltas", default="inf")
ap.add_argument("--iters", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--check", action="store_true", help="compare u/v/rho bitwise wave vs not")
args = ap.parse_args()

cfg = wl.CONFIGS[args.config]
K = args.iters or cfg.iters
z, P = wl.make_image(cfg)
st = torch.cuda.Stream()
zt = torch.from_numpy(z).cuda()
Pt = torch.from_numpy(P).cuda() if P is not None else None


def solver(kf, wave):
    s = rds.Solver(cfg.H, cfg.W, stream=st.cuda_stream, timing=True, k_fuse=kf, wave=wave)
    s.set_image(zt)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, Pt)
    return s


for dr in [float(x) for x in args.deltas.split(",")]:
    for kf in [int(k) for k in args.kf.split(",")]:
        res = {}
        for wave in (0, 1):
            s = solver(kf, wave)
            delta = wl.band_delta(dr, s.absmax())
            s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, delta, K)
            s.stats()
            ts = []
            for _ in range(args.reps):
                s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, delta, K)
                ts.append(s.stats()["loop_ms"])
            info = s.stats()
            lm = statistics.median(ts)
            px = min(info["n_active_tiles"] * 1024, cfg.H * cfg.W)
            row = {"config": args.config, "delta_rel": "inf" if math.isinf(dr) else dr,
                   "kf": kf, "wave": info["wave"], "loop_ms": lm, "setup_ms": info["setup_ms"],
                   "gpix_iter_s": px * K / lm / 1e6, "launches": info["launches"]}
            if args.check:
                p1, p2 = s.p()
                res[wave] = (s.u(), s.v(), p1, p2, s.mask())
            print(json.dumps(row), flush=True)
            s.close()
        if args.check:
            same = all(np.array_equal(a, b) for a, b in zip(res[0], res[1]))
            print(json.dumps({"config": args.config, "kf": kf, "delta_rel": str(dr),
                              "bitwise_equal": same}), flush=True)
