"""One fixed-K solve through the temporal wavefront (for ncu captures of k_wave)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--kf", type=int, default=6)
ap.add_argument("--iters", type=int, default=0)
ap.add_argument("--wave", type=int, default=1)
args = ap.parse_args()
cfg = wl.CONFIGS[args.config]
z, P = wl.make_image(cfg)
s = rds.Solver(cfg.H, cfg.W, k_fuse=args.kf, wave=args.wave, timing=True)
s.set_image(z)
s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
d = wl.band_delta(float("inf"), s.absmax())
for _ in range(2):
    s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, d, args.iters or cfg.iters)
print(s.stats())
torch.cuda.synchronize()
