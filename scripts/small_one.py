"""One fixed-K solve of the paper's image size (C0, 128 x 128, K = 200, delta = inf) on the
resident cluster (for ncu captures of k_small)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

cfg = wl.CONFIGS["C0"]
z, _ = wl.make_image(cfg)
s = rds.Solver(cfg.H, cfg.W, resident=1)
s.set_image(z)
s.set_fitting(cfg.c1, cfg.c2)
for _ in range(3):
    s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, float("inf"), cfg.iters)
print(s.stats())
torch.cuda.synchronize()
