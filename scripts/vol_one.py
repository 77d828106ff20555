"""One V1 solve (256^3, K = 20, delta = .2) for an ncu capture of the 3-D step kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

cfg = wl.VOL_CONFIGS["V1"]
z = wl.make_volume(cfg)
s = rds.Solver3(cfg.D, cfg.H, cfg.W)
s.set_image(torch.from_numpy(z).cuda())
s.set_fitting(cfg.c1, cfg.c2)
d = wl.band_delta(0.2, s.absmax())
for _ in range(2):
    s.solve(cfg.lam, cfg.theta, cfg.tau, d, 20)
torch.cuda.synchronize()
print(s.stats())
