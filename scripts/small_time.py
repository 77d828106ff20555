"""Median K-loop time of fixed-K solves on the resident cluster (k_small) for the paper's image
size (C0 128 x 128, K = 200) and neighbours (64^2, 256^2), delta = inf and 0.2 max|f|."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

cfg = wl.CONFIGS["C0"]
for n in (64, 128, 256):
    if n == 128:
        z, _ = wl.make_image(cfg)
    else:
        z = wl.make_image(cfg)[0]
        z = np.resize(z, (n, n)).astype(np.float32)
    s = rds.Solver(n, n, resident=1, timing=True)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2)
    am = s.absmax()
    for dr in (float("inf"), 0.2):
        d = wl.band_delta(dr, am)
        ts = []
        for _ in range(25):
            s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, d, cfg.iters)
            ts.append(s.stats()["loop_ms"])
        st = s.stats()
        print(json.dumps({"n": n, "delta_rel": str(dr), "loop_ms": statistics.median(ts[5:]),
                          "resident": st["resident"]}), flush=True)
    s.close()
torch.cuda.synchronize()
