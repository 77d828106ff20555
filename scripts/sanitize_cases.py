"""Small cases that launch every librds kernel once or more (2-D solves in every launch mode,
ragged and aligned widths, tolerance solves, q search, energies, fp64 mode and E1/E2, 3-D,
batches) -- the program run under compute-sanitizer (one tool per gpurun call).  numpy only."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402

rng = np.random.default_rng(0)
for (H, W, kf) in [(37, 61, 0), (64, 128, 7), (5, 3, 2), (130, 250, 5)]:
    z = rng.uniform(0, 1, (H, W)).astype(np.float32)
    s = rds.Solver(H, W, k_fuse=kf)
    s.set_image(z)
    s.set_fitting(0.75, 0.25)
    d = 0.3 * s.absmax()
    s.solve(4.0, 0.1, 0.125, d, 23)
    s.u(), s.mask(), s.v(), s.p(), s.labels(), s.fitting(), s.active_tiles(), s.energy()
    st = s.solve_tol(4.0, 0.1, 0.125, d, 40, 1e-3, 3)
    s.set_state(s.v(), *s.p())
    s.solve(4.0, 0.1, 0.125, math.inf, 9)
    s.solve_q(4.0, 0.1, 0.125, 0.4, 5)
    s.solve_gt(4.0, 0.1, 0.125, math.inf, 50, 1e-6, 7)
    s.u_gt(), s.compare_gt(0.5)
    s.close()
zb = rng.uniform(0, 1, (3, 33, 45)).astype(np.float32)
b = rds.BatchSolver(3, 33, 45)
b.set_image(zb)
b.set_fitting(0.75, 0.25)
b.solve(4.0, 0.1, 0.125, 0.3, 17)
b.u(), b.mask(), b.p(), b.energy()
b.close()
zv = rng.uniform(0, 1, (9, 20, 37)).astype(np.float32)
v = rds.Solver3(*zv.shape)
v.set_image(zv)
v.set_fitting(0.75, 0.25)
v.solve(4.0, 0.1, 1 / 12, 0.3, 11)
v.u(), v.mask(), v.p(), v.labels(), v.stats()
v.close()
print("sanitize cases done")
