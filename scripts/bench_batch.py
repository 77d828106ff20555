"""Serving many small images: B images of the paper's size (C0 recipe, 128 x 128, seeds
0..B-1) solved as one batch (rds_create_batch) vs one image at a time; K = 200, delta = inf.
Prints pixel-iterations per second for both (CUDA events, warm-up first)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

K = 200
st = torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


single = rds.Solver(128, 128, stream=st.cuda_stream)
z0 = wl.gen_disk(128, 128, seed=0)
single.set_image(torch.from_numpy(z0).cuda())
single.set_fitting(0.8, 0.2)
ms1 = timed(lambda: single.solve(5.0, 0.1, 0.125, np.float32(np.inf), K))
print(json.dumps({"mode": "one image", "images": 1, "ms": ms1,
                  "gpix_iter_s": 128 * 128 * K / (ms1 * 1e-3) / 1e9}), flush=True)
single.close()
for B in (64, 256, 1024):
    z = np.stack([wl.gen_disk(128, 128, seed=b) for b in range(B)])
    s = rds.BatchSolver(B, 128, 128, stream=st.cuda_stream)
    s.set_image(torch.from_numpy(z.reshape(B * 128, 128)).cuda())
    s.set_fitting(0.8, 0.2)
    ms = timed(lambda: s.solve(5.0, 0.1, 0.125, np.float32(np.inf), K))
    print(json.dumps({"mode": "batch", "images": B, "ms": ms, "ms_per_image": ms / B,
                      "gpix_iter_s": B * 128 * 128 * K / (ms * 1e-3) / 1e9,
                      "speedup_vs_one_at_a_time": B * ms1 / ms}), flush=True)
    s.close()
