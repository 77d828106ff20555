"""Resident grid (k_grid) vs the stencil / compact path on a config: K-loop time per delta
(stats loop_ms, CUDA events on the handle's stream), median of reps; bit-identity checked."""
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

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
shape = None
if "x" in name:
    shape = tuple(int(x) for x in name.split("x"))
    cfg = wl.CONFIGS["C1"]
    z = wl.random_image(*shape, seed=3)
    P = None
else:
    cfg = wl.CONFIGS[name]
    z, P = wl.make_image(cfg)
H, W = z.shape
st = torch.cuda.Stream()
out = {}
for mode, kw in (("stencil", dict(grid=0, compact=0, resident=0)), ("default_nogrid", dict(grid=0)),
                 ("grid", dict(grid=1, resident=0))):
    s = rds.Solver(H, W, stream=st.cuda_stream, timing=True, **kw)
    s.set_image(torch.from_numpy(z).cuda())
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, torch.from_numpy(P).cuda() if P is not None else None)
    am = s.absmax()
    for dr in (0.05, 0.1, 0.2, 0.4, math.inf):
        d = wl.band_delta(dr, am)
        s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, d, cfg.iters)
        ts = []
        for _ in range(5):
            s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, d, cfg.iters)
            ts.append(s.stats()["loop_ms"])
        info = s.stats()
        u = s.u()
        key = str(dr)
        if mode == "stencil":
            out[key] = u
            same = True
        else:
            same = bool(np.array_equal(out[key], u))
        lm = statistics.median(ts)
        print(json.dumps({"config": name, "mode": mode, "delta_rel": key, "loop_ms": lm,
                          "gpx_iter_s": H * W * cfg.iters / lm / 1e6,
                          "resident": info["resident"], "compact": info["compact"],
                          "same_as_stencil": same}), flush=True)
    s.close()
