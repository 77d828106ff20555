"""k_grid K-loop time on C1 (or HxW) at delta = inf: one JSON line (timing experiments)."""
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
cfg = wl.CONFIGS["C1"]
if "x" in name:
    H, W = (int(x) for x in name.split("x"))
    z, P = wl.random_image(H, W, seed=3), None
else:
    cfg = wl.CONFIGS[name]
    z, P = wl.make_image(cfg)
    H, W = z.shape
st = torch.cuda.Stream()
s = rds.Solver(H, W, stream=st.cuda_stream, timing=True, grid=1, resident=0)
s.set_image(torch.from_numpy(z).cuda())
s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, torch.from_numpy(P).cuda() if P is not None else None)
d = wl.band_delta(math.inf, s.absmax())
s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, d, cfg.iters)
ts = []
for _ in range(5):
    s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, d, cfg.iters)
    ts.append(s.stats()["loop_ms"])
lm = statistics.median(ts)
print(json.dumps({"config": name, "defs": os.environ.get("RDS_NVCC_DEFS", ""), "loop_ms": lm,
                  "us_per_iter": lm * 1e3 / cfg.iters, "gpx_iter_s": H * W * cfg.iters / lm / 1e6,
                  "resident": s.stats()["resident"]}), flush=True)
