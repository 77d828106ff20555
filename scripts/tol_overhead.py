"""Cost of the fused stopping rule: K-loop time of rds_solve (fixed K) vs rds_solve_tol with
tol = 0 (runs all K iterations, every check evaluated) for several check intervals."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = wl.CONFIGS[name]
z, P = wl.make_image(cfg)
st = torch.cuda.Stream()
s = rds.Solver(cfg.H, cfg.W, stream=st.cuda_stream, timing=True)
s.set_image(torch.from_numpy(z).cuda())
s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, torch.from_numpy(P).cuda() if P is not None else None)
d = wl.band_delta(0.2, s.absmax())
K = cfg.iters


def timed(fn, reps=3):
    fn()
    s.stats()
    ts = []
    for _ in range(reps):
        fn()
        ts.append(s.stats()["loop_ms"])
    return statistics.median(ts)


base = timed(lambda: s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, d, K))
print(json.dumps({"config": name, "mode": "fixed K", "loop_ms": base}), flush=True)
kf = s.stats()["k_fuse"]
for m in (kf, 2 * kf, 5 * kf, 10 * kf):
    t = timed(lambda: s.solve_tol(cfg.lambdas[0], cfg.theta, cfg.tau, d, K, 0.0, m))
    print(json.dumps({"config": name, "mode": f"tol, check every {m}", "loop_ms": t,
                      "overhead": t / base - 1}), flush=True)
s.close()
