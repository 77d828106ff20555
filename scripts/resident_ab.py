"""K-loop time of small images on the resident cluster (RDS_OPT_RESIDENT) vs the stencil:
C0 (the paper's 128 x 128 size, K = 200) and larger squares; one JSON line per case."""
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

cases = [("C0", None)] + [(f"rand{n}", n) for n in (64, 256)]
st = torch.cuda.Stream()
for name, n in cases:
    if n is None:
        cfg = wl.CONFIGS["C0"]
        z, _ = wl.make_image(cfg)
        K, drs = cfg.iters, cfg.delta_rels
    else:
        z = wl.gen_voronoi(N=n, seed=n, n_sites=20)[:n, :n].copy()
        K, drs = 200, (0.2, math.inf)
    for dr in drs:
        row = {"case": name, "H": z.shape[0], "W": z.shape[1], "K": K,
               "delta_rel": "inf" if math.isinf(dr) else dr}
        for res, per in ((0, 0), (0, 1), (1, 0)):
            s = rds.Solver(*z.shape, stream=st.cuda_stream, timing=True, resident=res,
                           persist=per)
            s.set_image(z)
            s.set_fitting(0.8, 0.2)
            d = wl.band_delta(dr, s.absmax())
            ts = []
            for _ in range(6):
                s.solve(5.0, 0.1, 0.125, d, K)
                ts.append(s.stats()["loop_ms"] + s.stats()["setup_ms"])
            info = s.stats()
            path = "resident" if info["resident"] else ("persist" if info["persist"] else "stencil")
            row[f"{path}_solve_ms"] = statistics.median(ts[1:])
            s.close()
        print(json.dumps(row), flush=True)
