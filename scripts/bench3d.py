"""f4 measurement: the 3-D volume path on V1 (256^3, K=200) -- voxel-iterations per second and
the HBM roofline of k_vol_step (36 B per voxel-iteration: read rho1..3, v, c'; write rho1..3,
v), CUDA events on the solve's stream, warm-up first.  One JSON line per delta."""
import argparse
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="V1")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--kz", default="0", help="comma list of planes per z-chunk (0 = auto)")
ap.add_argument("--kf", default="0", help="comma list of iterations per pass (0 = auto)")
args = ap.parse_args()
cfg = wl.VOL_CONFIGS[args.config]
z = wl.make_volume(cfg)
st = torch.cuda.Stream()
s = rds.Solver3(cfg.D, cfg.H, cfg.W, stream=st.cuda_stream)
s.set_image(torch.from_numpy(z).cuda())
s.set_fitting(cfg.c1, cfg.c2)
am = s.absmax()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
n = cfg.D * cfg.H * cfg.W
for kf, kz, dr in [(int(f), int(k), dr) for f in args.kf.split(",") for k in args.kz.split(",")
                   for dr in cfg.delta_rels]:
    s.set_kfuse(kf)
    s.set_kz(kz)
    d = wl.band_delta(dr, am)
    s.solve(cfg.lam, cfg.theta, cfg.tau, d, cfg.iters)  # warm (graph capture)
    ts = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.solve(cfg.lam, cfg.theta, cfg.tau, d, cfg.iters)
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    info = s.stats()
    gv = n * cfg.iters / (ms * 1e-3) / 1e9
    print(json.dumps({"config": cfg.name, "delta_rel": "inf" if math.isinf(dr) else dr,
                      "kf": kf, "iters": cfg.iters, "ms": ms, "gvoxel_iter_s": gv,
                      "rd_frac": info["n_rd"] / n, "kz": info["kz"],
                      "hbm_roofline": {"achieved_gbs": 36 * gv, "peak": peak,
                                       "frac": 36 * gv / peak}}), flush=True)
s.close()
