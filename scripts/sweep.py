"""Tuning sweep of the stencil launch configuration (k_fuse x item_rows) on one config.
Prints one JSON line per setting with the K-loop time (CUDA events, median of reps)."""
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
ap.add_argument("--config", default="C3")
ap.add_argument("--kf", default="3,5,7")
ap.add_argument("--rows", default="64,128,256")
ap.add_argument("--delta", type=float, default=math.inf)
ap.add_argument("--iters", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--ctas", default="0", help="cap on stencil CTAs per SM (0 = occupancy)")
ap.add_argument("--ws", default="0", help="RDS_OPT_WS values (warp-specialised stencil)")
ap.add_argument("--pro", default="2", help="RDS_OPT_PROLOGUE values (prologue form)")
args = ap.parse_args()

cfg = wl.CONFIGS[args.config]
K = args.iters or cfg.iters
z, P = wl.make_image(cfg)
st = torch.cuda.Stream()
s = rds.Solver(cfg.H, cfg.W, stream=st.cuda_stream, timing=True)
s.set_image(torch.from_numpy(z).cuda())
s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, torch.from_numpy(P).cuda() if P is not None else None)
am = s.absmax()
delta = wl.band_delta(args.delta, am)
for kf, rows, ctas, ws, pro in [(int(a), int(b), int(c), int(d), int(e))
                                for a in args.kf.split(",") for b in args.rows.split(",")
                                for c in args.ctas.split(",") for d in args.ws.split(",")
                                for e in args.pro.split(",")]:
    if True:
        s.set_option(rds.RDS_OPT_WS, ws)
        s.set_option(rds.RDS_OPT_PROLOGUE, pro)
        s.set_option(rds.RDS_OPT_KFUSE, kf)
        s.set_option(rds.RDS_OPT_ITEM_ROWS, rows)
        s.set_option(rds.RDS_OPT_CTAS_PER_SM, ctas)
        s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, delta, K)  # warm (graph capture)
        s.stats()
        ts = []
        for _ in range(args.reps):
            s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, delta, K)
            ts.append(s.stats()["loop_ms"])
        info = s.stats()
        lm = statistics.median(ts)
        px = info["n_active_tiles"] * 1024
        print(json.dumps({"config": args.config, "kf": kf, "rows": rows, "ctas": ctas, "ws": ws, "pro": pro,
                          "defs": os.environ.get("RDS_NVCC_DEFS", ""), "loop_ms": lm,
                          "gpix_iter_s": px * K / lm / 1e6, "items": info["n_active_items"],
                          "launches": info["launches"]}), flush=True)
s.close()
