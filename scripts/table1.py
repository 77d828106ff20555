"""The paper's evaluation protocol (§4, Table 1 and the Fig. 3 timing
study) on the synthetic stand-in images: for each q, the restricted solve (q -> q^ by
rds_band_for_fraction) run to the paper's delta_stop = 1e-2 with the fused stopping rule,
E1 (Tanimoto) and E2 (L2) against u^GT = the unrestricted float64 solve to 1e-10
(rds_solve_gt), and the GPU time of the restricted solve -- on the dense stencil and on the
compacted RD path (f3, RDS_OPT_COMPACT = 1), whose cost follows q.  One JSON line per q.
The paper's own images are not distributed (PAPER.md:160-195 are [FIGURE] placeholders), so
its Table 1 values are context, not targets."""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C0")
ap.add_argument("--lam", type=float, default=0.0)
ap.add_argument("--qs", default="0,0.05,0.1,0.2,0.3,0.4,0.6,0.8,1")
ap.add_argument("--stop", type=float, default=1e-2, help="delta_stop of the proposed method")
ap.add_argument("--gt-tol", type=float, default=1e-10)
ap.add_argument("--check-every", type=int, default=10)
ap.add_argument("--max-iters", type=int, default=2000000)
args = ap.parse_args()

cfg = wl.CONFIGS[args.config]
lam = args.lam or cfg.lambdas[0]
z, P = wl.make_image(cfg)
st = torch.cuda.Stream()
s = rds.Solver(cfg.H, cfg.W, stream=st.cuda_stream, timing=True)
s.set_image(z)
s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(st)
gt = s.solve_gt(lam, cfg.theta, cfg.tau, math.inf, args.max_iters, args.gt_tol,
                args.check_every)
ev1.record(st)
ev1.synchronize()
print(json.dumps({"config": cfg.name, "gt": gt, "gt_ms": ev0.elapsed_time(ev1),
                  "lambda": lam}), flush=True)
c = rds.Solver(cfg.H, cfg.W, stream=st.cuda_stream, timing=True, compact=1)
c.set_image(z)
c.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
for q in [float(x) for x in args.qs.split(",")]:
    delta = s.band_for_fraction(q)
    r = s.solve_tol(lam, cfg.theta, cfg.tau, delta, args.max_iters, args.stop,
                    args.check_every)  # warm (graph capture)
    r = s.solve_tol(lam, cfg.theta, cfg.tau, delta, args.max_iters, args.stop,
                    args.check_every)
    e1, e2 = s.compare_gt(0.5)
    rc = c.solve_tol(lam, cfg.theta, cfg.tau, delta, args.max_iters, args.stop,
                     args.check_every)
    rc = c.solve_tol(lam, cfg.theta, cfg.tau, delta, args.max_iters, args.stop,
                     args.check_every)
    print(json.dumps({"q": q, "delta": float(delta), "iters": r["iters"],
                      "residual": r["residual"], "E1": e1, "E2": e2,
                      "rd_frac": r["n_rd"] / (cfg.H * cfg.W), "loop_ms": r["loop_ms"],
                      "setup_ms": r["setup_ms"], "compact_iters": rc["iters"],
                      "compact_loop_ms": rc["loop_ms"], "compact_setup_ms": rc["setup_ms"]}),
          flush=True)
s.close()
c.close()
