"""Balance of the row-strip cuts for restricted solves on ONE B200: each strip's own solve
(its rows, K iterations, no exchange) timed alone, for the near-equal cuts and the
weighted cuts of strips.row_weights from the GPU's band labels (active 8 x 112 cells per row
band, or RD pixels per row).  The
slowest strip is the critical path of a G-GPU run; the balance whole / (G x slowest) is its
parallel efficiency before the halo exchange.  One JSON line per (config, delta, G, cuts)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1807_11534_b200 import rds, strips  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402


def timed(fn, reps=3):
    st = torch.cuda.current_stream()
    best = None
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        t = a.elapsed_time(b)
        best = t if best is None or t < best else best
    return best


ap = argparse.ArgumentParser()
ap.add_argument("--config", nargs="+", default=["C2", "C4"])
ap.add_argument("--delta-rel", type=float, nargs="+", default=[0.1, 0.2])
ap.add_argument("--G", type=int, nargs="+", default=[2, 4, 8])
ap.add_argument("--seg", type=int, default=14)
ap.add_argument("--iters", type=int, default=200)
a = ap.parse_args()
torch.cuda.set_stream(torch.cuda.Stream())
stream = torch.cuda.current_stream().cuda_stream
for name in a.config:
    cfg = wl.CONFIGS[name]
    z, P = wl.make_image(cfg)
    H, W = z.shape
    zt = torch.from_numpy(z).cuda()
    Pt = None if P is None else torch.from_numpy(P).cuda()
    whole = rds.Solver(H, W, stream=stream)
    whole.set_image(zt)
    whole.set_fitting(cfg.c1, cfg.c2, cfg.gamma, Pt)
    am = whole.absmax()
    par = (cfg.lambdas[0], cfg.theta, cfg.tau)
    for dr in a.delta_rel:
        delta = wl.band_delta(dr, am)
        whole.solve(*par, delta, 0)
        lab = whole.labels()
        wts = {"equal": None, "cells": strips.row_weights(lab),
               "pixels": strips.row_weights(lab, cell=None)}
        t_whole = timed(lambda: whole.solve(*par, delta, a.iters))
        for G in a.G:
            for cuts in ("equal", "cells", "pixels"):
                plan = strips.partition(H, G, a.seg, wts[cuts])
                ts = []
                for st in plan:
                    e = rds.Solver(st.rows, W, stream=stream)
                    e.set_image(zt[st.r0:st.r0 + st.rows].contiguous())
                    e.set_fitting(cfg.c1, cfg.c2, cfg.gamma,
                                  None if Pt is None else Pt[st.r0:st.r0 + st.rows].contiguous())
                    ts.append(timed(lambda: e.solve(*par, delta, a.iters)))
                    e.close()
                print(json.dumps(dict(config=name, delta_rel=dr, G=G, cuts=cuts, iters=a.iters,
                                      whole_ms=t_whole, max_strip_ms=max(ts),
                                      strip_ms=[round(t, 4) for t in ts],
                                      rows=[st.hi - st.lo for st in plan],
                                      balance=t_whole / (G * max(ts)))), flush=True)
    whole.close()
