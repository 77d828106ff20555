"""Cost of the row-strip decomposition (paper_1807_11534_b200/strips.py) on ONE B200.

Runs the G strips of one image one after another on the same device (the in-process form,
`strips.solve_local`, exchange through device buffers) and compares with the whole-image
solve: the ratio is the price of the redundant halo rows plus the per-segment exchange
kernels and host-driven segmenting, i.e. what G GPUs would pay on top of the NCCL transfer
itself (G x the per-strip time would be the multi-GPU critical path).  One JSON line per
(G, seg_iters).  Multi-GPU runs (torchrun, NCCL) use strips.StripSolver; not available here.

usage: python scripts/strips_bench.py [--config C4] [--G 2 4 8] [--seg 7 14 28] [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1807_11534_b200 import rds, strips  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402


def timed(fn, reps):
    st = torch.cuda.current_stream()
    best = None
    for _ in range(reps + 1):  # first call warms up (graphs, allocations)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        t = a.elapsed_time(b)
        best = t if best is None or t < best else best
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--G", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--seg", type=int, nargs="+", default=[7, 14, 28])
    ap.add_argument("--delta-rel", type=float, default=float("inf"))
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.config]
    z, P = wl.make_image(cfg)
    H, W = z.shape
    K = a.iters or cfg.iters
    torch.cuda.set_stream(torch.cuda.Stream())  # torch allocations, events and librds share it
    stream = torch.cuda.current_stream().cuda_stream
    zt = torch.from_numpy(z).cuda()
    Pt = None if P is None else torch.from_numpy(P).cuda()
    whole = rds.Solver(H, W, stream=stream)
    whole.set_image(zt)
    whole.set_fitting(cfg.c1, cfg.c2, cfg.gamma, Pt)
    delta = wl.band_delta(a.delta_rel, whole.absmax())
    par = (cfg.lambdas[0], cfg.theta, cfg.tau)
    t_whole = timed(lambda: whole.solve(*par, delta, K), a.reps)
    print(json.dumps(dict(config=a.config, H=H, W=W, iters=K, delta_rel=a.delta_rel,
                          mode="whole", ms=t_whole)), flush=True)
    u_whole = whole.u()
    whole.close()
    del whole
    for G in a.G:
        for s in a.seg:
            try:
                plan = strips.partition(H, G, s)
            except ValueError as e:
                print(json.dumps(dict(G=G, seg=s, skipped=str(e))))
                continue
            engines = []
            for st in plan:
                e = rds.Solver(st.rows, W, stream=stream)
                e.set_image(zt[st.r0:st.r0 + st.rows].contiguous())
                e.set_fitting(cfg.c1, cfg.c2, cfg.gamma,
                              None if Pt is None else Pt[st.r0:st.r0 + st.rows].contiguous())
                engines.append(e)
            t = timed(lambda: strips.solve_local(engines, plan, *par, delta, K, s,
                                                 device="cuda"), a.reps)
            exact = all((e.u()[st.owned] == u_whole[st.lo:st.hi]).all()
                        for st, e in zip(plan, engines))
            rows = sum(st.rows for st in plan)
            print(json.dumps(dict(config=a.config, G=G, seg=s, mode="strips sequential",
                                  ms=t, over_whole=t / t_whole, held_rows_over_H=rows / H,
                                  segments=len(strips.segments(K, s)),
                                  exchange_mb_per_segment=sum(m for *_, m in
                                                              strips.exchange_plan(plan))
                                  * W * 12 / 1e6,
                                  bitwise_equal_u=bool(exact))), flush=True)
            for e in engines:
                e.close()
            del engines


if __name__ == "__main__":
    main()
