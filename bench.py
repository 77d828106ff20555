#!/usr/bin/env python
"""Benchmark of the restricted-domain dual iteration on B200 (BASELINE.json metric).

Workload (default): C3 = BASELINE.json configs[3], the headline -- 4096x4096 Voronoi image
(200 cells, sigma 0.15), Chan-Vese f (c1=.8, c2=.2), lambda=5, theta=.1, tau=.125,
K=1000 iterations, delta in {0.1, 0.2, 0.4, inf} * max|f|.  One step = the whole hot path
(fused fitting/band/init, tile compaction, K iterations, output u/mask, energy and gap) for
every delta of the sweep.

Metric: active Gpixel-iter/s = sum over the sweep of (pixels in active 32x32 tiles) x K,
divided by the step time; higher is better.  Also reported: RD-pixel-iter/s, restricted vs
full speedup per delta, the stencil kernel's roofline, the CPU oracle baseline, e2e through
the C ABI with host buffers, clocks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 (torchrun): replicas only -- every rank solves the same workload on its own GPU, no
data-path collective; value = all ranks' work / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1807_11534_b200 import workloads as wl  # noqa: E402

METRIC = "active Gpixel-iter/s at 4096^2 fp32 (restricted-domain dual iteration, C3 delta sweep)"


def _metric(cfg):
    """BASELINE.json's metric on the headline config C3; the same quantity, named for its own
    image size, on the other configs (parity-test cases run through --config)."""
    if cfg.name == "C3":
        return METRIC
    return (f"active Gpixel-iter/s at {cfg.H}x{cfg.W} fp32 (restricted-domain dual iteration, "
            f"{cfg.name} delta sweep)")


def _l2_note(cfg):
    ws = 28 * cfg.H * cfg.W / 2**20  # rho1, rho2, v, c read + rho1, rho2, v written, fp32
    if ws > 126e6 / 2**20:
        return f"no flush: per-iteration working set {ws:.0f} MiB > 126 MB L2"
    return (f"no flush: per-iteration working set {ws:.1f} MiB fits the 126 MB L2 (not the "
            f"headline config; an L2-resident solve is what this size runs as)")
UNIT = "Gpixel-iter/s"
BYTES_PER_PX_ITER = 28  # read rho1, rho2, v, c (16 B) + write rho1, rho2, v (12 B)
# Compute roofline of one pixel-iteration: 2 MUFU ops (sqrt, rcp) on the
# 16-lane/clk/SM MUFU pipe and 15 FP32 ops on the 128-lane/clk/SM FMA pipe (both measured
# in scripts/micro/); MUFU binds: 8 pixel-iterations per clock per SM.
MUFU_PER_PX_ITER = 2
FP32_PER_PX_ITER = 15
MUFU_LANES_PER_SM = 16
FP32_LANES_PER_SM = 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--kf", type=int, default=0, help="iterations per HBM round trip (0=lib default)")
    ap.add_argument("--rows", type=int, default=0, help="rows per work item (0=lib default)")
    ap.add_argument("--iters", type=int, default=0, help="override K (diagnostics only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layout", default="replicas", choices=["replicas", "strips"],
                    help="N>1: independent replicas (default, weak scaling) or one image in "
                         "row strips with halo exchange (strong scaling)")
    ap.add_argument("--seg", type=int, default=28, help="strips: iterations between halo "
                                                       "refreshes")
    ap.add_argument("--no-compact", action="store_true",
                    help="skip the f3 compacted-RD section (restricted_compact)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


# ------------------------------------------------------------------------------------------
# distributed plumbing (replicas)
# ------------------------------------------------------------------------------------------

class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            backend = "nccl" if _cuda() else "gloo"
            if _cuda():
                torch.cuda.set_device(self.local)  # bind this rank's GPU before NCCL init
            dist.init_process_group(backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            import torch

            if _cuda():
                self.pg.barrier(device_ids=[self.local])
            else:
                self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cuda" if _cuda() else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cuda" if _cuda() else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


def _cuda():
    import torch

    return torch.cuda.is_available()


def throughput(total_work: float, t_ms: float) -> float:
    """Whole-job Gpixel-iter/s: work summed over ranks / max-over-ranks device time."""
    return total_work / (t_ms * 1e-3) / 1e9


# ------------------------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ------------------------------------------------------------------------------------------

class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# CPU oracle baseline / reference arm
# ------------------------------------------------------------------------------------------

def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_rate(cfg, z, P, deltas_rel, seconds, iters_hint=None, threads=0):
    """Time the oracle (as it stands) on the full image with a bounded iteration count,
    following BASELINE.md §3: the timed region is the oracle's K-loop alone
    (oracle.last_loop_seconds(): no labels, initialisation, allocation or copies); labels and
    active tiles for the work count are formed outside it.  Returns (px-iter/s counted like
    the GPU metric, threads used, sample description, loop seconds)."""
    import oracle

    oracle.set_threads(threads or (os.cpu_count() or 1))
    f = oracle.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)
    am = oracle.absmax(f)
    lam = cfg.lambdas[0]
    if iters_hint:
        per_delta = iters_hint
    else:  # calibrate on 2 loop iterations at delta = inf
        oracle.solve(f, np.inf, lam, np.float32(cfg.theta), cfg.tau, 2)
        t_it = max(oracle.last_loop_seconds() / 2, 1e-6)
        per_delta = max(2, int(seconds / t_it / len(deltas_rel)))
    work, dt = 0, 0.0
    for dr in deltas_rel:
        delta = wl.band_delta(dr, am)
        n_act = len(oracle.tiles(oracle.labels(f, delta), 32, 32)) * 32 * 32
        oracle.solve(f, delta, lam, np.float32(cfg.theta), cfg.tau, per_delta)
        dt += oracle.last_loop_seconds()
        work += min(n_act, cfg.H * cfg.W) * per_delta
    used = oracle.get_threads()
    sample = (f"oracle fp64 K-loop only (setup excluded) on the full {cfg.H}x{cfg.W} "
              f"{cfg.name} image, {per_delta} iterations per delta for delta_rel in "
              f"{_js(list(deltas_rel))} (of K={cfg.iters}), {used} OpenMP threads")
    return work / dt, used, sample, dt


def cpu_baseline(cfg, z, P, seconds):
    """cpu_baseline object: all host cores; plus one thread for configs up to 2048^2
    (BASELINE.md §3)."""
    r, cores, sample, dt = oracle_rate(cfg, z, P, cfg.delta_rels, seconds)
    out = {"value": r / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
           "loop_s": dt, "cpu_model": cpu_model(), "nproc": os.cpu_count()}
    if cfg.H * cfg.W <= 2048 * 2048:
        r1, _, s1, dt1 = oracle_rate(cfg, z, P, cfg.delta_rels, seconds / 2, threads=1)
        out["single_thread"] = {"value": r1 / 1e9, "unit": UNIT, "cores": 1, "sample": s1,
                                "loop_s": dt1}
    import oracle

    oracle.set_threads(os.cpu_count() or 1)
    return out


REF_ITERS_PER_DELTA = 20


def run_reference(args, dist):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only).  Each step runs
    REF_ITERS_PER_DELTA iterations per delta on the full image; the step time is the sum of
    the oracle's K-loop times (setup excluded)."""
    if dist.rank != 0:
        return
    cfg = wl.CONFIGS[args.config]
    z, P = wl.make_image(cfg)
    import oracle

    oracle.build()
    for _ in range(args.warmup):
        oracle_rate(cfg, z, P, cfg.delta_rels, 0, iters_hint=2)
    times, works = [], []
    for _ in range(args.steps):
        r, cores, sample, dt = oracle_rate(cfg, z, P, cfg.delta_rels, 0,
                                           iters_hint=REF_ITERS_PER_DELTA)
        times.append(dt)
        works.append(r * dt)
    value = sum(works) / sum(times) / 1e9
    line = {
        "impl": "reference", "metric": _metric(cfg), "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.desc}", "delta_rels": _js(cfg.delta_rels),
                   "iters_per_step_per_delta": REF_ITERS_PER_DELTA, "iters_of_config": cfg.iters},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample, "cpu_model": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _js(xs):
    return [("inf" if (isinstance(x, float) and math.isinf(x)) else x) for x in xs]


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------

def run_ours(args, dist):
    import torch

    assert torch.cuda.is_available(), "bench.py --impl ours needs a CUDA device"
    torch.cuda.set_device(dist.local)
    from paper_1807_11534_b200 import rds

    cfg = wl.CONFIGS[args.config]
    K = args.iters or cfg.iters
    lam = cfg.lambdas[0]
    z, P = wl.make_image(cfg)
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    s = rds.Solver(cfg.H, cfg.W, stream=sp, k_fuse=args.kf, item_rows=args.rows, timing=True)
    zt = torch.from_numpy(z).cuda()
    Pt = torch.from_numpy(P).cuda() if P is not None else None
    s.set_image(zt)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, Pt)
    am = s.absmax()
    deltas = [wl.band_delta(dr, am) for dr in cfg.delta_rels]

    def step(collect=None):
        for dr, d in zip(cfg.delta_rels, deltas):
            s.solve(lam, cfg.theta, cfg.tau, d, K)
            e = s.energy()  # S8, synchronises the stream
            if collect is not None:
                st = s.stats()
                collect.append((dr, st, e))

    # warm-up (also captures the K-loop graphs)
    for _ in range(max(args.warmup, 3)):
        step()
    # per-delta characterisation (untimed pass with per-solve event times)
    info = []
    step(info)
    torch.cuda.synchronize()

    clocks = Clocks(dist.local)
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    loop_ms = []
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for _ in range(args.steps):
            for dr, d in zip(cfg.delta_rels, deltas):
                s.solve(lam, cfg.theta, cfg.tau, d, K)
                s.energy()
                loop_ms.append((dr, s.stats()))
        ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    ck = clocks.stop()
    t_ms = dist.max(ev0.elapsed_time(ev1))

    # work accounting
    act_px = {dr: st["n_active_tiles"] * 32 * 32 for dr, st, _ in info}
    act_px = {dr: min(v, cfg.H * cfg.W) for dr, v in act_px.items()}  # ragged tiles clipped
    rd_px = {dr: st["n_rd"] for dr, st, _ in info}
    work_step = sum(act_px[dr] for dr in cfg.delta_rels) * K
    rd_step = sum(rd_px[dr] for dr in cfg.delta_rels) * K
    total_work = dist.sum(work_step * args.steps)
    value = throughput(total_work, t_ms)
    ms_per_step = t_ms / args.steps

    # stencil roofline: the K-loop is only stencil launches; average per-launch duration
    per = {}
    for dr, st in loop_ms:
        per.setdefault(dr, []).append(st)
    per_delta = []
    t_full = statistics.median(x["loop_ms"] for x in per[cfg.delta_rels[-1]]) \
        if math.isinf(cfg.delta_rels[-1]) else None
    launch_ms_all, bytes_all, pxit_all = [], [], []
    for dr, st, e in info:
        lm = statistics.median(x["loop_ms"] for x in per[dr])
        sm = statistics.median(x["setup_ms"] for x in per[dr])
        n_items = st["n_active_cells"]
        item_px = n_items * st["item_rows"] * st["item_cols"]
        launches = st["launches"]
        px = act_px[dr]
        path = "compact" if st["compact"] else ("resident" if st.get("resident") else "stencil")
        if path == "stencil":  # the stencil's roofline: its launches only
            launch_ms_all.append(lm / launches)
            bytes_all.append(BYTES_PER_PX_ITER * px * K / launches)
            pxit_all.append(px * K / launches)
        per_delta.append({
            "delta_rel": "inf" if math.isinf(dr) else dr, "path": path,
            "loop_ms": lm, "setup_ms": sm,
            "active_tile_frac": st["n_active_tiles"] / st["n_tiles"],
            "rd_frac": st["n_rd"] / (cfg.H * cfg.W),
            "rd_decoupled_frac": st["rdc_decoupled"] / max(1, st["n_rd"]),
            "rd_grouped_frac": st["rdc_grouped"] / max(1, st["n_rd"]),
            "active_cell_frac": n_items / st["n_items"], "work_items": st["n_active_items"],
            "tile_gpix_iter_s": px * K / (lm * 1e-3) / 1e9,
            "rd_gpix_iter_s": st["n_rd"] * K / (lm * 1e-3) / 1e9,
            "speedup_vs_full": (t_full / lm) if t_full else None,
            "gap": e["gap"], "E_v": e["E_v"],
        })
    kernel = "k_stencil"
    if not launch_ms_all:  # no delta ran on the stencil (small images: the resident cluster)
        kernel = "+".join(sorted({p["path"] for p in per_delta}))
        for p in per_delta:
            px = act_px[p["delta_rel"] if p["delta_rel"] != "inf" else math.inf]
            launch_ms_all.append(p["loop_ms"])
            bytes_all.append(BYTES_PER_PX_ITER * px * K)
            pxit_all.append(px * K)
    launch_ms = statistics.mean(launch_ms_all)
    bytes_per_launch = statistics.mean(bytes_all)
    achieved_gbs = bytes_per_launch / (launch_ms * 1e-3) / 1e9
    peaks = _peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    clock_mhz = ck.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    n_sm = torch.cuda.get_device_properties(dist.local).multi_processor_count
    px_per_clk_sm = min(MUFU_LANES_PER_SM / MUFU_PER_PX_ITER, FP32_LANES_PER_SM / FP32_PER_PX_ITER)
    alu_peak = n_sm * px_per_clk_sm * clock_mhz * 1e6 / 1e9  # Gpx-iter/s at the observed clock
    achieved_px = statistics.mean(pxit_all) / (launch_ms * 1e-3) / 1e9
    st0 = info[0][1]
    traffic = _traffic_from_profile(st0["k_fuse"])
    # K3 fuses k_fuse iterations per HBM round trip, so it is bound by its arithmetic (the MUFU
    # and FMA pipes), not by HBM: the primary roofline is the compute one; the
    # HBM roofline of the minimum-traffic one-iteration-per-pass schedule (north_star, SURVEY
    # §8(d) R1) is reported beside it and exceeds 1 by design.
    roofline = {
        "bound": "alu", "kernel": kernel, "achieved": achieved_px, "peak": alu_peak,
        "unit": "Gpixel-iter/s", "frac": achieved_px / alu_peak,
        "traffic": traffic,
        "basis": (f"active pixel-iterations per launch / mean launch time {launch_ms:.4f} ms; "
                  f"peak = {n_sm} SM x {px_per_clk_sm:g} px-iter/clk (MUFU: {MUFU_PER_PX_ITER} "
                  f"ops per px-iter at {MUFU_LANES_PER_SM}/clk/SM; FMA pipe: {FP32_PER_PX_ITER} "
                  f"at {FP32_LANES_PER_SM}/clk/SM, both measured, profiles/micro_*.txt) x "
                  f"{clock_mhz:.0f} MHz observed during the timed region"),
        "k_fuse": st0["k_fuse"],
        "hbm": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved_gbs / hbm_peak,
                "dram_frac": (traffic / (launch_ms * 1e-3) / 1e9 / hbm_peak) if traffic else None,
                "basis": (f"{BYTES_PER_PX_ITER} B per active pixel-iteration (read rho1, rho2, v, "
                          f"c; write rho1, rho2, v) x active px x {st0['k_fuse']} fused "
                          f"iterations per launch / mean launch time: the minimum-traffic "
                          f"schedule's roofline (SURVEY 8(d) R1), > 1 with temporal blocking; "
                          f"dram_frac = measured DRAM bytes per launch (traffic, ncu) / launch "
                          f"time / peak; peak = MEASURED_PEAKS.json hbm_gbs (measured copy)")},
    }

    # K1, K2, band flags, items; energy partial + final; the compact path's index build,
    # gather and scatter (+ the coupled / decoupled split: count, scan, fill; st["launches"]
    # counts its k_rdc_iso launch)
    launches_per_step = sum(st["launches"] + 4 + 2 + (5 if st["compact"] else 0)
                            + (3 if st.get("rdc_decoupled", 0) else 0)
                            # grouping: init, the label rounds, count, class (+ fill when it is
                            # kept; st["launches"] counts the k_rdc_grp launches)
                            + ((3 + st["rdc_label_rounds"] + (1 if st["rdc_grouped"] else 0))
                               if st.get("rdc_label_rounds", 0) else 0) for _, st, _ in info)
    line = {
        "metric": _metric(cfg), "value": value, "unit": UNIT, "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.desc}", "H": cfg.H, "W": cfg.W, "iters": K,
                   "lambda": lam, "theta": cfg.theta, "tau": cfg.tau,
                   "delta_rels": _js(cfg.delta_rels), "k_fuse": st0["k_fuse"],
                   "item_rows": st0["item_rows"], "item_cols": st0["item_cols"],
                   "l2": _l2_note(cfg),
                   "parallelism": f"replicas x{dist.world}"},
        "rd_gpix_iter_s": dist.sum(rd_step * args.steps) / (t_ms * 1e-3) / 1e9,
        "per_delta": per_delta,
        # the paper's "+25% restricted-code overhead at q = 1": here the K-loop
        # is the same kernel at every delta (the label is folded into c'), so the overhead of
        # the restriction machinery is the band/tile setup (K1 + K2) of a delta = inf solve
        "restricted_overhead": _overhead(per_delta),
        "roofline": roofline,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": ck,
    }
    if not args.no_e2e:
        line["e2e"] = e2e(args, s, cfg, z, P, deltas, K, lam, dist, work_step)
    s.close()
    if not args.no_compact:
        line["restricted_compact"] = compact_section(cfg, zt, Pt, am, K, lam, sp, per_delta)
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, z, P, args.cpu_seconds)
    if dist.rank == 0:
        print(json.dumps(line), flush=True)


def e2e(args, s, cfg, z, P, deltas, K, lam, dist, work_step):
    """Same metric through the C ABI with HOST buffers: each step copies z (and P) from
    pinned host memory, solves every delta and reads back each mask and the energies."""
    import torch

    zh = torch.from_numpy(z).pin_memory()
    Ph = torch.from_numpy(P).pin_memory() if P is not None else None
    masks = [torch.empty((cfg.H, cfg.W), dtype=torch.uint8).pin_memory() for _ in deltas]
    h2d = z.nbytes + (P.nbytes if P is not None else 0)
    d2h = sum(m.numel() for m in masks) + 6 * 8 * len(deltas)

    def one():
        s.set_image(zh.numpy())
        s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, Ph.numpy() if Ph is not None else None)
        for d, m in zip(deltas, masks):
            s.solve(lam, cfg.theta, cfg.tau, d, K)
            s.mask(m.numpy())
            s.energy()

    one()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    torch.cuda.synchronize()
    dt = dist.max(time.perf_counter() - t0)
    value = dist.sum(work_step * args.steps) / dt / 1e9
    return {"value": value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": 1e3 * dt / args.steps,
            "path": "rds_set_image/rds_set_fitting (pinned host) -> rds_solve -> rds_get_mask "
                    "(host) + rds_energy per delta"}


RDC_BYTES_PER_RD_ITER = 40  # k_rdc_iter: record (16 B) in + out, packed codes (8 B)
L2_READ_GBS = 17900.0       # measured L2-resident read bandwidth, profiles/micro_l2_bw.txt


def compact_section(cfg, zt, Pt, am, K, lam, sp, per_delta):
    """f3 beside the headline (untimed for `value`): the same sweep, plus two thinner bands,
    solved with RDS_OPT_COMPACT = 2 (the library takes the compacted RD iteration where its
    cost model predicts a win, else the dense stencil).  Whole-solve times (setup + K-loop,
    CUDA events, median of 3) against the dense delta = inf solve: the paper's restricted vs
    full speedup once the work scales with the RD pixels rather than the tiles they touch."""
    import statistics

    from paper_1807_11534_b200 import rds

    full = [p for p in per_delta if p["delta_rel"] == "inf"]
    if not full:
        return None
    t_full = full[0]["loop_ms"] + full[0]["setup_ms"]
    s = rds.Solver(cfg.H, cfg.W, stream=sp, timing=True, compact=2)
    s.set_image(zt)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, Pt)
    out = []
    for dr in sorted(set(cfg.delta_rels) | {0.02, 0.05}):
        d = wl.band_delta(dr, am)
        s.solve(lam, cfg.theta, cfg.tau, d, K)
        ts, st = [], None
        for _ in range(3):
            s.solve(lam, cfg.theta, cfg.tau, d, K)
            st = s.stats()
            ts.append(st["loop_ms"] + st["setup_ms"])
        t = statistics.median(ts)
        row = {"delta_rel": "inf" if math.isinf(dr) else dr,
               "path": "compact" if st["compact"] else "dense",
               "rd_frac": st["n_rd"] / (cfg.H * cfg.W), "solve_ms": t,
               "rd_decoupled_frac": st["rdc_decoupled"] / max(1, st["n_rd"]),
               "rd_grouped_frac": st["rdc_grouped"] / max(1, st["n_rd"]),
               "speedup_vs_full": t_full / t,
               "rd_gpix_iter_s": st["n_rd"] * K / (t * 1e-3) / 1e9}
        if st["compact"]:
            # k_rdc_iter moves 40 algorithmic bytes per RD pixel-iteration (own record in and
            # out, packed codes) against the measured L2 read bandwidth; it is latency / grid
            # barrier bound, so this fraction stays well below 1
            lm = statistics.median(ts) - st["setup_ms"]
            if st["rdc_decoupled"] + st["rdc_grouped"] == st["n_rd"]:
                # no record goes through L2 per pass (k_rdc_iso: registers; k_rdc_grp: shared
                # memory): bound by the two MUFU ops per RD pixel-iteration like the stencil
                # (8 px-iter/clk/SM; one scalar instruction stream per pixel, no packed pairs,
                # so instruction issue sits below that: DESIGN.md §6)
                import torch

                n_sm = torch.cuda.get_device_properties(0).multi_processor_count
                peak = (n_sm * MUFU_LANES_PER_SM / MUFU_PER_PX_ITER
                        * _peaks().get("sm_max_mhz", 1965.0) * 1e6 / 1e9)
                ach = st["n_rd"] * K / (lm * 1e-3) / 1e9
                row["roofline"] = {"bound": "alu", "achieved": ach, "peak": peak,
                                   "unit": "G RD-pixel-iter/s", "frac": ach / peak}
            else:
                gbs = RDC_BYTES_PER_RD_ITER * st["n_rd"] * K / (lm * 1e-3) / 1e9
                row["roofline"] = {"bound": "l2", "achieved": gbs, "peak": L2_READ_GBS,
                                   "unit": "GB/s", "frac": gbs / L2_READ_GBS}
        out.append(row)
    s.close()
    return {"per_delta": out, "full_dense_solve_ms": t_full,
            "basis": "RDS_OPT_COMPACT=2 solve (setup + K-loop) vs the dense delta=inf solve"}


def _overhead(per_delta):
    full = [p for p in per_delta if p["delta_rel"] == "inf"]
    if not full:
        return None
    p = full[0]
    return {"setup_ms": p["setup_ms"], "loop_ms": p["loop_ms"],
            "setup_over_loop": p["setup_ms"] / p["loop_ms"],
            "basis": "K1 fitting/band/init + K2 tile and item compaction vs the K-loop, delta = inf"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def _traffic_from_profile(kf):
    """dram__bytes_read.sum + dram__bytes_write.sum per stencil launch from the committed
    ncu --set full capture of the same configuration (profiles/stencil_dram_bytes.json)."""
    path = os.path.join(ROOT, "profiles", "stencil_dram_bytes.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        if int(d.get("k_fuse", -1)) == int(kf):
            return d.get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


# ------------------------------------------------------------------------------------------
# --layout strips: one image over the ranks (opt-in, strong scaling)
# ------------------------------------------------------------------------------------------

def run_strips(args, dist):
    """ONE image split in row strips over the ranks (paper_1807_11534_b200/strips.py: halo
    exchange by torch.distributed point-to-point, NCCL), the C-config delta sweep as one step.
    value = whole-image pixel-iterations / max-over-ranks time; strong scaling.  With one rank
    this times the segmented solve (rds_solve + rds_solve_continue every seg iterations) of a
    single strip without any exchange."""
    import torch
    import torch.distributed as tdist

    assert torch.cuda.is_available(), "bench.py --layout strips needs a CUDA device"
    torch.cuda.set_device(dist.local)
    from paper_1807_11534_b200 import strips

    own_pg = not tdist.is_initialized()
    if own_pg:  # one rank: a single-process group for StripSolver
        tdist.init_process_group("nccl", store=tdist.HashStore(), rank=0, world_size=1,
                                 device_id=torch.device("cuda", dist.local))
    cfg = wl.CONFIGS[args.config]
    K = args.iters or cfg.iters
    lam = cfg.lambdas[0]
    z, P = wl.make_image(cfg)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    zt = torch.from_numpy(z).cuda()
    Pt = torch.from_numpy(P).cuda() if P is not None else None
    ss = strips.StripSolver(cfg.H, cfg.W, args.seg)
    ss.set_image(zt)
    ss.set_fitting(cfg.c1, cfg.c2, cfg.gamma, Pt)
    am = ss.absmax()
    deltas = [wl.band_delta(dr, am) for dr in cfg.delta_rels]

    def step():
        for d in deltas:
            ss.solve(lam, cfg.theta, cfg.tau, d, K)
            ss.energy()

    for _ in range(max(args.warmup, 3)):
        step()
    clocks = Clocks(dist.local)
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    ck = clocks.stop()
    t_ms = dist.max(ev0.elapsed_time(ev1))
    work = float(cfg.H * cfg.W) * K * len(deltas) * args.steps
    me = ss.me
    line = {
        "metric": _metric(cfg), "value": throughput(work, t_ms), "unit": UNIT,
        "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.desc}", "H": cfg.H, "W": cfg.W, "iters": K,
                   "delta_rels": _js(cfg.delta_rels),
                   "parallelism": f"row strips x{dist.world}, halo refresh every {args.seg} "
                                  f"iterations", "rows_held_rank0": me.rows,
                   "l2": "no flush: per-iteration working set > L2 at C3/C4"},
        "work_basis": "whole-image pixel-iterations (every tile of C3 is active)",
        "clocks": ck,
    }
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    ss.engine.close()
    if own_pg:
        tdist.destroy_process_group()


def main():
    args = parse()
    dist = Dist()
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        elif args.layout == "strips":
            run_strips(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
