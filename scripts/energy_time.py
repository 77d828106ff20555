"""rds_energy (K5) time on a config: CUDA events around each call on the handle's stream
(the call's kernels plus its 56-byte read-back), median of reps; the HBM roofline of the
streaming kernel at 21 algorithmic bytes per pixel (v, u, f, rho1, rho2: 4 B each; label: 1 B)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
for name in sys.argv[1:] or ["C3"]:
    cfg = wl.CONFIGS[name]
    z, P = wl.make_image(cfg)
    st = torch.cuda.Stream()
    s = rds.Solver(cfg.H, cfg.W, stream=st.cuda_stream)
    s.set_image(torch.from_numpy(z).cuda())
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, torch.from_numpy(P).cuda() if P is not None else None)
    s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, wl.band_delta(0.2, s.absmax()), 20)
    ts = []
    for _ in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        e = s.energy()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts[2:])
    gbs = 21.0 * cfg.H * cfg.W / (ms * 1e-3) / 1e9
    print(json.dumps({"config": name, "energy_ms": ms, "algorithmic_gbs": gbs,
                      "hbm_frac": gbs / peak, "gap": e["gap"]}), flush=True)
    s.close()
