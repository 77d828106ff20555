"""One compacted-RD solve of C3 (ncu target for k_rdc_iter / k_rdc_iso / k_rdc_grp): python scripts/compact_one.py
[--delta-rel 0.05] [--iters 30]."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1807_11534_b200 import rds  # noqa: E402
from paper_1807_11534_b200 import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--delta-rel", type=float, default=0.05)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--split", type=int, default=None, help="RDS_OPT_RDC_SPLIT (default: the library's)")
a = ap.parse_args()
z, _ = wl.make_image("C3")
s = rds.Solver(*z.shape, compact=1, timing=True, rdc_split=a.split)
s.set_image(z)
s.set_fitting(0.8, 0.2)
s.solve(5.0, 0.1, 0.125, wl.band_delta(a.delta_rel, s.absmax()), a.iters)
st = s.stats()
print("compact", st["compact"], "n_rd", st["n_rd"], "decoupled", st["rdc_decoupled"], "grouped",
      st["rdc_grouped"], "loop_ms", st["loop_ms"])
