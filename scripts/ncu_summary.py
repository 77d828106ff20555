"""Summarise an ncu report: key throughput metrics, stall breakdown, SASS op mix."""
import builtins
import collections
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__shared_mem_per_block_static',
        'sm__inst_executed.sum.per_cycle_active', 'sm__inst_executed.sum', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__cycles_elapsed.avg.per_second', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'smsp__inst_executed.avg.per_cycle_active']


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


def main(rep, out=None):
    lines = []

    def print(*a):  # noqa: A001 - tee into the summary file
        builtins.print(*a)
        lines.append(" ".join(str(x) for x in a))

    raw = list(csv.reader(io.StringIO(run(['ncu', '-i', rep, '--page', 'raw', '--csv']))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    print(f"== {rep}: {vals[hdr.index('Kernel Name')][:90]}")
    for i, h in enumerate(hdr):
        if h in KEYS:
            print(f"  {h:70s} {vals[i]:>14s} {units[i]}")
    st = {h.replace('smsp__pcsamp_warps_issue_stalled_', ''): float(vals[i] or 0)
          for i, h in enumerate(hdr) if h.startswith('smsp__pcsamp_warps_issue_stalled_')
          and not h.endswith('_not_issued')}
    tot = sum(st.values()) or 1
    print("  stalls (pc samples %):", ", ".join(f"{k} {100*v/tot:.1f}" for k, v in
                                              sorted(st.items(), key=lambda kv: -kv[1]) if v / tot > 0.005))
    src = list(csv.reader(io.StringIO(run(['ncu', '-i', rep, '--page', 'source', '--csv']))))
    shdr = src[1]
    ix = {h: i for i, h in enumerate(shdr)}
    ops = collections.Counter()
    for r in src[2:]:
        n = int(r[ix['Instructions Executed']] or 0)
        s = r[ix['Source']].strip()
        if not s:
            continue
        op = s.split()[0]
        if op.startswith('@'):
            op = s.split()[1]
        ops[op.split('.')[0]] += n
    tot = sum(ops.values())
    print("  op mix (% of warp instr):", ", ".join(f"{k} {100*v/tot:.1f}" for k, v in ops.most_common(14)))
    print(f"  warp instructions executed: {tot/1e6:.2f} M")
    get = {h: vals[i] for i, h in enumerate(hdr)}
    res = {"kernel": get.get("Kernel Name"),
           "gpu_time_us": float(get["gpu__time_duration.sum"]),
           "dram_bytes_per_launch": (float(get["dram__bytes_read.sum"]) +
                                     float(get["dram__bytes_write.sum"])) * _scale(units[hdr.index("dram__bytes_read.sum")]),
           "issue_active_pct": float(get.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0) or 0),
           "registers": int(float(get["launch__registers_per_thread"]))}
    if out:
        with open(out, "w") as fh:
            fh.write("\n".join(lines) + "\n")
    return res


def _scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


if __name__ == '__main__':
    import argparse
    import json

    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--out", help="write the text summary of the (single) report here")
    ap.add_argument("--json", help="write dram bytes per launch here (profiles/stencil_dram_bytes.json)")
    ap.add_argument("--kf", type=int, default=0)
    ap.add_argument("--config", default="")
    a = ap.parse_args()
    for rep in a.reports:
        res = main(rep, a.out)
        if a.json:
            res.update({"k_fuse": a.kf, "config": a.config, "report": rep})
            with open(a.json, "w") as fh:
                json.dump(res, fh, indent=1)
