"""Per-loop static schedule summary of one kernel in a cuobjdump -sass listing: for the
innermost loops (backward branches), instruction count, sum of encoded stall cycles (the
single-warp schedule length), and FMA-pipe / MUFU pipe cycles (FFMA2-class = 2, FFMA-class
= 1, MUFU = 8 per warp instruction on sm_100a, measured in scripts/micro/).
usage: python scripts/sass_loops.py <listing.sass> <function-substring>"""
import re
import sys

path, name = sys.argv[1], sys.argv[2]
body, on, prev = [], False, None
for ln in open(path).read().split("\n"):
    if "Function : " in ln:
        on = name in ln
        continue
    if not on:
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?)\s*/\* (0x[0-9a-f]+) \*/", ln)
    if m:
        prev = (int(m.group(1), 16), m.group(2))
        continue
    m2 = re.match(r"\s+/\* (0x[0-9a-f]+) \*/", ln)
    if m2 and prev:
        hiw = int(m2.group(1), 16)
        body.append((prev[0], prev[1], (hiw >> 41) & 0xF))
        prev = None


def op(ins):
    t = ins.split()
    if t[0].startswith("@"):
        t = t[1:]
    return t[0].rstrip(";").split(".")[0]


loops = []
for a, ins, _ in body:
    if " BRA " in f" {ins} " or ins.split()[0] == "BRA" or (ins.startswith("@") and "BRA" in ins):
        tgt = re.search(r"0x([0-9a-f]+)", ins)
        if tgt and int(tgt.group(1), 16) < a:
            loops.append((int(tgt.group(1), 16), a))
loops = sorted(set(loops), key=lambda x: x[1] - x[0], reverse=True)
for lo, hi in loops[:4]:
    ins = [(op(i), s) for a, i, s in body if lo <= a <= hi]
    n = len(ins)
    st = sum(s for _, s in ins)
    fma2 = sum(1 for o, _ in ins if o in ("FFMA2", "FADD2", "FMUL2"))
    fma1 = sum(1 for o, _ in ins if o in ("FFMA", "FADD", "FMUL", "IMAD", "HFMA2"))
    mufu = sum(1 for o, _ in ins if o == "MUFU")
    print(f"{name} loop {lo:#x}-{hi:#x}: {n} instr, stall sum {st}, FMA-pipe {2 * fma2 + fma1} cyc, "
          f"MUFU {8 * mufu} cyc ({mufu})")
