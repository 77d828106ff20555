"""List every loop (backward branch target .. branch) of one function in a cuobjdump -sass
listing with its instruction mix; innermost first (smallest span)."""
import re
import sys
from collections import Counter

path, name = sys.argv[1], sys.argv[2]
body, on = [], False
for ln in open(path).read().split("\n"):
    if "Function : " in ln:
        on = name in ln
        continue
    if on:
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", ln)
        if m:
            body.append((int(m.group(1), 16), m.group(2)))


def op(ins):
    t = ins.split()
    if t[0].startswith("@"):
        t = t[1:]
    return t[0].split(".")[0]


loops = []
for a, ins in body:
    if re.search(r"\bBRA\b", ins):
        tgt = re.search(r"0x([0-9a-f]+)", ins)
        if tgt and int(tgt.group(1), 16) < a:
            loops.append((int(tgt.group(1), 16), a))
for lo, hi in sorted(set(loops), key=lambda x: x[1] - x[0]):
    c = Counter(op(i) for a, i in body if lo <= a <= hi)
    print(f"loop {lo:#x}-{hi:#x} ({sum(c.values())} instr):",
          ", ".join(f"{k} {v}" for k, v in c.most_common(14)))
