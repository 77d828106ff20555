"""Instruction mix of one kernel in a cuobjdump -sass listing (static counts).

usage: python scripts/sass_mix.py <listing.sass> <function-substring>
Counts every instruction of the function, and separately those inside its innermost loops
(a backward BRA's target .. the BRA), which is where the stencil spends its time."""
import re
import sys
from collections import Counter

path, name = sys.argv[1], sys.argv[2]
lines = open(path).read().split("\n")
body, on = [], False
for ln in lines:
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


tot = Counter(op(i) for _, i in body)
# loops: backward branches
loops = []
for a, ins in body:
    m = re.match(r"(@!?U?P\w+ )?BRA (`\(\.L_x_\d+\)|0x[0-9a-f]+)", ins)
    if m:
        tgt = re.search(r"0x([0-9a-f]+)", ins)
        if tgt and int(tgt.group(1), 16) < a:
            loops.append((int(tgt.group(1), 16), a))
print(f"{name}: {len(body)} instructions")
print("all :", ", ".join(f"{k} {v}" for k, v in tot.most_common(24)))
for lo, hi in sorted(loops, key=lambda x: x[1] - x[0], reverse=True)[:3]:
    c = Counter(op(i) for a, i in body if lo <= a <= hi)
    print(f"loop {lo:#x}-{hi:#x} ({sum(c.values())} instr):", ", ".join(f"{k} {v}" for k, v in c.most_common(24)))
