"""Decode the scheduling control bits of a cuobjdump -sass listing (sm_100a, 128-bit
instructions): stall count (bits 105-108), yield (109), write/read barrier, wait mask.
usage: python scripts/sass_ctrl.py <listing.sass> <function-substring> [lo_addr hi_addr]"""
import re
import sys

path, name = sys.argv[1], sys.argv[2]
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 62
lines = open(path).read().split("\n")
on = False
prev = None
for ln in lines:
    if "Function : " in ln:
        on = name in ln
        continue
    if not on:
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?)\s*/\* (0x[0-9a-f]+) \*/", ln)
    if m:
        prev = (int(m.group(1), 16), m.group(2), int(m.group(3), 16))
        continue
    m2 = re.match(r"\s+/\* (0x[0-9a-f]+) \*/", ln)
    if m2 and prev:
        hiw = int(m2.group(1), 16)
        addr, ins, low = prev
        prev = None
        if not (lo <= addr <= hi):
            continue
        stall = (hiw >> 41) & 0xF
        yld = (hiw >> 45) & 1
        wbar = (hiw >> 46) & 7
        rbar = (hiw >> 49) & 7
        wmask = (hiw >> 52) & 0x3F
        print(f"{addr:6x} s{stall:2d} y{yld} w{wbar} r{rbar} m{wmask:02x}  {ins}")
