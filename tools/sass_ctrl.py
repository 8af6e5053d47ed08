#!/usr/bin/env python
"""Decode SASS control bits (stall, yield, write/read scoreboard, wait mask) from cuobjdump -sass
output (Volta+ 128-bit encoding: bits 105-108 stall, 109 yield, 110-112 wbar, 113-115 rbar,
116-121 wait mask). Usage: cuobjdump -sass -fun NAME lib.so | python tools/sass_ctrl.py [from to]"""
import re
import sys

lines = sys.stdin.read().splitlines()
out = []
k = 0
while k < len(lines):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);?\s*/\* (0x[0-9a-f]+) \*/", lines[k])
    if m and k + 1 < len(lines):
        m2 = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[k + 1])
        if m2:
            hi = int(m2.group(1), 16)
            stall = (hi >> 41) & 0xF
            yld = (hi >> 45) & 1
            wb = (hi >> 46) & 7
            rb = (hi >> 49) & 7
            wm = (hi >> 52) & 0x3F
            out.append((int(m.group(1), 16), m.group(2).strip(), stall, yld, wb, rb, wm))
            k += 2
            continue
    k += 1
lo = int(sys.argv[1], 16) if len(sys.argv) > 1 else 0
hi_ = int(sys.argv[2], 16) if len(sys.argv) > 2 else 1 << 40
for a, ins, st, y, wb, rb, wm in out:
    if lo <= a <= hi_:
        w = "".join(str(s) for s in range(6) if wm >> s & 1)
        print(f"{a:05x} st{st:2d} {'Y' if y else ' '} wb{wb if wb != 7 else '-'} rb{rb if rb != 7 else '-'} wait[{w:6s}] {ins[:80]}")
