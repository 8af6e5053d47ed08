#!/usr/bin/env python
"""Summarise an ncu report's SASS source page: stall reasons, top stalled instructions,
shared-memory wavefronts per instruction (actual vs ideal). Tuning aid (reads gpurun_out/)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
col = {h: k for k, h in enumerate(hdr)}
f = lambda r, h: float(r[col[h]] or 0)
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {s: sum(f(r, s) for r in data) for s in st}
T = sum(tot.values()) or 1
print("stalls:", ", ".join(f"{s[6:]} {100 * v / T:.1f}%" for s, v in sorted(tot.items(), key=lambda x: -x[1]) if v / T > 0.005))
print("instructions executed:", sum(f(r, "Instructions Executed") for r in data))
ss = "Warp Stall Sampling (All Samples)"
print("--- top stalled")
for r in sorted(data, key=lambda r: -f(r, ss))[:top]:
    why = {s[6:]: int(f(r, s)) for s in st if f(r, s) > 0.15 * max(1, f(r, ss))}
    print(f"{r[0][-5:]} {r[1][:64]:64s} {int(f(r, ss)):7d} {int(f(r, 'Instructions Executed')):10d} {why}")
wf, wfi = "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal"
sh = [r for r in data if f(r, wf) > 0]
print("--- shared wavefronts total", sum(f(r, wf) for r in sh), "ideal", sum(f(r, wfi) for r in sh))
for r in sorted(sh, key=lambda r: -f(r, wf))[:top]:
    n = max(1, f(r, "Instructions Executed"))
    print(f"{r[0][-5:]} {r[1][:50]:50s} wf/inst {f(r, wf) / n:5.2f} ideal {f(r, wfi) / n:5.2f} n {int(n)}")
