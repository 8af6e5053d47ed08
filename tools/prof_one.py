#!/usr/bin/env python
"""One warm multiply_x2 on a cfg5-style X (driver for ncu captures).

python tools/prof_one.py --n N --m M [--reps K] [--window S]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2102_08505_b200 as eb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--m", type=int, default=64)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--window", type=int, default=0)
ap.add_argument("--ablate", type=int, default=0)
ap.add_argument("--ring-kernel", type=int, default=0)
a = ap.parse_args()
X = synth.cfg5(a.n, a.m)
x = eb.Mat.from_host(X)
ctx = eb.Context(0)
if a.window:
    ctx.set_option(eb.OPT_WINDOW, a.window)
if a.ring_kernel:
    ctx.set_option(eb.OPT_RING_KERNEL, a.ring_kernel)
if a.ablate:
    ctx.set_option(eb.OPT_ABLATE, a.ablate)
y = eb.Mat.empty(a.n, a.m)
st, _, _ = ctx.multiply_x2(x, y, 1e-5)
w = ((ctx.overflow_info()[1] + 31) // 32) * 32 if st == eb.ERR_OVERFLOW else a.m
y = eb.Mat.empty(a.n, w)
for _ in range(a.reps):
    st, tx, tx2 = ctx.multiply_x2(x, y, 1e-5)
    assert st == eb.OK or a.ablate
torch.cuda.synchronize()
print("ok", a.n, a.m, w, tx, tx2)
