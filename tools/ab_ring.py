#!/usr/bin/env python
"""A/B of the ring-path kernels on cfg5 X^2 (ELLPACK_OPT_RING_KERNEL): row-kernel device time
(CUDA events around each launch, ELLPACK_OPT_PROFILE) and whole-step time, with every variant's
output compared bitwise with the first one's.

python tools/ab_ring.py [--n N] [--m M] [--reps K] [--kernels 1,2,3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2102_08505_b200 as eb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=262144)
ap.add_argument("--m", type=int, default=256)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--kernels", default="1,2,3")
ap.add_argument("--warps", type=int, default=0)
a = ap.parse_args()
eb.build()
X = synth.cfg5(a.n, a.m)
x = eb.Mat.from_host(X)
ref = None
for rk in [int(v) for v in a.kernels.split(",")]:
    ctx = eb.Context(0)
    ctx.set_option(eb.OPT_RING_KERNEL, rk)
    if a.warps:
        ctx.set_option(eb.OPT_WARPS, a.warps)
    y = eb.Mat.empty(a.n, a.m)
    st, _, _ = ctx.multiply_x2(x, y, 1e-5)
    w = ((ctx.overflow_info()[1] + 31) // 32) * 32 if st == eb.ERR_OVERFLOW else a.m
    del y
    y = eb.Mat.empty(a.n, w)
    for _ in range(2):
        st, tx, tx2 = ctx.multiply_x2(x, y, 1e-5)
    torch.cuda.synchronize()
    ctx.set_option(eb.OPT_PROFILE, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        st, tx, tx2 = ctx.multiply_x2(x, y, 1e-5)
    e1.record()
    torch.cuda.synchronize()
    kms, kn = ctx.kernel_time()
    launch = ctx.last_launch()
    same = None
    if ref is None:
        ref = (y.nnz.clone(), y.col.clone(), y.val.clone(), tx, tx2)
    else:
        live = torch.arange(w, device="cuda")[None, :] < ref[0][:, None]
        same = bool(torch.equal(ref[0], y.nnz) and torch.equal(ref[1][live], y.col[live])
                    and torch.equal(ref[2][live].view(torch.int64), y.val[live].view(torch.int64))
                    and (tx, tx2) == (ref[3], ref[4]))
    print(json.dumps({"ring_kernel": rk, "status": st, "kernel_ms": kms / kn, "step_ms": e0.elapsed_time(e1) / a.reps,
                      "launch": launch, "bitwise_same_as_first": same, "n": a.n, "m": a.m}), flush=True)
    del y
    ctx.close()
    torch.cuda.empty_cache()
