#!/usr/bin/env python
"""Small-problem latency probe: cfg1 X^2 calls and one SP2 run on the soft-matter H (N=512), for an
ncu launch list (gpu__time_duration per kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2102_08505_b200 as eb  # noqa: E402
import synth  # noqa: E402

eb.build()
ctx = eb.Context(0)
X = synth.cfg1()
x = eb.Mat.from_host(X)
y = eb.Mat.empty(X.n, 256)
for _ in range(3):
    ctx.multiply_x2(x, y, 1e-5)
loop = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctx.set_option(eb.OPT_SP2_DEVICE_LOOP, loop)
H = synth.model_hamiltonian(512, "soft_matter", tau_store=1e-5)
h = eb.Mat.from_host(H)
d = eb.Mat.empty(512, 512)
r = ctx.sp2_run(h, 256, 1e-8, d, threshold=1e-5, max_iter=8)
torch.cuda.synchronize()
print("ok", r.iterations, [it["width"] for it in r.iters], [it["products"] for it in r.iters])
