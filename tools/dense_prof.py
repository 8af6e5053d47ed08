#!/usr/bin/env python
"""One forced-dense X^2 of a filled symmetric N x N matrix (for ncu -k regex:dense_gemm).
python tools/dense_prof.py [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2102_08505_b200 as eb  # noqa: E402
import synth  # noqa: E402

eb.build()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rng = np.random.default_rng(n)
a = rng.standard_normal((n, n)) * 0.01
X = synth.from_dense((a + a.T) * 0.5)
ctx = eb.Context(0)
ctx.set_option(eb.OPT_DENSE, 2)
x = eb.Mat.from_host(X)
y = eb.Mat.empty(n, n)
st = ctx.multiply_x2(x, y, 0.0)
torch.cuda.synchronize()
print("ok", n, st, ctx.last_launch()["path"])
