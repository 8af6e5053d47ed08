#!/usr/bin/env python
"""Dense GEMM device time (ELLPACK_OPT_PROFILE around the GEMM launch) for a forced-dense X^2 of a filled
symmetric N x N matrix. python tools/dense_time.py N [N ...]; one JSON line per N."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2102_08505_b200 as eb  # noqa: E402
import synth  # noqa: E402

eb.build()
for n in [int(v) for v in sys.argv[1:]] or [8192]:
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) * 0.01
    a = (a + a.T) * 0.5
    X = synth.Ell(val=np.ascontiguousarray(a), col=np.tile(np.arange(n, dtype=np.int32), (n, 1)),
                  nnz=np.full(n, n, dtype=np.int32))
    ctx = eb.Context(0)
    ctx.set_option(eb.OPT_DENSE, 2)
    ctx.set_option(eb.OPT_DENSE_KERNEL, int(os.environ.get("DENSE_KERNEL", "0")))
    x = eb.Mat.from_host(X)
    y = eb.Mat.empty(n, n + (n & 1))
    for _ in range(2):
        ctx.multiply_x2(x, y, 0.0)
    torch.cuda.synchronize()
    ctx.set_option(eb.OPT_DENSE, 2)
    ctx.set_option(eb.OPT_PROFILE, 1)
    for _ in range(5):
        ctx.multiply_x2(x, y, 0.0)
    kms, kn = ctx.kernel_time()
    T = (n + 127) // 128
    tiles = T * (T + 1) // 2 if T * (T + 1) // 2 >= 118 else 8 * T * T / 8
    fmas = (T * (T + 1) // 2 if T * (T + 1) // 2 >= 118 else T * T) * 128 * 128 * T * 128
    print(json.dumps({"n": n, "gemm_ms": kms / kn, "tflops": 2 * fmas / (kms / kn * 1e-3) / 1e12}), flush=True)
    ctx.close()
    del x, y
    torch.cuda.empty_cache()
