#!/usr/bin/env python
"""Where should an SP2 step switch to the dense regime? cfg3 (N = 12288) with every step sparse
(ELLPACK_OPT_DENSE 1) and with every step dense (2), host loop, per-iteration device time of the step
(sp2_iter_rec.step_ms) beside its product count P: the crossover calibrates the automatic rule
(N^3 < ratio x P). One JSON line per iteration and mode."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2102_08505_b200 as eb  # noqa: E402
import synth  # noqa: E402

eb.build()
K = int(sys.argv[1]) if len(sys.argv) > 1 else 40
which = sys.argv[2] if len(sys.argv) > 2 else "cfg3"
if which in ("cfg3", "cfg4"):
    H, cf = (synth.cfg3(), synth.CFG3) if which == "cfg3" else (synth.cfg4(), synth.CFG4)
    nocc, tol, tau = cf["nocc"], cf["tol"], cf["threshold"]
else:
    H = synth.model_hamiltonian(int(which.split(":")[1]), which.split(":")[0], tau_store=1e-5)
    nocc, tol, tau = H.n // 2, 1e-8, 1e-5
n = H.n
for mode in (1, 2):
    ctx = eb.Context(0)
    ctx.set_option(eb.OPT_DENSE, mode)
    ctx.set_option(eb.OPT_SP2_DEVICE_LOOP, 1)
    h = eb.Mat.from_host(H)
    d = eb.Mat.empty(n, n + (n & 1))
    ctx.sp2_run(h, nocc, tol, d, threshold=tau, max_iter=3)
    torch.cuda.synchronize()
    r = ctx.sp2_run(h, nocc, tol, d, threshold=tau, max_iter=K)
    for k, it in enumerate(r.iters):
        print(json.dumps({"mode": "sparse" if mode == 1 else "dense", "it": k, "width": it["width"],
                          "products": it["products"], "exec": it["products_exec"], "step_ms": it["step_ms"],
                          "n3_over_P": n ** 3 / max(it["products"], 1)}), flush=True)
    ctx.close()
    del h, d
    torch.cuda.empty_cache()
