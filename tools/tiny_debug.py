import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2102_08505_b200 as eb, synth, oracle
from tests.helpers import same_bits
eb.build()
for validate in (1, 0):
    for (n, w, kmin) in ((1, 4, 1), (7, 8, 0), (512, 32, 15)):
        X = synth.random_sparse(n, w, kmin, w, seed=5) if n != 512 else synth.cfg1()
        ctx = eb.Context(0)
        ctx.set_option(eb.OPT_VALIDATE, validate)
        try:
            x = eb.Mat.from_host(X); y = eb.Mat.empty(n, min(n + (n & 1), 1024) if n > 1 else 2)
            st, tx, tx2 = ctx.multiply_x2(x, y, 1e-5)
            Y = oracle.Ell.empty(n, y.w if hasattr(y, 'w') else min(n + (n & 1), 1024))
            print("validate", validate, "n", n, "st", st, ctx.last_launch()["path"], flush=True)
        except Exception as e:
            print("validate", validate, "n", n, "ERR", e, flush=True)
            try:
                torch.cuda.synchronize()
            except Exception as e2:
                print("  torch:", e2, flush=True)
            sys.exit(1)
        ctx.close()
