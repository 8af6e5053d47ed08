#!/usr/bin/env python
"""Kernel-time sweep of the fused row kernel on cfg5-style X^2 (tuning aid; not the bench).

python tools/sweep.py --sizes 262144:256 32768:64 --windows 0 --warps 0 1 2 4
Prints one JSON line per (size, window, warps): row-kernel ms (CUDA events on the
launching stream, mean of --reps launches), GFLOP/s and algorithmic GB/s.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2102_08505_b200 as eb  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", nargs="+", default=["262144:256"])
    ap.add_argument("--windows", nargs="+", type=int, default=[0])
    ap.add_argument("--warps", nargs="+", type=int, default=[0])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ablate", nargs="+", type=int, default=[0],
                    help="timing-only ablations (results wrong; needs a -DELL_ABLATE=1 build, e.g. "
                         "tools/variants.py ELL_ABLATE=1): 1 no row stores, 2 no accumulate, 4 no gathers, "
                         "8 no emission")
    args = ap.parse_args()
    eb.build()
    for sz in args.sizes:
        n, m = map(int, sz.split(":"))
        X = synth.cfg5(n, m)
        P = synth.products(X, X)
        x = eb.Mat.from_host(X)
        ctx = eb.Context(0)
        y = eb.Mat.empty(n, m)
        st, _, _ = ctx.multiply_x2(x, y, 1e-5)
        req = ctx.overflow_info()[1] if st == eb.ERR_OVERFLOW else int(y.nnz.max().item())
        w = ((req + 31) // 32) * 32
        del y
        y = eb.Mat.empty(n, w)
        ctx.close()
        for win, wp, ab in [(a, b, c) for a in args.windows for b in args.warps for c in args.ablate]:
            if True:
                ctx = eb.Context(0)
                if ab:
                    ctx.set_option(eb.OPT_ABLATE, ab)
                if win:
                    ctx.set_option(eb.OPT_WINDOW, win)
                if wp:
                    ctx.set_option(eb.OPT_WARPS, wp)
                ctx.multiply_x2(x, y, 1e-5)
                ctx.set_option(eb.OPT_PROFILE, 1)
                for _ in range(args.reps):
                    s, _, _ = ctx.multiply_x2(x, y, 1e-5)
                ms, k = ctx.kernel_time()
                ms /= max(k, 1)
                nnz_c = int(y.nnz.sum().item())
                Bc = 12 * (int(X.nnz.sum()) + nnz_c) + 8 * n
                print(json.dumps({"n": n, "m": m, "window": win, "warps": wp, "ablate": ab, "status": s, "ms": ms,
                                  "gflops": 2 * P / ms / 1e6, "alg_GBps": Bc / ms / 1e6,
                                  "products": P, "out_w": w}), flush=True)
                ctx.close()
        del x, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
