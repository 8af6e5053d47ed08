#!/usr/bin/env python
"""Long randomized GPU-vs-oracle sweep (bitwise): multiply (both paths, in place / beta / alpha
corners, literal-width overflow reports), small SP2 runs (both branch rules, narrow GROW starts,
symmetric step; regimes cycled: automatic, sparse only, every step dense on the host loop) and X^2 in the
dense regime (symmetric / non-symmetric, both GEMM kernels, sizes 1..3000). A validation run, not part
of the test suite:
    python tools/fuzz_gpu.py --mult 400 --sp2 40 --x2dense 60
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2102_08505_b200 as eb  # noqa: E402


def bits(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


def same(g, o):
    if not np.array_equal(g.nnz, o.nnz):
        return False
    for i in range(o.n):
        k = int(o.nnz[i])
        if not (np.array_equal(g.col[i, :k], o.col[i, :k]) and bits(g.val[i, :k], o.val[i, :k])):
            return False
    return True


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mult", type=int, default=400)
    ap.add_argument("--sp2", type=int, default=40)
    ap.add_argument("--seed", type=int, default=77)
    ap.add_argument("--x2dense", type=int, default=0)
    ap.add_argument("--x2small", type=int, default=0, help="X^2 on the small-matrix kernel (N <= 1024)")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    ctx = eb.Context(0)
    bad = 0
    for t in range(a.mult):
        n = int(rng.integers(1, 5000))
        w = int(rng.choice([2, 4, 8, 16, 32, 64, 100, 128, 200, 256, 300]))
        kmax = int(rng.integers(1, w + 1))
        kmin = int(rng.integers(0, kmax + 1))
        band = int(rng.choice([1, 2, 10, 100, 1000, 20000]))
        pe = float(rng.choice([0.0, 0.05, 0.5]))
        alpha, beta = [(1.0, 0.0), (0.75, -1.5), (-1.0, 2.0), (0.0, 1.0), (2.0, 0.5)][t % 5]
        tau = float(rng.choice([0.0, 1e-8, 1e-5, 1e-2, 1.0]))
        A = synth.random_sparse(n, w, kmin, kmax, band, pe, float(rng.choice([1e-3, 1.0, 1e3])), seed=t * 3 + 1)
        B = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=t * 3 + 2)
        C0 = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=t * 3 + 3)
        lit = oracle.multiply(A, B, C0.copy(), alpha, beta, tau)
        wo = max(w, ((lit.required_width + 31) // 32) * 32)
        Co = C0.widened(wo).copy()
        r = oracle.multiply(A, B, Co, alpha, beta, tau)
        g = eb.Mat.from_host(C0, w=wo)
        st = ctx.multiply(eb.Mat.from_host(A), eb.Mat.from_host(B), g, alpha, beta, tau, ok=(0, 3))
        ok = st == eb.OK and r.status == oracle.OK and same(g.to_host(), Co)
        if lit.status != oracle.OK:
            g2 = eb.Mat.from_host(C0)
            st2 = ctx.multiply(eb.Mat.from_host(A), eb.Mat.from_host(B), g2, alpha, beta, tau, ok=(0, 3))
            ok = ok and st2 == eb.ERR_OVERFLOW and ctx.overflow_info() == (lit.overflow_rows, lit.required_width)
        if not ok:
            bad += 1
            print("MULT MISMATCH", t, (n, w, kmin, kmax, band, pe, alpha, beta, tau), flush=True)
    print(f"multiply: {a.mult - bad}/{a.mult} bitwise", flush=True)
    bad_s = 0
    for t in range(a.sp2):
        n = int(rng.integers(16, 900))
        m = int(rng.choice([8, 16, 32, 64]))
        partners = int(rng.integers(1, max(2, m // 3)))
        band = int(rng.choice([4, 16, 64, 300]))
        tau = float(rng.choice([0.0, 1e-7, 1e-5, 1e-4]))
        rule = int(rng.integers(0, 2))
        w0 = int(rng.choice([0, 8, 16]))
        H = synth.sym_banded(n, m, partners, band, 1, -1.0, 1.0, 0, band / 4.0, 0.0, 500 + t)
        nocc = int(rng.integers(1, n))
        o = oracle.sp2(H, nocc, 1e-9, oracle.SP2Opts(threshold=tau, max_iter=60, branch_rule=rule, initial_width=w0),
                       d_width=n + (n & 1))
        c2 = eb.Context(0)
        if w0:
            c2.set_option(eb.OPT_SP2_WIDTH0, w0)
        regime = t % 3  # 0 automatic, 1 sparse only, 2 every step dense (host loop)
        c2.set_option(eb.OPT_DENSE, regime)
        if regime == 2:
            c2.set_option(eb.OPT_SP2_DEVICE_LOOP, 1)
        d = eb.Mat.empty(n, n + (n & 1))
        g = c2.sp2_run(eb.Mat.from_host(H), nocc, 1e-9, d, threshold=tau, max_iter=60, branch_rule=rule)
        ok = (g.status == o.status and g.iterations == o.iterations and g.final_width == o.final_width
              and g.regrows == o.regrows and bits(g.trD, o.trD)
              and all(x["branch"] == y["branch"] and bits(x["trS"], y["trS"]) for x, y in zip(g.iters, o.iters))
              and same(d.to_host(), o.D))
        c2.close()
        if not ok:
            bad_s += 1
            print("SP2 MISMATCH", t, (n, m, partners, band, tau, rule, w0, nocc, regime), g.status, o.status,
                  g.iterations, o.iterations, g.final_width, o.final_width, flush=True)
    print(f"sp2: {a.sp2 - bad_s}/{a.sp2} bitwise", flush=True)
    bad_t = 0
    for t in range(a.x2small):  # X^2, N <= 1024, width <= 64: the small-matrix kernel (tiny.cu)
        n = int(rng.integers(1, 1025))
        w = int(rng.choice([2, 4, 8, 16, 30, 32, 34, 48, 64]))  # the ABI stores 16-byte slot pairs (R20)
        kmax = int(rng.integers(1, w + 1))
        kmin = int(rng.integers(0, kmax + 1))
        band = int(rng.choice([1, 5, 40, 300, 2000]))
        pe = float(rng.choice([0.0, 0.1, 0.6]))
        tau = float(rng.choice([0.0, 1e-9, 1e-5, 1e-2, 10.0]))
        X = synth.random_sparse(n, w, kmin, kmax, band, pe, float(rng.choice([1e-3, 1.0, 1e3])), seed=90000 + t)
        lit = oracle.x2(X, oracle.Ell.empty(n, w), tau)
        wo = max(2, ((lit.required_width + 31) // 32) * 32)
        Y = oracle.Ell.empty(n, wo)
        r = oracle.x2(X, Y, tau)
        x = eb.Mat.from_host(X)
        y = eb.Mat.empty(n, wo)
        st, tx, tx2 = ctx.multiply_x2(x, y, tau)
        ok = (st == eb.OK and r.status == oracle.OK and ctx.last_launch()["path"] == "small" and same(y.to_host(), Y)
              and bits(tx, r.trace_x) and bits(tx2, r.trace_x2))
        if lit.status != oracle.OK:
            st2, _, _ = ctx.multiply_x2(x, eb.Mat.empty(n, w), tau)
            ok = ok and st2 == eb.ERR_OVERFLOW and ctx.overflow_info() == (lit.overflow_rows, lit.required_width)
        if not ok:
            bad_t += 1
            print("X2 SMALL MISMATCH", t, (n, w, kmin, kmax, band, pe, tau), st, r.status, flush=True)
    print(f"x2 small: {a.x2small - bad_t}/{a.x2small} bitwise", flush=True)
    bad_d = 0
    for t in range(a.x2dense):
        n = int(rng.choice([1, 2, 3, 127, 128, 129, 255, 300, 511, 700, 1023, 1300, 1800, 2048, 2500, 3000]))
        sym = bool(t % 2)
        w = int(rng.choice([2, 8, 32, 64]))
        tau = float(rng.choice([0.0, 1e-9, 1e-5, 1e-2]))
        if sym:
            X = synth.sym_banded(n, w, int(rng.integers(1, max(2, w // 3))), int(rng.choice([1, 16, 200, 5000])), 1,
                                 -1.0, 1.0, 0, 8.0, 0.0, 900 + t)
        else:
            X = synth.random_sparse(n, w, 0, w, int(rng.choice([1, 16, 200, 5000])), 0.1, 1.0, seed=900 + t)
        wo = n + (n & 1)
        Y = synth.Ell.empty(n, wo)
        r = oracle.x2(X, Y, tau)
        c3 = eb.Context(0)
        c3.set_option(eb.OPT_DENSE, 2)
        kernel = int(rng.integers(0, 2))
        c3.set_option(eb.OPT_DENSE_KERNEL, kernel)
        y = eb.Mat.empty(n, wo)
        st, tx, tx2 = c3.multiply_x2(eb.Mat.from_host(X), y, tau)
        ok = (st == r.status and c3.last_launch()["path"] == "dense" and same(y.to_host(), Y)
              and bits(tx, r.trace_x) and bits(tx2, r.trace_x2))
        c3.close()
        if not ok:
            bad_d += 1
            print("X2 DENSE MISMATCH", t, (n, sym, w, tau, kernel), st, r.status, flush=True)
    if a.x2dense:
        print(f"x2 dense: {a.x2dense - bad_d}/{a.x2dense} bitwise", flush=True)
    ctx.close()
    return 1 if bad or bad_s or bad_d else 0


if __name__ == "__main__":
    sys.exit(main())
