"""GPU parity of the dense regime (csrc/dense.cu, ELLPACK_OPT_DENSE): the X^2 / SP2 step as a dense
FP64 GEMM over the scattered operand, then the row epilogue. Every output entry is the same ascending-k
fma chain as the oracle's plus exact-zero terms, so the comparison is bitwise (values, patterns,
traces, overflow counts, SP2 branches and stop iterations), on symmetric operands (one dense copy,
upper-triangle tiles mirrored) and non-symmetric ones (A^T and B copies, every tile), at sizes that
are not multiples of the 128 tile."""
import numpy as np
import pytest

import oracle
import synth
from tests.helpers import same_bits
from tests.test_gpu_parity import _compare_sp2, gpu_x2, ora_x2, same_bits_scalar, up

pytestmark = pytest.mark.gpu


def _ctx(E, dense=2, loop=1, sym=1, kernel=0):
    c = E.Context(0)
    c.set_option(E.OPT_DENSE, dense)
    c.set_option(E.OPT_SP2_DEVICE_LOOP, loop)
    c.set_option(E.OPT_SP2_SYMMETRIC, sym)
    c.set_option(E.OPT_DENSE_KERNEL, kernel)
    return c


def _sym(n, seed):
    return synth.sym_banded(n, 32, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, seed)


# 128-row tiles from 118 tiles on (sym: N >= 1793, otherwise N >= 1281), 16-row tiles below
@pytest.mark.parametrize("kind,n,tau", [("sym", 200, 0.0), ("sym", 517, 1e-5), ("sym", 1000, 1e-7),
                                        ("nonsym", 130, 0.0), ("nonsym", 300, 1e-4), ("nonsym", 645, 1e-6),
                                        ("cfg1", 512, 1e-5), ("sym", 2000, 1e-6), ("sym", 1921, 0.0),
                                        ("nonsym", 1500, 1e-6), ("nonsym", 1283, 0.0)])
def test_x2_dense_forced_bitwise(ellpack_lib, kind, n, tau):
    E = ellpack_lib
    if kind == "sym":
        X = _sym(n, n)
    elif kind == "cfg1":
        X = synth.cfg1()
    else:
        X = synth.random_sparse(n, 40, 0, 40, band=n // 3 if n < 1000 else None, p_empty=0.05, seed=n)
    wo = n + (n & 1)  # ELLPACK widths are even
    r, Y = ora_x2(X, wo, tau)
    c = _ctx(E)
    try:
        st, Yg, tx, tx2 = gpu_x2(c, X, wo, tau)
        assert c.last_launch()["path"] == "dense"
        assert st == r.status == E.OK
        assert same_bits(Yg, Y)
        assert same_bits_scalar(tx, r.trace_x) and same_bits_scalar(tx2, r.trace_x2)
        # overflow through the dense epilogue: exact rows over the width and required width
        w = max(2, (r.required_width // 2) & ~1)
        r2, _ = ora_x2(X, w, tau)
        st2, _, _, _ = gpu_x2(c, X, w, tau)
        assert st2 == r2.status == E.ERR_OVERFLOW
        assert c.overflow_info() == (r2.overflow_rows, r2.required_width)
    finally:
        c.close()


@pytest.mark.parametrize("n,seed,tau,sym", [(300, 2, 0.0, 1), (517, 5, 1e-6, 1), (517, 5, 1e-6, 0),
                                            (700, 9, 1e-5, 1), (1900, 3, 1e-6, 1), (1300, 4, 1e-6, 0)])
def test_sp2_dense_forced_bitwise(ellpack_lib, n, seed, tau, sym):
    """Every SP2 step dense (ELLPACK_OPT_DENSE 2): bitwise the oracle's run; with the symmetric
    option off the GEMM takes the non-symmetric route (A^T copy, all tiles)."""
    E = ellpack_lib
    H = _sym(n, seed)
    wd = n + (n & 1)
    K = 100 if n < 1000 else 8  # large N: a window of the run (the oracle's steps grow as N w^2)
    o = oracle.sp2(H, n // 2, 1e-10, oracle.SP2Opts(threshold=tau, max_iter=K), d_width=wd)
    c = _ctx(E, dense=2, sym=sym)
    try:
        d = E.Mat.empty(n, wd)
        g = c.sp2_run(up(H), n // 2, 1e-10, d, threshold=tau, max_iter=K)
        _compare_sp2(g, o)
        assert same_bits(d.to_host(), o.D)
        assert all(it["regime"] == "dense" for it in g.iters)
        T = (n + 127) // 128
        for it in g.iters:  # FMAs of the non-empty k blocks of the computed tiles
            assert it["products_exec"] % (16 * 128 * 128) == 0
            assert 0 < it["products_exec"] <= T * T * (T * 8) * 16 * 128 * 128
    finally:
        c.close()


def test_sp2_dense_auto_switches_mid_run(ellpack_lib):
    """Automatic regime on the host loop: the early, narrow iterates run on the sparse kernels, the
    filled-in ones on the dense GEMM -- one run, bitwise the oracle's."""
    E = ellpack_lib
    H = synth.cfg1()
    n = H.n
    o = oracle.sp2(H, n // 2, 1e-8, oracle.SP2Opts(threshold=1e-5, max_iter=100), d_width=n)
    c = _ctx(E, dense=0, loop=1)
    try:
        d = E.Mat.empty(n, n)
        g = c.sp2_run(up(H), n // 2, 1e-8, d, threshold=1e-5, max_iter=100)
        _compare_sp2(g, o)
        assert same_bits(d.to_host(), o.D)
        regimes = [it["regime"] for it in g.iters]
        assert regimes[0] == "sparse" and "dense" in regimes
    finally:
        c.close()


@pytest.mark.parametrize("n,sym", [(512, 1), (300, 0), (1000, 1)])
def test_sp2_device_loop_dense_bitwise(ellpack_lib, n, sym):
    """The automatic choice for N <= 1024: the device-resident loop (one graph launch) with every
    step dense, (alpha, beta, old_mode) read from device memory by the epilogue; bitwise."""
    E = ellpack_lib
    H = synth.cfg1() if n == 512 else _sym(n, 4)
    wd = n + (n & 1)
    o = oracle.sp2(H, n // 2, 1e-8, oracle.SP2Opts(threshold=1e-5, max_iter=100), d_width=wd)
    c = _ctx(E, dense=0, loop=0, sym=sym)
    try:
        d = E.Mat.empty(n, wd)
        s0 = c.host_syncs()
        g = c.sp2_run(up(H), n // 2, 1e-8, d, threshold=1e-5, max_iter=100)
        assert c.host_syncs() - s0 < 20  # the device loop: a fixed number, not one per iteration
        _compare_sp2(g, o)
        assert same_bits(d.to_host(), o.D)
        assert all(it["regime"] == "dense" for it in g.iters)
    finally:
        c.close()


def test_dense_off_keeps_sparse_kernels(ellpack_lib):
    E = ellpack_lib
    X = _sym(400, 1)
    c = _ctx(E, dense=1)
    try:
        st, _, _, _ = gpu_x2(c, X, 400, 1e-5)
        assert st == E.OK and c.last_launch()["path"] != "dense"
        d = E.Mat.empty(400, 400)
        g = c.sp2_run(up(X), 200, 1e-10, d, threshold=1e-6, max_iter=100)
        assert all(it["regime"] == "sparse" for it in g.iters)
    finally:
        c.close()


def test_cfg4_window_every_step_dense_bitwise(ellpack_lib):
    """cfg4 (N = 65536 lattice, the bench's K = 6 window) with every step forced dense -- the
    65536 x 65536 arrays, 128-row symmetric tiles with mostly-empty k blocks -- against the oracle."""
    E = ellpack_lib
    H, cf = synth.cfg4(), synth.CFG4
    n, K = H.n, 6
    dw = min(n, 8192)
    o = oracle.sp2(H, cf["nocc"], cf["tol"], oracle.SP2Opts(threshold=cf["threshold"], max_iter=K), d_width=dw)
    c = _ctx(E, dense=2, loop=1)
    try:
        d = E.Mat.empty(n, dw)
        g = c.sp2_run(up(H), cf["nocc"], cf["tol"], d, threshold=cf["threshold"], max_iter=K)
        assert all(it["regime"] == "dense" for it in g.iters)
        _compare_sp2(g, o)
        assert same_bits(d.to_host(), o.D)
    finally:
        c.close()


def test_cfg3_dense_equals_sparse_through_the_fill(ellpack_lib):
    """cfg3 at full size through the densifying phase (48 iterations: widths 448 -> ~12000, where the
    oracle needs ~20 min per step): every step dense and every step on the sparse kernels (each
    bitwise the oracle on the earlier windows) give the same bits -- iterate records, traces, D."""
    E = ellpack_lib
    H, cf = synth.cfg3(), synth.CFG3
    n, K = H.n, 48
    res = {}
    for dense in (1, 2):
        c = _ctx(E, dense=dense, loop=1)
        try:
            d = E.Mat.empty(n, n)
            g = c.sp2_run(up(H), cf["nocc"], cf["tol"], d, threshold=cf["threshold"], max_iter=K)
            assert all(it["regime"] == ("dense" if dense == 2 else "sparse") for it in g.iters)
            res[dense] = (g, d.to_host())
        finally:
            c.close()
    (gs, ds), (gd, dd) = res[1], res[2]
    assert gs.iterations == gd.iterations == K and gs.stop == gd.stop
    assert gs.final_width == gd.final_width and gs.final_width > 11000
    for a, b in zip(gs.iters, gd.iters):
        assert (a["branch"], a["width"], a["required"], a["products"]) == (b["branch"], b["width"], b["required"],
                                                                          b["products"])
        assert all(same_bits_scalar(a[k], b[k]) for k in ("trX", "trS", "e"))
    assert same_bits_scalar(gs.trD, gd.trD)
    assert same_bits(ds, dd)


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("kind,n,tau", [("sym", 2000, 1e-6), ("nonsym", 1500, 0.0)])
def test_x2_dense_both_gemm_kernels_bitwise(ellpack_lib, kernel, kind, n, tau):
    """The dense GEMM's two kernels for 128-row tiles -- FP64 FMAs (1) and the FP64 MMA (2, reading
    R23) -- each bitwise the oracle."""
    E = ellpack_lib
    X = _sym(n, n) if kind == "sym" else synth.random_sparse(n, 40, 0, 40, band=None, p_empty=0.05, seed=n)
    wo = n + (n & 1)
    r, Y = ora_x2(X, wo, tau)
    c = _ctx(E, kernel=kernel)
    try:
        st, Yg, tx, tx2 = gpu_x2(c, X, wo, tau)
        assert c.last_launch()["path"] == "dense" and st == r.status == E.OK
        assert same_bits(Yg, Y)
        assert same_bits_scalar(tx, r.trace_x) and same_bits_scalar(tx2, r.trace_x2)
    finally:
        c.close()


@pytest.mark.parametrize("kernel", [1, 2])
def test_sp2_dense_both_gemm_kernels_bitwise(ellpack_lib, kernel):
    E = ellpack_lib
    n = 1900
    H = _sym(n, 3)
    o = oracle.sp2(H, n // 2, 1e-10, oracle.SP2Opts(threshold=1e-6, max_iter=8), d_width=n)
    c = _ctx(E, dense=2, kernel=kernel)
    try:
        d = E.Mat.empty(n, n)
        g = c.sp2_run(up(H), n // 2, 1e-10, d, threshold=1e-6, max_iter=8)
        _compare_sp2(g, o)
        assert same_bits(d.to_host(), o.D)
    finally:
        c.close()


@pytest.mark.parametrize("n", [1, 2, 127, 129])
def test_x2_dense_degenerate_sizes(ellpack_lib, n):
    """The dense regime at sizes around one 128 tile and on an all-empty operand (every tile empty:
    nothing stored, nothing emitted, traces +0)."""
    E = ellpack_lib
    rng = np.random.default_rng(n)
    dense = np.where(rng.random((n, n)) < 0.3, rng.standard_normal((n, n)), 0.0)
    dense = (dense + dense.T) * 0.5
    wo = n + (n & 1)
    for X in (synth.from_dense(dense, w=wo), synth.from_dense(np.zeros((n, n)), w=wo)):
        r, Y = ora_x2(X, wo, 0.0)
        c = _ctx(E)
        try:
            st, Yg, tx, tx2 = gpu_x2(c, X, wo, 0.0)
            assert c.last_launch()["path"] == "dense" and st == r.status == E.OK
            assert same_bits(Yg, Y)
            assert same_bits_scalar(tx, r.trace_x) and same_bits_scalar(tx2, r.trace_x2)
        finally:
            c.close()


def test_cfg4_bench_window_k10_regimes_agree(ellpack_lib):
    """The cfg4 window bench.py times (K = 10, SURVEY §8d "SP2 protocol"): its iterations 6-9 are beyond
    what the oracle finishes in a test (~10^12 products); the automatic regime (dense from iteration 3
    on) equals the sparse kernels bit for bit there, and the first 6 iterations of either equal the
    oracle (test_sp2_bench_window_bitwise, test_cfg4_window_every_step_dense_bitwise)."""
    import torch
    E = ellpack_lib
    H, cf = synth.cfg4(), synth.CFG4
    n, K = H.n, 10
    dw = min(n, 8192)
    torch.cuda.empty_cache()  # the two 34 GB dense arrays must fit in 60 % of the free memory
    res = {}
    for dense in (0, 1):
        c = _ctx(E, dense=dense, loop=0)
        try:
            d = E.Mat.empty(n, dw)
            g = c.sp2_run(up(H), cf["nocc"], cf["tol"], d, threshold=cf["threshold"], max_iter=K)
            res[dense] = (g, d.to_host())
        finally:
            c.close()
    (ga, da), (gs, ds) = res[0], res[1]
    assert "dense" in [it["regime"] for it in ga.iters]
    assert ga.iterations == gs.iterations == K and ga.final_width == gs.final_width
    for a, b in zip(ga.iters, gs.iters):
        assert (a["branch"], a["width"], a["required"], a["products"]) == (b["branch"], b["width"], b["required"],
                                                                          b["products"])
        assert all(same_bits_scalar(a[k], b[k]) for k in ("trX", "trS", "e"))
    assert same_bits(da, ds)


def test_sp2_dense_allocation_failure_falls_back(ellpack_lib):
    """A dense step whose arrays cannot be allocated (ELLPACK_OPT_SP2_MEM_CAP fault injection) runs
    on the sparse kernels instead, and so does the rest of the run: bitwise the oracle."""
    E = ellpack_lib
    n = 700
    H = _sym(n, 9)
    o = oracle.sp2(H, n // 2, 1e-10, oracle.SP2Opts(threshold=1e-5, max_iter=100), d_width=n)
    c = _ctx(E, dense=2)
    c.set_option(E.OPT_SP2_MEM_CAP, 8_600_000)  # below 2 x 768^2 doubles (9.4 MB); two 700-wide iterates fit
    try:
        d = E.Mat.empty(n, n)
        g = c.sp2_run(up(H), n // 2, 1e-10, d, threshold=1e-5, max_iter=100)
        _compare_sp2(g, o)
        assert same_bits(d.to_host(), o.D)
        assert all(it["regime"] == "sparse" for it in g.iters)
    finally:
        c.close()
