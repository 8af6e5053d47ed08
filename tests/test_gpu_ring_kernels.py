"""Every ring-path kernel (ELLPACK_OPT_RING_KERNEL: the legacy one-warp ring kernel, the split-row
kernel with 1 and with 2 warps per row) is bitwise the oracle on the ring-path shapes: B rows of
1..4 64-entry groups, ragged and empty rows, the Old operand (beta != 0, the SP2 SQUARE and EXPAND
steps), the x2 traces, and the literal-width overflow report."""
import numpy as np
import pytest

import oracle
import synth
from tests.helpers import same_bits
from tests.test_gpu_parity import FAST, _compare_sp2, eb, up

pytestmark = pytest.mark.gpu

KERNELS = [1, 2, 3, 4]


@pytest.fixture(scope="module", params=KERNELS, ids=lambda k: {1: "legacy", 2: "split_w1", 3: "split_w2", 4: "ws"}[k])
def kctx(request, ellpack_lib):
    c = ellpack_lib.Context(0)
    c.set_option(ellpack_lib.OPT_RING_KERNEL, request.param)
    yield c, request.param
    c.close()


@pytest.mark.parametrize("case", FAST, ids=lambda c: f"n{c[0]}w{c[1]}")
@pytest.mark.parametrize("alpha,beta,tau", [(1.0, 0.0, 0.0), (0.75, -1.5, 1e-3), (-1.0, 2.0, 1e-6)])
def test_ring_kernels_multiply_bitwise(kctx, case, alpha, beta, tau):
    ctx, rk = kctx
    n, w, kmin, kmax, band, pe = case
    A = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=11 * n + 1)
    B = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=11 * n + 2)
    C0 = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=11 * n + 3)
    lit = oracle.multiply(A, B, C0.widened(w).copy(), alpha, beta, tau)
    wo = max(w, ((lit.required_width + 31) // 32) * 32)
    Co = C0.widened(wo).copy()
    r = oracle.multiply(A, B, Co, alpha, beta, tau)
    assert r.status == oracle.OK
    g = up(C0.widened(wo))
    assert ctx.multiply(up(A), up(B), g, alpha, beta, tau) == eb().OK
    # in place with beta != 0: C_old is copied aside first, so the split kernels apply (the
    # warp-specialized experiment takes no Old operand: the split kernel instead)
    assert ctx.last_launch()["path"] == ("ring" if rk == 1 else ("ws" if rk == 4 and beta == 0.0 else "split"))
    assert same_bits(g.to_host(), Co)
    if lit.status != oracle.OK:
        g2 = up(C0.widened(w))
        assert ctx.multiply(up(A), up(B), g2, alpha, beta, tau) == eb().ERR_OVERFLOW
        assert ctx.overflow_info() == (lit.overflow_rows, lit.required_width)


@pytest.mark.parametrize("n,m", [(4096, 64), (32768, 128), (8192, 256)])
def test_ring_kernels_x2_traces_bitwise(kctx, n, m):
    ctx, rk = kctx
    X = synth.cfg5(n, m)
    lit = oracle.x2(X, synth.Ell.empty(n, m), 1e-5)
    w = ((lit.required_width + 31) // 32) * 32
    Y = synth.Ell.empty(n, w)
    r = oracle.x2(X, Y, 1e-5)
    y = eb().Mat.empty(n, w)
    st, tx, tx2 = ctx.multiply_x2(up(X), y, 1e-5)
    assert st == eb().OK and (tx, tx2) == (r.trace_x, r.trace_x2)
    assert same_bits(y.to_host(), Y)
    y2 = eb().Mat.empty(n, m)
    assert ctx.multiply_x2(up(X), y2, 1e-5)[0] == eb().ERR_OVERFLOW
    assert ctx.overflow_info() == (lit.overflow_rows, lit.required_width)


@pytest.mark.parametrize("n,seed,tau,rule", [(1024, 6, 1e-6, 0), (1500, 21, 1e-5, 1), (2048, 3, 1e-7, 0)])
def test_ring_kernels_sp2_bitwise(kctx, n, seed, tau, rule):
    """SP2 steps (Old = X_n: SQUARE with the norm, EXPAND with beta = 2) on whichever ring kernel."""
    ctx, rk = kctx
    H = synth.sym_banded(n, 32, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, seed)
    o = oracle.sp2(H, n // 2, 1e-10, oracle.SP2Opts(threshold=tau, max_iter=100, branch_rule=rule), d_width=n)
    d = eb().Mat.empty(n, n)
    g = ctx.sp2_run(up(H), n // 2, 1e-10, d, threshold=tau, max_iter=100, branch_rule=rule)
    _compare_sp2(g, o)
    assert same_bits(d.to_host(), o.D)
