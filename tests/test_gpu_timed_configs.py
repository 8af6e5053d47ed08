"""Parity at the configurations bench.py times, in the launch configuration it times them in
(VERDICT r1 "Next round" item 2):

- cfg5 X^2, N = 262144, M = 256 (the headline multiply): EVERY row, compared with the oracle in
  16384-row blocks (SURVEY §8d "compare in row blocks of 16384 rows"), plus tr X and tr X^2;
- SP2 on cfg3 over the K = 10 window bench.py times and on cfg4 over the first 6 iterations of its
  K = 10 window (GROW, symmetric step on, automatic regime), iterate by iterate;
- SP2 on the paper's soft-matter model Hamiltonian at N = 16384 to the stop rule (bench.py
  --workload sp2 --sp2-model soft_matter).
All bitwise.
"""
import numpy as np
import pytest

import oracle
import synth
from synth import Ell
from tests.helpers import same_bits
from tests.test_gpu_parity import _compare_sp2, eb, up

pytestmark = pytest.mark.gpu


def test_cfg5_full_size_every_row_bitwise(ctx):
    import torch
    X = synth.cfg5(262144, 256)
    x = up(X)
    y = eb().Mat.empty(X.n, 256)
    st, _, _ = ctx.multiply_x2(x, y, 1e-5)  # literal width -> required width (reading R2), as bench.py
    assert st == eb().ERR_OVERFLOW
    req = ctx.overflow_info()[1]
    w = ((req + 31) // 32) * 32
    del y
    y = eb().Mat.empty(X.n, w)
    st, tx, tx2 = ctx.multiply_x2(x, y, 1e-5)
    assert st == eb().OK
    blk = 16384
    ds = np.zeros(X.n)  # pre-drop diagonal of X^2, assembled from the blocks (tr X^2, R5)
    kept_max = 0
    for r0 in range(0, X.n, blk):
        r1 = r0 + blk
        A = Ell.empty(X.n, X.w)  # X restricted to the block's rows (rows are independent)
        A.val[r0:r1], A.col[r0:r1], A.nnz[r0:r1] = X.val[r0:r1], X.col[r0:r1], X.nnz[r0:r1]
        Y = Ell.empty(X.n, w)
        ro = oracle.multiply(A, X, Y, 1.0, 0.0, 1e-5, want_diag=True)
        assert ro.status == oracle.OK
        ds[r0:r1] = ro.diag_s[r0:r1]
        kept_max = max(kept_max, ro.required_width)
        gn = y.nnz[r0:r1].cpu().numpy()
        assert np.array_equal(gn, Y.nnz[r0:r1]), r0
        gc = y.col[r0:r1].cpu().numpy()
        gv = y.val[r0:r1].cpu().numpy()
        live = np.arange(w)[None, :] < gn[:, None]
        assert np.array_equal(gc[live], Y.col[r0:r1][live]), r0
        assert np.array_equal(gv[live].view(np.uint64), Y.val[r0:r1][live].view(np.uint64)), r0
        del A, Y, gc, gv
    assert kept_max == req  # the literal-width call's required width is the oracle's max kept count
    assert tx == oracle.trace(X) and tx2 == oracle.canonical_sum(ds)
    torch.cuda.synchronize()


@pytest.mark.parametrize("cfg,K", [(3, 10), (4, 6)])
def test_sp2_bench_window_bitwise(ctx, cfg, K):
    """The windows bench.py times (D of width min(N, 8192), GROW, default symmetric step, automatic
    regime), iterate by iterate against the oracle: cfg3's whole K = 10 window; cfg4's first 6 of its
    10 iterations (the rest: test_cfg4_bench_window_k10_regimes_agree)."""
    H, cf = (synth.cfg3(), synth.CFG3) if cfg == 3 else (synth.cfg4(), synth.CFG4)
    n = H.n
    dw = min(n + (n & 1), 8192)
    o = oracle.sp2(H, cf["nocc"], cf["tol"], oracle.SP2Opts(threshold=cf["threshold"], max_iter=K), d_width=dw)
    d = eb().Mat.empty(n, dw)
    g = ctx.sp2_run(up(H), cf["nocc"], cf["tol"], d, threshold=cf["threshold"], max_iter=K)
    assert g.status == o.status and g.iterations == K
    _compare_sp2(g, o)
    assert same_bits(d.to_host(), o.D)


def test_sp2_soft_matter_16384_to_stop_bitwise(ctx):
    n = 16384
    H = synth.model_hamiltonian(n, "soft_matter", tau_store=1e-5)
    dw = min(n, 8192)
    o = oracle.sp2(H, n // 2, 1e-8, oracle.SP2Opts(threshold=1e-5, max_iter=100), d_width=dw)
    d = eb().Mat.empty(n, dw)
    g = ctx.sp2_run(up(H), n // 2, 1e-8, d, threshold=1e-5, max_iter=100)
    assert g.status == o.status
    _compare_sp2(g, o)
    assert same_bits(d.to_host(), o.D)
