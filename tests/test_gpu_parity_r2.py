"""GPU parity for the round-2 pins and boundary checks (the sm_100a path through the C ABI vs the
CPU oracle, bitwise):

- c6 single rounding with non-dyadic alpha/beta and planted cancellations (add, scale_add_identity),
  the fixtures of tests/test_oracle_pins_c6_c10.py;
- the c10 (vi) stop-rule fixtures (STAGNATED exactly at n + 1 = min_iter with e_n = stag_gate);
- FAIL at X0 reports the exact overflow-row count (§8c-c4) on both sides;
- the iterate-memory fallbacks (headroom -> exact width; the symmetric step's U -> whole rows) give
  the same bits (ELLPACK_OPT_SP2_MEM_CAP fault injection);
- one host synchronisation per SP2 iteration (f3, first half) with bitwise-unchanged results;
- ellpack_ctx_attach_nccl rejects row blocks that are not equal multiples of 256 (1-rank comm).
"""
import numpy as np
import pytest

import oracle
import synth
from synth import from_dense
from tests.helpers import same_bits
from tests.test_gpu_parity import _compare_sp2, eb, up
from tests.test_oracle_pins_c6_c10 import (_ALPHAS, _BETAS, _bits_equal, _brute_add, _ell,
                                           _find_stagnation_fixture, _rows)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(12))
def test_c6_add_non_dyadic_gpu_bitwise(ctx, seed):
    rng = np.random.default_rng(600 + seed)
    n = int(rng.integers(10, 24)) * 7  # a few hundred rows: several warps, both paths' tails
    Am = rng.random((n, n)) < 0.05
    Bm = rng.random((n, n)) < 0.05
    A = np.where(Am, rng.standard_normal((n, n)), 0.0)
    B = np.where(Bm, rng.standard_normal((n, n)), 0.0)
    alpha, beta = _ALPHAS[seed % 4], _BETAS[(seed // 4) % 4]
    plant = Am & Bm & (rng.random((n, n)) < 0.5)
    B = np.where(plant, -alpha * A / beta, B)
    tau = [0.0, 1e-15, 1e-3][seed % 3]
    w = int(2 * max((Am | Bm).sum(axis=1).max(), 1) + 2)
    w += w & 1
    Ao, Be = _ell(A, Am, w), _ell(B, Bm, w)
    r = oracle.add(Ao, Be, alpha, beta, tau)
    assert r.status == oracle.OK
    if n <= 120:
        assert _bits_equal(_rows(Ao), _brute_add(A, Am, B, Bm, alpha, beta, tau))
    g = up(_ell(A, Am, w))
    assert ctx.add(g, up(Be), alpha, beta, tau) == eb().OK
    assert same_bits(g.to_host(), Ao)


@pytest.mark.parametrize("seed", range(8))
def test_c6_scale_add_identity_cancellation_gpu_bitwise(ctx, seed):
    rng = np.random.default_rng(700 + seed)
    n = int(rng.integers(200, 900))
    Am = rng.random((n, n)) < 0.02
    Am = Am | Am.T
    A = np.where(Am, rng.uniform(-2.0, 0.0, (n, n)), 0.0)
    emin, emax = -6.38 + 0.1 * seed, 5.09 - 0.07 * seed
    dl = emax - emin
    alpha, beta = -1.0 / dl, emax / dl
    diag = np.diag(A).copy()
    for i in range(n):
        if rng.random() < 0.5:
            Am[i, i] = True
            diag[i] = emax * (1.0 + rng.integers(-4, 5) * 2.0 ** -52)
        elif rng.random() < 0.5:
            Am[i, i] = False
            diag[i] = 0.0
    np.fill_diagonal(A, diag)
    tau = [0.0, 1e-17, 1e-5][seed % 3]
    w = int(Am.sum(axis=1).max() + 2)
    w += w & 1
    Ao = _ell(A, Am, w)
    r = oracle.scale_add_identity(Ao, alpha, beta, tau)
    assert r.status == oracle.OK
    g = up(_ell(A, Am, w))
    assert ctx.scale_add_identity(g, alpha, beta, tau) == eb().OK
    assert same_bits(g.to_host(), Ao)


@pytest.mark.parametrize("tau,nlev,seeds", [(0.0, 9, range(0, 400)), (1e-3, 12, range(400, 800)),
                                              (0.0, 30, range(800, 1200))])
def test_c10_stagnation_fixtures_gpu(ctx, tau, nlev, seeds):
    """The stop iteration of each stop-rule fixture, on the GPU: STAGNATED at exactly n + 1."""
    h, nocc, recs, n = _find_stagnation_fixture(tau, nlev, seeds)
    gate = recs[n][3]
    H = from_dense(np.diag(h), w=2)
    for min_iter, g_ in ((n + 1, gate), (n + 2, gate), (n + 1, float(np.nextafter(gate, -np.inf)))):
        o = oracle.sp2(H, nocc, 0.0, oracle.SP2Opts(threshold=tau, max_iter=60, min_iter=min_iter, stag_gate=g_),
                       d_width=len(h) + (len(h) & 1))
        d = eb().Mat.empty(len(h), len(h) + (len(h) & 1))
        g = ctx.sp2_run(up(H), nocc, 0.0, d, threshold=tau, max_iter=60, min_iter=min_iter, stag_gate=g_)
        _compare_sp2(g, o)
        assert same_bits(d.to_host(), o.D)
    assert o.iterations != n + 1  # (the last variant: gate one ulp below e_n)


def test_sp2_fail_at_x0_overflow_rows_gpu(ctx):
    H = synth.sym_banded(300, 40, 10, 30, 1, -1.0, 1.0, 0, 10.0, 0.0, 31)
    o = oracle.sp2(H, 150, 1e-8, oracle.SP2Opts(threshold=0.0, on_overflow=0, initial_width=16), d_width=300)
    assert o.status == oracle.OVERFLOW and o.fail_iter == -1 and o.overflow_rows > 0
    d = eb().Mat.empty(300, 300)
    g = ctx.sp2_run(up(H), 150, 1e-8, d, on_overflow=eb().SP2_FAIL, initial_width=16)
    assert g.status == eb().ERR_OVERFLOW
    assert (g.fail_iter, g.required_width, g.overflow_rows) == (o.fail_iter, o.required_width, o.overflow_rows)
    assert ctx.overflow_info() == (o.overflow_rows, o.required_width)


@pytest.mark.parametrize("slack", [8, 4096])
def test_sp2_iterate_memory_fallbacks_bitwise(ellpack_lib, slack):
    """ELLPACK_OPT_SP2_MEM_CAP = room for X_n and X_{n+1} at the final width (+ slack columns): the
    x8 / x4 headroom widths "do not fit" (fallback to the exact width, slot released first) and,
    with little slack, neither does the symmetric step's upper triangle (whole rows instead)."""
    E = ellpack_lib
    n = 1024
    H = synth.sym_banded(n, 32, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, 6)
    o = oracle.sp2(H, n // 2, 1e-10, oracle.SP2Opts(threshold=1e-6, max_iter=100), d_width=n)
    assert o.final_width > 256  # the general path (and its symmetric route) runs
    ctx = E.Context(0)
    ctx.set_option(E.OPT_SP2_DEVICE_LOOP, 1)  # headroom widths and the symmetric step: the host loop
    ctx.set_option(E.OPT_DENSE, 1)  # the sparse kernels' U buffer fallback
    ctx.set_option(E.OPT_SP2_MEM_CAP, 8 * n * (2 * o.final_width + slack))
    d = E.Mat.empty(n, n)
    g = ctx.sp2_run(up(H), n // 2, 1e-10, d, threshold=1e-6, max_iter=100)
    _compare_sp2(g, o)
    assert same_bits(d.to_host(), o.D)
    ctx.close()


def test_sp2_one_host_sync_per_iteration(ellpack_lib):
    """f3 (first half): every SP2 iteration waits on the device exactly once (the probe of X_{n+1}
    travels with the step's status); two windows differ by exactly their iteration count."""
    E = ellpack_lib
    n = 2048
    H = synth.sym_banded(n, 32, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, 3)
    syncs = {}
    for K in (4, 12):
        ctx = E.Context(0)
        ctx.set_option(E.OPT_SP2_DEVICE_LOOP, 1)  # the host loop: one synchronisation per iteration
        ctx.set_option(E.OPT_SP2_SYMMETRIC, 0)
        d = E.Mat.empty(n, n)
        s0 = ctx.host_syncs()
        # the initial width n: no physical regrow (which redoes a step) inside the window
        g = ctx.sp2_run(up(H), n // 2, 0.0, d, threshold=1e-7, max_iter=K, min_iter=100, initial_width=n)
        syncs[K] = ctx.host_syncs() - s0
        assert g.iterations == K
        o = oracle.sp2(H, n // 2, 0.0, oracle.SP2Opts(threshold=1e-7, max_iter=K, min_iter=100, initial_width=n),
                       d_width=n)
        _compare_sp2(g, o)
        assert same_bits(d.to_host(), o.D)
        ctx.close()
    assert syncs[12] - syncs[4] == 8, syncs


def test_attach_nccl_checks_row_blocks(ellpack_lib):
    import torch  # noqa: F401  (torch's libnccl.so.2 for the library's dlopen)
    E = ellpack_lib
    uid = E.Context.nccl_unique_id()
    ctx = E.Context(0)
    with pytest.raises(E.EllpackError) as ei:
        ctx.attach_nccl(1, 0, uid, 0, 1000)  # not a multiple of 256 rows
    assert ei.value.status == E.ERR_ARG
    ctx.close()
    ctx = E.Context(0)
    ctx.attach_nccl(1, 0, E.Context.nccl_unique_id(), 0, 1024)
    X = synth.cfg5(2048, 32)
    with pytest.raises(E.EllpackError) as ei:  # operands must be the N the blocks cover
        ctx.multiply_x2(up(X), E.Mat.empty(2048, 1024), 1e-5)
    assert ei.value.status == E.ERR_DIM
    ctx.close()


# ---------------------------------------------- f3: the device-resident SP2 loop (CUDA graph)

DEVLOOP = [
    # (n, m, partners, band, seed, tau, rule, width0, nocc_frac, on_overflow)
    (512, 32, 6, 12, 2, 0.0, 0, 0, 0.5, 1),
    (600, 64, 10, 100, 14, 1e-4, 1, 0, 0.5, 1),
    (513, 32, 8, 64, 13, 1e-4, 0, 16, 0.7, 1),
    (1024, 32, 6, 12, 6, 1e-6, 0, 8, 0.5, 1),
    (2048, 32, 6, 12, 3, 1e-7, 1, 0, 0.5, 1),
    (300, 40, 10, 30, 31, 0.0, 0, 64, 0.5, 0),   # FAIL inside the loop: exact report
]


@pytest.mark.parametrize("case", DEVLOOP, ids=lambda c: f"n{c[0]}tau{c[5]}r{c[6]}f{c[9]}")
def test_sp2_device_loop_bitwise(ellpack_lib, case):
    """§8f-f3: the loop as one CUDA-graph launch (branch, stop and width rules on the device) is
    bitwise the oracle and the host loop, report included, with a constant number of host
    synchronisations per run (none per iteration)."""
    E = ellpack_lib
    n, m, partners, band, seed, tau, rule, w0, frac, onov = case
    H = synth.sym_banded(n, m, partners, band, 1, -1.0, 1.0, 0, band / 4.0, 0.0, seed)
    nocc = int(frac * n)
    o = oracle.sp2(H, nocc, 1e-9, oracle.SP2Opts(threshold=tau, max_iter=100, branch_rule=rule, initial_width=w0,
                                                 on_overflow=onov), d_width=n + (n & 1))
    res = {}
    for loop in (2, 1):
        ctx = E.Context(0)
        ctx.set_option(E.OPT_SP2_DEVICE_LOOP, loop)
        ctx.set_option(E.OPT_SP2_SYMMETRIC, 0)
        if w0:
            ctx.set_option(E.OPT_SP2_WIDTH0, w0)
        d = E.Mat.empty(n, n + (n & 1))
        s0 = ctx.host_syncs()
        g = ctx.sp2_run(up(H), nocc, 1e-9, d, threshold=tau, max_iter=100, branch_rule=rule, on_overflow=onov)
        res[loop] = (g, ctx.host_syncs() - s0, d.to_host())
        assert g.status == o.status
        if o.status == oracle.OVERFLOW:
            assert (g.fail_iter, g.required_width, g.overflow_rows) == (o.fail_iter, o.required_width, o.overflow_rows)
        else:
            _compare_sp2(g, o)
            assert same_bits(res[loop][2], o.D)
        ctx.close()
    if o.status != oracle.OVERFLOW:
        assert res[1][1] >= res[2][1] + o.iterations - 2  # the host loop waits once per iteration


def test_sp2_device_loop_syncs_do_not_grow_with_iterations(ellpack_lib):
    E = ellpack_lib
    n = 1024
    H = synth.sym_banded(n, 32, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, 3)
    syncs = {}
    for K in (4, 16):
        ctx = E.Context(0)
        ctx.set_option(E.OPT_SP2_DEVICE_LOOP, 2)
        d = E.Mat.empty(n, n)
        ctx.sp2_run(up(H), n // 2, 0.0, d, threshold=1e-7, max_iter=K, min_iter=100)  # graph built
        s0 = ctx.host_syncs()
        g = ctx.sp2_run(up(H), n // 2, 0.0, d, threshold=1e-7, max_iter=K, min_iter=100)
        syncs[K] = ctx.host_syncs() - s0
        assert g.iterations == K
        o = oracle.sp2(H, n // 2, 0.0, oracle.SP2Opts(threshold=1e-7, max_iter=K, min_iter=100), d_width=n)
        _compare_sp2(g, o)
        assert same_bits(d.to_host(), o.D)
        ctx.close()
    assert syncs[16] == syncs[4], syncs


# --------------------------------------- f1: halo exchange overlapped with the interior rows

@pytest.mark.parametrize("nranks", [1, 2, 4, 8])
@pytest.mark.parametrize("m,kernel", [(64, 0), (256, 0), (64, 1)])
def test_multiply_x2_halo_interior_boundary_bitwise(ellpack_lib, nranks, m, kernel):
    """ellpack_multiply_x2_halo splits a rank's block into interior rows (computed while the halo
    travels) and boundary rows (after it): emulated ranks (ellpack_ctx_set_rows) on one GPU, every
    ring kernel, the union of the blocks bitwise the one-rank product (§8c-c12)."""
    E = ellpack_lib
    n = 32768
    X = synth.cfg5(n, m)
    w = {64: 864, 256: 5248}[m]
    full = E.Context(0)
    y1 = E.Mat.empty(n, w)
    st, tx, tx2 = full.multiply_x2(up(X), y1, 1e-5)
    assert st == E.OK
    full.close()
    x = up(X)
    yp = E.Mat.empty(n, w)
    for (r0, r1) in E.row_partition(n, nranks):
        c = E.Context(0)
        if kernel:
            c.set_option(E.OPT_RING_KERNEL, kernel)
        if nranks > 1:
            c.set_rows(r0, r1)
        st, tx_h, tx2_h = c.multiply_x2_halo(x, yp, 1e-5)
        assert st == E.OK
        if nranks == 1:
            assert (tx_h, tx2_h) == (tx, tx2)
        c.close()
    assert same_bits(yp.to_host(), y1.to_host())


def test_multiply_x2_halo_one_rank_communicator(ellpack_lib):
    import torch  # noqa: F401
    E = ellpack_lib
    n = 4096
    X = synth.cfg5(n, 64)
    Y = synth.Ell.empty(n, 1024)
    r = oracle.x2(X, Y, 1e-5)
    ctx = E.Context(0)
    ctx.attach_nccl(1, 0, E.Context.nccl_unique_id(), 0, n)
    y = E.Mat.empty(n, 1024)
    st, tx, tx2 = ctx.multiply_x2_halo(up(X), y, 1e-5)
    assert st == E.OK and (tx, tx2) == (r.trace_x, r.trace_x2)
    assert same_bits(y.to_host(), Y)
    ctx.close()


def test_sp2_symmetric_step_with_communicator(ellpack_lib):
    """The symmetric step with a communicator (1-rank comm on this pool): the upper route runs (the
    executed products are about half the pattern's), the U halo and the all-reduced reach are on the
    path, and every iterate is bitwise the oracle's."""
    import torch  # noqa: F401
    E = ellpack_lib
    n = 1024
    H = synth.sym_banded(n, 32, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, 6)
    o = oracle.sp2(H, n // 2, 1e-10, oracle.SP2Opts(threshold=1e-6, max_iter=100), d_width=n)
    ctx = E.Context(0)
    ctx.attach_nccl(1, 0, E.Context.nccl_unique_id(), 0, n)
    ctx.set_option(E.OPT_DENSE, 1)  # the sparse kernels' symmetric route (the dense regime: below)
    d = E.Mat.empty(n, n)
    g = ctx.sp2_run(up(H), n // 2, 1e-10, d, threshold=1e-6, max_iter=100)
    _compare_sp2(g, o)
    assert same_bits(d.to_host(), o.D)
    assert any(it["products_exec"] < 0.75 * it["products"] for it in g.iters)  # the upper route ran
    ctx.close()


@pytest.mark.parametrize("dense", [2, 0])
def test_sp2_dense_with_communicator(ellpack_lib, dense):
    """The dense regime with a communicator (1-rank comm): forced, and chosen automatically from
    all-reduced inputs only (band model, fixed rates) -- bitwise the oracle."""
    E = ellpack_lib
    n = 1024
    H = synth.sym_banded(n, 32, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, 6)
    o = oracle.sp2(H, n // 2, 1e-10, oracle.SP2Opts(threshold=1e-6, max_iter=100), d_width=n)
    ctx = E.Context(0)
    ctx.attach_nccl(1, 0, E.Context.nccl_unique_id(), 0, n)
    ctx.set_option(E.OPT_DENSE, dense)
    d = E.Mat.empty(n, n)
    g = ctx.sp2_run(up(H), n // 2, 1e-10, d, threshold=1e-6, max_iter=100)
    _compare_sp2(g, o)
    assert same_bits(d.to_host(), o.D)
    regimes = [it["regime"] for it in g.iters]
    assert (all(r == "dense" for r in regimes) if dense == 2 else "dense" in regimes)
    ctx.close()


@pytest.mark.parametrize("n,nranks", [(8192, 2), (8192, 4), (1024, 4)])
def test_dense_row_blocks_bitwise(ellpack_lib, n, nranks):
    """A rank's rows in the dense regime (ellpack_ctx_set_rows, emulated ranks): GEMM tiles of its
    row blocks only (row offset; 128-row and 16-row tiles), X^T = X read from the one dense copy; the
    union of the blocks equals the single-rank product bit for bit."""
    E = ellpack_lib
    X = synth.cfg5(n, 64)
    wo = 1024
    full = E.Context(0)
    y1 = E.Mat.empty(n, wo)
    assert full.multiply_x2(up(X), y1, 1e-5)[0] == E.OK
    full.close()
    yp = E.Mat.empty(n, wo)
    x = up(X)
    for (r0, r1) in E.row_partition(n, nranks):
        c = E.Context(0)
        c.set_option(E.OPT_DENSE, 2)
        c.set_rows(r0, r1)
        c.multiply_x2(x, yp, 1e-5)
        assert c.last_launch()["path"] == "dense"
        c.close()
    assert same_bits(yp.to_host(), y1.to_host())


def test_small_x2_graph_replay_bitwise(ellpack_lib):
    """N <= 1024 X^2 is captured once as a CUDA graph and replayed: the replay reads the operands'
    CURRENT contents (rewritten in place between calls), a new tau or a changed option re-captures,
    an overflow is reported through the replay, and every call equals the oracle bitwise with one
    host synchronisation."""
    import torch
    ctx = ellpack_lib.Context(0)
    ctx.set_option(ellpack_lib.OPT_SMALL_KERNEL, 1)  # the general path's graph (row kernel + sums)
    try:
        n, w = 600, 24
        Xs = [synth.random_sparse(n, w, 4, w, band=40, seed=900 + s) for s in range(3)]
        x = up(Xs[0])
        y = ellpack_lib.Mat.empty(n, 256)

        def check(X, tau, w_out=256, y_=None, syncs=1):
            y_ = y if y_ is None else y_
            s0 = ctx.host_syncs()
            st, tx, tx2 = ctx.multiply_x2(x, y_, tau)
            assert ctx.host_syncs() - s0 == syncs
            Y = oracle.Ell.empty(n, w_out)
            r = oracle.x2(X, Y, tau)
            assert st == r.status
            if st == ellpack_lib.OK:
                assert same_bits(y_.to_host(), Y)
                assert np.float64(tx).view(np.uint64) == np.float64(r.trace_x).view(np.uint64)
                assert np.float64(tx2).view(np.uint64) == np.float64(r.trace_x2).view(np.uint64)
            else:
                assert ctx.overflow_info() == (r.overflow_rows, r.required_width)
            return st

        for k in range(6):  # capture, replays, operands rewritten in place between replays
            X = Xs[k % 3]
            if k:
                h = up(X)
                x.val.copy_(h.val)
                x.col.copy_(h.col)
                x.nnz.copy_(h.nnz)
                torch.cuda.synchronize()
            assert check(X, 1e-5) == ellpack_lib.OK
        assert ctx.last_launch()["path"] == "general"
        l0 = ctx.kernel_launches()
        check(Xs[2], 1e-5)
        assert ctx.kernel_launches() - l0 == 2  # the captured kernels are counted on every replay
        assert check(Xs[2], 0.0) == ellpack_lib.OK  # new tau: re-capture
        wpc = ctx.last_launch()["warps_per_cta"]
        ctx.set_option(ellpack_lib.OPT_WARPS, 1 if wpc != 1 else 2)  # any option change: re-capture
        assert check(Xs[2], 1e-3) == ellpack_lib.OK
        assert ctx.last_launch()["warps_per_cta"] == (1 if wpc != 1 else 2)
        ctx.set_option(ellpack_lib.OPT_WINDOW, 64)  # a forced window: not graphed, still bitwise
        assert check(Xs[2], 1e-3, syncs=2) == ellpack_lib.OK  # probed: the window is planned on the host
        assert ctx.last_launch()["S"] == 64
        ctx.set_option(ellpack_lib.OPT_WINDOW, 0)
        assert check(Xs[2], 1e-3) == ellpack_lib.OK
        assert ctx.last_launch()["S"] > 64
        ys = ellpack_lib.Mat.empty(n, 8)  # too narrow: the overflow comes back through the replay
        assert check(Xs[2], 1e-9, 8, ys) == ellpack_lib.ERR_OVERFLOW
        assert check(Xs[2], 1e-9, 8, ys) == ellpack_lib.ERR_OVERFLOW
    finally:
        ctx.close()


@pytest.mark.parametrize("n,w,kmin,band,p_empty,seed", [
    (1, 4, 1, None, 0.0, 0), (7, 8, 0, None, 0.3, 1), (33, 16, 2, 8, 0.0, 2), (129, 32, 1, 40, 0.1, 3),
    (256, 32, 32, None, 0.0, 4), (600, 24, 4, 40, 0.0, 5), (1000, 48, 8, 300, 0.05, 6),
    (1024, 64, 60, None, 0.0, 7), (513, 40, 0, 64, 0.5, 8)])
def test_small_kernel_bitwise(ellpack_lib, n, w, kmin, band, p_empty, seed):
    """The small-matrix kernel (tiny.cu: N <= 1024, input width <= 64, the default for
    ellpack_multiply_x2 there) against the oracle and against the general path
    (ELLPACK_OPT_SMALL_KERNEL 1), bitwise: values, patterns, traces, literal-width overflow reports;
    one launch and one host synchronisation per call, replayed from the captured graph."""
    X = synth.random_sparse(n, w, kmin, w, band=band, p_empty=p_empty, seed=1700 + seed)
    x = up(X)
    outs = {}
    for small in (0, 1):
        ctx = ellpack_lib.Context(0)
        try:
            ctx.set_option(ellpack_lib.OPT_SMALL_KERNEL, small)
            for tau, w_out in ((1e-5, min(n + (n & 1), 1024)), (0.0, min(n + (n & 1), 1024)), (1e-9, 4)):
                y = ellpack_lib.Mat.empty(n, w_out)
                Y = oracle.Ell.empty(n, w_out)
                r = oracle.x2(X, Y, tau)
                for rep in range(2):  # capture, then a replay
                    l0, s0 = ctx.kernel_launches(), ctx.host_syncs()
                    st, tx, tx2 = ctx.multiply_x2(x, y, tau)
                    assert st == r.status
                    assert ctx.host_syncs() - s0 == 1
                    if small == 0:
                        assert ctx.kernel_launches() - l0 == 1
                    if st == ellpack_lib.OK:
                        assert same_bits(y.to_host(), Y)
                        assert np.float64(tx).view(np.uint64) == np.float64(r.trace_x).view(np.uint64)
                        assert np.float64(tx2).view(np.uint64) == np.float64(r.trace_x2).view(np.uint64)
                        outs.setdefault((tau, w_out), []).append((y.to_host(), tx, tx2))
                    else:
                        assert ctx.overflow_info() == (r.overflow_rows, r.required_width)
        finally:
            ctx.close()
    for k, v in outs.items():  # both paths, every call: the same bits
        for (a, ta, ta2) in v[1:]:
            assert same_bits(a, v[0][0]) and (ta, ta2) == (v[0][1], v[0][2])
