"""GPU parity: the sm_100a path (through the C ABI) vs the CPU oracle on identical seeded inputs.

The bar (BJ north_star): with the pinned ascending-k fma
order and canonical trace tree both sides compute the same IEEE result, so every
comparison here is BITWISE (values, patterns, nnz, traces, overflow reports,
SP2 branch sequences) -- stricter than the 1e-12 per-entry / 1e-10 trace
tolerance the north star allows. fnorm_diff (order unpinned, diagnostic) is
compared at 1e-12 relative.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from synth import Ell, from_dense
from tests.helpers import entries_of, load_golden, same_bits, ell_from_entries

pytestmark = pytest.mark.gpu


def eb():
    import paper_2102_08505_b200 as m
    return m


def same_bits_scalar(a, b):
    return np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64)


def up(e: Ell, w=None):
    return eb().Mat.from_host(e, w=w)


def gpu_x2(ctx, X: Ell, w_out: int, tau: float):
    x = up(X)
    y = eb().Mat.empty(X.n, w_out)
    st, tx, tx2 = ctx.multiply_x2(x, y, tau)
    return st, y.to_host(), tx, tx2


def ora_x2(X: Ell, w_out: int, tau: float):
    Y = Ell.empty(X.n, w_out)
    r = oracle.x2(X, Y, tau)
    return r, Y


# ----------------------------------------------------------------- configs 1, 2, 5

def test_cfg1_x2_bitwise_and_literal_overflow(ctx):
    X = synth.cfg1()
    tau = synth.CFG1["threshold"]
    r, Y = ora_x2(X, 256, tau)
    st, G, tx, tx2 = gpu_x2(ctx, X, 256, tau)
    assert r.status == oracle.OK and st == eb().OK
    assert same_bits(G, Y)
    assert (tx, tx2) == (r.trace_x, r.trace_x2)
    # literal M = 32 (reading R2): OVERFLOW with the oracle's exact report
    r32, _ = ora_x2(X, 32, tau)
    st32, _, _, _ = gpu_x2(ctx, X, 32, tau)
    assert r32.status == oracle.OVERFLOW and st32 == eb().ERR_OVERFLOW
    assert ctx.overflow_info() == (r32.overflow_rows, r32.required_width)


def test_cfg2_multiply_bitwise_in_place(ctx):
    A, B, C = synth.cfg2()
    cf = synth.CFG2
    # literal width M = 128 -> overflow report
    Cl = C.copy()
    rl = oracle.multiply(A, B, Cl, cf["alpha"], cf["beta"], cf["threshold"])
    g = up(C)
    stl = ctx.multiply(up(A), up(B), g, cf["alpha"], cf["beta"], cf["threshold"])
    assert rl.status == oracle.OVERFLOW and stl == eb().ERR_OVERFLOW
    assert ctx.overflow_info() == (rl.overflow_rows, rl.required_width)
    w = ((rl.required_width + 31) // 32) * 32
    Co = C.widened(w)
    r = oracle.multiply(A, B, Co, cf["alpha"], cf["beta"], cf["threshold"])
    g = up(C, w=w)
    st = ctx.multiply(up(A), up(B), g, cf["alpha"], cf["beta"], cf["threshold"])
    assert r.status == oracle.OK and st == eb().OK
    assert same_bits(g.to_host(), Co)


@pytest.mark.parametrize("m", [64, 128, 256])
def test_cfg5_small_n_x2_bitwise(ctx, m):
    X = synth.cfg5(32768, m)
    r, Y = ora_x2(X, 32 * m, 1e-5)
    assert r.status == oracle.OK
    w = ((r.required_width + 31) // 32) * 32
    st, G, tx, tx2 = gpu_x2(ctx, X, w, 1e-5)
    assert st == eb().OK
    assert same_bits(G, Y)
    assert (tx, tx2) == (r.trace_x, r.trace_x2)


def _sample_rows_oracle(X: Ell, rows, w_out, tau):
    """Oracle X^2 restricted to `rows` (A = X with other rows emptied; B = X)."""
    A = Ell.empty(X.n, X.w)
    for i in rows:
        A.val[i] = X.val[i]
        A.col[i] = X.col[i]
        A.nnz[i] = X.nnz[i]
    Y = Ell.empty(X.n, w_out)
    r = oracle.multiply(A, X, Y, 1.0, 0.0, tau)
    return r, Y


def test_cfg5_full_size_sampled_rows_bitwise(ctx):
    """BASELINE cfg5 largest (N=262144, M=256) in the bench's launch configuration."""
    X = synth.cfg5(262144, 256)
    x = up(X)
    y = eb().Mat.empty(X.n, 256)
    st, _, _ = ctx.multiply_x2(x, y, 1e-5)  # literal width -> required width (reading R2)
    assert st == eb().ERR_OVERFLOW
    w = ((ctx.overflow_info()[1] + 31) // 32) * 32
    y = eb().Mat.empty(X.n, w)
    st, tx, tx2 = ctx.multiply_x2(x, y, 1e-5)
    assert st == eb().OK
    rng = np.random.default_rng(0)
    rows = sorted(set(rng.integers(0, X.n, 384).tolist()) | {0, 1, X.n - 1, X.n // 2})
    r, Y = _sample_rows_oracle(X, rows, w, 1e-5)
    assert r.status == oracle.OK
    idx = torch_index(rows)
    gv, gc, gn = y.val[idx].cpu().numpy(), y.col[idx].cpu().numpy(), y.nnz[idx].cpu().numpy()
    for t, i in enumerate(rows):
        k = int(Y.nnz[i])
        assert gn[t] == k
        assert np.array_equal(gc[t, :k], Y.col[i, :k])
        assert np.array_equal(gv[t, :k].view(np.uint64), Y.val[i, :k].view(np.uint64))
    # traces: the exact tr(X) of the oracle; tr(X^2) = ||X||_F^2 property (P5) at any size
    assert tx == oracle.trace(X)
    live = np.arange(X.w)[None, :] < X.nnz[:, None]
    fro2 = math.fsum((X.val[live] ** 2).tolist())
    assert abs(tx2 - fro2) <= 1e-12 * fro2


def torch_index(rows):
    import torch
    return torch.tensor(rows, dtype=torch.long, device="cuda")


def test_x2_of_symmetric_is_bitwise_symmetric_gpu(ctx):
    """P4 on the GPU alone (no oracle needed): cfg5 N=32768, M=64."""
    X = synth.cfg5(32768, 64)
    st, G, _, _ = gpu_x2(ctx, X, 1024, 1e-5)
    assert st == eb().OK
    import scipy.sparse as sp
    rows = np.repeat(np.arange(G.n), G.nnz)
    mask = np.arange(G.w)[None, :] < G.nnz[:, None]
    M = sp.csr_matrix((G.val[mask], (rows, G.col[mask])), shape=(G.n, G.n))
    D = (M - M.T)
    assert D.count_nonzero() == 0


# --------------------------------------------------------------------- edge cases

EDGE = [
    # (n, w, kmin, kmax, band, p_empty, w_out)
    (1, 2, 0, 1, 1, 0.0, 2),
    (2, 2, 1, 2, 2, 0.0, 2),
    (31, 8, 0, 8, 31, 0.2, 32),
    (33, 8, 8, 8, 6, 0.0, 40),      # full rows (nnz = w)
    (1000, 16, 0, 16, 40, 0.3, 200),
    (4097, 32, 1, 32, 300, 0.05, 700),
]


@pytest.mark.parametrize("case", EDGE, ids=lambda c: f"n{c[0]}w{c[1]}")
@pytest.mark.parametrize("alpha,beta,tau", [(1.0, 0.0, 0.0), (0.75, -1.5, 1e-3), (0.0, 2.0, 0.0), (-1.0, 0.5, 0.1)])
def test_multiply_edge_cases_bitwise(ctx, case, alpha, beta, tau):
    n, w, kmin, kmax, band, pe, wo = case
    A = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=n + 1)
    B = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=n + 2)
    C = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=n + 3).widened(wo)
    Co = C.copy()
    r = oracle.multiply(A, B, Co, alpha, beta, tau)
    g = up(C)
    if beta == 0.0:
        g.val.fill_(float("nan"))  # C_old must never be read when beta == 0 (R13)
    st = ctx.multiply(up(A), up(B), g, alpha, beta, tau)
    assert st == (eb().OK if r.status == oracle.OK else eb().ERR_OVERFLOW)
    if r.status == oracle.OK:
        assert same_bits(g.to_host(), Co)
    else:
        assert ctx.overflow_info() == (r.overflow_rows, r.required_width)


# Ring fast path with wide B rows: every group count G = 1..4 (B rows up to 256 entries),
# row lengths straddling the 64-entry group and 16-entry bin boundaries, empty rows, and the
# Old operand (beta != 0). The half-bandwidth keeps the ring within the fast path's limit.
FAST = [
    # (n, w, kmin, kmax, band, p_empty)
    (2048, 64, 48, 64, 500, 0.02),    # G = 1
    (2500, 128, 1, 128, 800, 0.05),   # G = 2, ragged
    (3001, 192, 120, 192, 1200, 0.0),  # G = 3
    (3000, 256, 180, 256, 1800, 0.01),  # G = 4, bins up to 16
]


@pytest.mark.parametrize("case", FAST, ids=lambda c: f"n{c[0]}w{c[1]}")
@pytest.mark.parametrize("alpha,beta,tau", [(1.0, 0.0, 0.0), (0.75, -1.5, 1e-3)])
def test_fast_path_wide_rows_bitwise(ctx, case, alpha, beta, tau):
    n, w, kmin, kmax, band, pe = case
    A = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=7 * n + 1)
    B = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=7 * n + 2)
    C0 = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=7 * n + 3)
    lit = oracle.multiply(A, B, C0.widened(w).copy(), alpha, beta, tau)  # literal width -> required
    wo = max(w, ((lit.required_width + 31) // 32) * 32)
    Co = C0.widened(wo).copy()
    r = oracle.multiply(A, B, Co, alpha, beta, tau)
    assert r.status == oracle.OK
    g = up(C0.widened(wo))
    st = ctx.multiply(up(A), up(B), g, alpha, beta, tau)
    assert st == eb().OK
    assert same_bits(g.to_host(), Co)
    # and the literal width reports the oracle's overflow exactly
    if lit.status != oracle.OK:
        g2 = up(C0.widened(w))
        assert ctx.multiply(up(A), up(B), g2, alpha, beta, tau) == eb().ERR_OVERFLOW
        assert ctx.overflow_info() == (lit.overflow_rows, lit.required_width)


def _fuzz_cases(count=24, seed=2102):
    rng = np.random.default_rng(seed)
    out = []
    for t in range(count):
        n = int(rng.choice([1, 7, 31, 32, 33, 100, 257, 1000, 2049, 3000]))
        w = int(rng.choice([2, 8, 32, 64, 96, 128, 200, 256, 300]))
        kmax = int(min(w, max(1, rng.integers(1, w + 1))))
        kmin = int(rng.integers(0, kmax + 1))
        band = int(rng.choice([1, 4, 50, 300, 5000]))
        pe = float(rng.choice([0.0, 0.1, 0.5]))
        ab = [(1.0, 0.0, 0.0), (0.75, -1.5, 1e-3), (-1.0, 2.0, 1e-6), (0.0, 1.0, 0.0), (2.0, 0.5, 0.5)][t % 5]
        out.append((t, n, w, kmin, kmax, band, pe) + ab)
    # the general path for sure: B rows over 256 entries; a half-bandwidth beyond any ring
    out += [(count, 1500, 300, 257, 300, 2000, 0.0, 1.0, 0.0, 1e-6),
            (count + 1, 2500, 300, 200, 300, 1500, 0.05, 0.75, -1.5, 1e-3),
            (count + 2, 8000, 32, 16, 32, 8000, 0.0, 1.0, 0.0, 0.0),
            (count + 3, 8000, 32, 8, 32, 8000, 0.1, -1.0, 2.0, 1e-6)]
    return out


@pytest.mark.parametrize("case", _fuzz_cases(), ids=lambda c: f"t{c[0]}n{c[1]}w{c[2]}")
def test_random_multiply_fuzz_bitwise(ctx, case):
    """Seeded random shapes across both paths (ring and general: B rows up to 300 entries,
    half-bandwidths up to 5000), ragged/empty rows and the alpha/beta/tau corners; the output
    width is the oracle's required width, and the literal width's overflow report must match."""
    t, n, w, kmin, kmax, band, pe, alpha, beta, tau = case
    w += w & 1
    A = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=1000 + 3 * t)
    B = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=1001 + 3 * t)
    C0 = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=1002 + 3 * t)
    lit = oracle.multiply(A, B, C0.copy(), alpha, beta, tau)
    wo = max(w, ((lit.required_width + 31) // 32) * 32)
    wo += wo & 1
    Co = C0.widened(wo).copy()
    r = oracle.multiply(A, B, Co, alpha, beta, tau)
    assert r.status == oracle.OK
    g = up(C0.widened(wo))
    assert ctx.multiply(up(A), up(B), g, alpha, beta, tau) == eb().OK
    assert same_bits(g.to_host(), Co)
    if lit.status != oracle.OK:
        g2 = up(C0)
        assert ctx.multiply(up(A), up(B), g2, alpha, beta, tau) == eb().ERR_OVERFLOW
        assert ctx.overflow_info() == (lit.overflow_rows, lit.required_width)


@pytest.mark.parametrize("window", [32, 64, 256])
@pytest.mark.parametrize("beta", [0.0, 0.5])
def test_multipass_window_and_stash_bitwise(ellpack_lib, window, beta):
    """Force rows wider than the dense window: multi-pass cursors + in-place stash paths."""
    ctx = ellpack_lib.Context(0)
    ctx.set_option(ellpack_lib.OPT_WINDOW, window)
    A = synth.random_sparse(3000, 24, 0, 24, 200, 0.05, 1.0, seed=71)
    B = synth.random_sparse(3000, 48, 0, 48, 150, 0.05, 1.0, seed=72)
    C = synth.random_sparse(3000, 24, 0, 24, 300, 0.05, 1.0, seed=73).widened(1024)
    Co = C.copy()
    r = oracle.multiply(A, B, Co, 1.25, beta, 1e-4)
    g = up(C)
    st = ctx.multiply(up(A), up(B), g, 1.25, beta, 1e-4)
    assert r.status == oracle.OK and st == ellpack_lib.OK
    assert same_bits(g.to_host(), Co)
    # x2 + traces under multi-pass
    X = synth.cfg5(4096, 64)
    rr, Y = ora_x2(X, 1024, 1e-5)
    st, G, tx, tx2 = gpu_x2(ctx, X, 1024, 1e-5)
    assert same_bits(G, Y) and (tx, tx2) == (rr.trace_x, rr.trace_x2)
    # add family in place with multi-pass stash
    A2 = A.widened(64)
    ga = up(A2)
    Bd = synth.random_sparse(3000, 24, 0, 24, 300, 0.05, 1.0, seed=74)
    r2 = oracle.add(A2, Bd, 0.5, -1.0, 0.0)
    st2 = ctx.add(ga, up(Bd), 0.5, -1.0, 0.0)
    assert r2.status == oracle.OK and st2 == ellpack_lib.OK
    assert same_bits(ga.to_host(), A2)
    ctx.close()


def test_aliasing_and_argument_errors(ctx):
    X = synth.cfg1()
    x = up(X, w=256)
    with pytest.raises(eb().EllpackError) as e:
        ctx.multiply(x, up(X), x, 1.0, 0.0, 0.0)
    assert e.value.status == eb().ERR_ARG
    with pytest.raises(eb().EllpackError) as e:
        ctx.multiply_x2(x, x, 0.0)
    assert e.value.status == eb().ERR_ARG
    with pytest.raises(eb().EllpackError) as e:
        ctx.multiply_x2(up(X), eb().Mat.empty(X.n, 256), -1.0)
    assert e.value.status == eb().ERR_ARG
    with pytest.raises(eb().EllpackError) as e:
        ctx.multiply(up(X), up(synth.cfg5(32768, 64)), eb().Mat.empty(X.n, 256), 1.0, 0.0, 0.0)
    assert e.value.status == eb().ERR_DIM


# ------------------------------------------------------------- add / reductions

def test_add_family_trace_fnorm_gershgorin(ctx):
    A = synth.random_sparse(2000, 20, 0, 20, 100, 0.1, 1.0, seed=81)
    B = synth.random_sparse(2000, 20, 0, 20, 100, 0.1, 1.0, seed=82)
    for alpha, beta, tau in [(1.0, 0.0, 0.0), (0.5, -2.0, 1e-3), (1.0, -1.0, 0.0)]:
        Ao = A.widened(48)
        r = oracle.add(Ao, B, alpha, beta, tau)
        g = up(A, w=48)
        st = ctx.add(g, up(B), alpha, beta, tau)
        assert st == eb().OK and r.status == oracle.OK
        assert same_bits(g.to_host(), Ao)
    # B identical to A: (alpha + beta) A
    Ao = A.widened(24)
    oracle.add(Ao, Ao, 0.5, 0.25, 0.0)
    g = up(A, w=24)
    ctx.add(g, g, 0.5, 0.25, 0.0)
    assert same_bits(g.to_host(), Ao)
    for alpha, beta, tau in [(1.0, 0.5, 0.0), (-0.125, 0.75, 1e-2)]:
        Ao = A.widened(22)
        oracle.scale_add_identity(Ao, alpha, beta, tau)
        g = up(A, w=22)
        ctx.scale_add_identity(g, alpha, beta, tau)
        assert same_bits(g.to_host(), Ao)
    Ao = A.widened(22)
    oracle.add_identity(Ao, -0.5, 0.0)
    g = up(A, w=22)
    ctx.add_identity(g, -0.5, 0.0)
    assert same_bits(g.to_host(), Ao)
    # full row without a diagonal -> OVERFLOW
    F = synth.random_sparse(64, 4, 4, 4, 63, 0.0, 1.0, seed=5)
    Fo = F.copy()
    r = oracle.add_identity(Fo, 1.0, 0.0)
    st = ctx.add_identity(up(F), 1.0, 0.0)
    assert (r.status == oracle.OVERFLOW) == (st == eb().ERR_OVERFLOW)
    # trace / fnorm / gershgorin
    H = synth.cfg3(n=4096)
    assert ctx.trace(up(H)) == oracle.trace(H)
    assert ctx.gershgorin(up(H)) == oracle.gershgorin(H)
    f_o = oracle.fnorm_diff(A, B)
    f_g = ctx.fnorm_diff(up(A), up(B))
    assert abs(f_g - f_o) <= 1e-12 * f_o


@pytest.mark.parametrize("seed", range(10))
def test_x2_fuzz_bitwise(ctx, seed):
    """Seeded random (non-symmetric) X for the x2 entry point: output, tr X and tr X^2 bitwise
    (both paths: B rows up to 300 entries, half-bandwidths up to beyond any ring)."""
    rng = np.random.default_rng(9100 + seed)
    n = int(rng.choice([1, 2, 63, 300, 1025, 4000, 9000]))
    w = int(rng.choice([2, 8, 32, 128, 256, 300]))
    kmax = int(rng.integers(1, w + 1))
    kmin = int(rng.integers(0, kmax + 1))
    band = int(rng.choice([2, 20, 700, 9000]))
    X = synth.random_sparse(n, w, kmin, kmax, band, float(rng.choice([0.0, 0.3])), 1.0, seed=seed + 40)
    tau = float(rng.choice([0.0, 1e-5, 1e-1]))
    lit = oracle.x2(X, synth.Ell.empty(n, w), tau)
    wo = max(2, ((lit.required_width + 31) // 32) * 32)
    Y = synth.Ell.empty(n, wo)
    r = oracle.x2(X, Y, tau)
    assert r.status == oracle.OK
    y = eb().Mat.empty(n, wo)
    st, tx, tx2 = ctx.multiply_x2(up(X), y, tau)
    assert st == eb().OK
    assert same_bits_scalar(tx, r.trace_x) and same_bits_scalar(tx2, r.trace_x2)
    assert same_bits(y.to_host(), Y)


@pytest.mark.parametrize("seed", range(8))
def test_glue_ops_fuzz_bitwise(ctx, seed):
    """Seeded random shapes for the SP2 glue (§8a-a6, §8c-c6..c8): add, add_identity,
    scale_add_identity (incl. OVERFLOW reports), trace, Gershgorin; bitwise vs the oracle."""
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.choice([1, 5, 33, 256, 257, 1500, 4099]))
    w = int(rng.choice([2, 4, 16, 40, 64, 130]))
    kmax = int(rng.integers(0, w + 1))
    kmin = int(rng.integers(0, kmax + 1))
    band = int(rng.choice([1, 3, 60, 5000]))
    pe = float(rng.choice([0.0, 0.2]))
    A = synth.random_sparse(n, w, kmin, kmax, band, pe, float(rng.choice([1e-3, 1.0, 50.0])), seed=seed * 3 + 1)
    B = synth.random_sparse(n, w, kmin, kmax, band, pe, 1.0, seed=seed * 3 + 2)
    alpha, beta = float(rng.normal()), float(rng.normal())
    tau = float(rng.choice([0.0, 1e-6, 1e-2, 0.5]))
    wo = int(rng.choice([w, w + 2, 2 * w]))
    for op in ("add", "add_identity", "scale_add_identity"):
        Ao = A.widened(wo)
        if op == "add":
            r = oracle.add(Ao, B, alpha, beta, tau)
            g = up(A, w=wo)
            st = ctx.add(g, up(B), alpha, beta, tau)
        elif op == "add_identity":
            r = oracle.add_identity(Ao, beta, tau)
            g = up(A, w=wo)
            st = ctx.add_identity(g, beta, tau)
        else:
            r = oracle.scale_add_identity(Ao, alpha, beta, tau)
            g = up(A, w=wo)
            st = ctx.scale_add_identity(g, alpha, beta, tau)
        if r.status == oracle.OK:
            assert st == eb().OK, op
            assert same_bits(g.to_host(), Ao), op
        else:
            assert st == eb().ERR_OVERFLOW, op
            assert ctx.overflow_info() == (r.overflow_rows, r.required_width), op
    assert same_bits_scalar(ctx.trace(up(A)), oracle.trace(A))
    lo, hi = ctx.gershgorin(up(A))
    olo, ohi = oracle.gershgorin(A)
    assert same_bits_scalar(lo, olo) and same_bits_scalar(hi, ohi)


@pytest.mark.parametrize("case", load_golden("hand_vectors.json") + load_golden("spec_examples.json"),
                         ids=lambda c: c["id"])
def test_golden_vectors_on_gpu(ctx, case):
    """The printed / hand-derived vectors, run through the CUDA path (same expectations as the oracle)."""
    op, exp = case["op"], case["expect"]
    if op == "x2":
        X = ell_from_entries(case["X"])
        st, G, tx, tx2 = gpu_x2(ctx, X, max(2, X.n + (X.n & 1)), case["tau"])
        assert entries_of(G) == [tuple(e) for e in exp["X2"]["entries"]]
        assert (tx, tx2) == (exp["trace_x"], exp["trace_x2"])
    elif op == "multiply":
        A, B = ell_from_entries(case["A"]), ell_from_entries(case["B"])
        C = ell_from_entries(case["C"], w=max(2, A.n + (A.n & 1)))
        g = up(C)
        ctx.multiply(up(A), up(B), g, case["alpha"], case["beta"], case["tau"])
        assert entries_of(g.to_host()) == [tuple(e) for e in exp["C"]["entries"]]
    elif op == "trace":
        assert ctx.trace(up(ell_from_entries(case["A"]))) == exp["trace"]
    elif op == "fnorm_diff":
        assert ctx.fnorm_diff(up(ell_from_entries(case["A"])), up(ell_from_entries(case["B"]))) == exp["fnorm"]
    elif op == "gershgorin":
        assert ctx.gershgorin(up(ell_from_entries(case["H"]))) == (exp["emin"], exp["emax"])
    elif op == "scale_add_identity":
        g = up(ell_from_entries(case["A"], w=4))
        ctx.scale_add_identity(g, case["alpha"], case["beta"], case["tau"])
        assert entries_of(g.to_host()) == [tuple(e) for e in exp["A"]["entries"]]
    elif op == "sp2":
        H = ell_from_entries(case["H"], w=4)
        d = eb().Mat.empty(H.n, 4)
        r = ctx.sp2_run(up(H), case["nocc"], case["tol"], d, threshold=case["tau"],
                        max_iter=case.get("max_iter", 100), min_iter=case.get("min_iter", 20))
        D = d.to_host()
        if "D_dense_within_1e-6" in exp:
            assert np.max(np.abs(D.to_dense() - np.array(exp["D_dense_within_1e-6"]))) <= 1e-6
            return
        assert r.iterations == exp["iterations"]
        assert [it["branch"] for it in r.iters] == exp["branches"]
        if "e" in exp:
            assert [it["e"] for it in r.iters] == exp["e"]
            assert (r.emin, r.emax) == (exp["emin"], exp["emax"]) and r.stop == exp["stop"]
        if "trD" in exp:
            assert r.trD == exp["trD"]
        assert entries_of(D) == [tuple(e) for e in exp["D"]["entries"]]


# ---------------------------------------------------------------------------- SP2

def _compare_sp2(g, o):
    assert g.iterations == o.iterations
    assert g.stop == o.stop
    assert (g.emin, g.emax) == (o.emin, o.emax)
    assert g.regrows == o.regrows and g.final_width == o.final_width
    for a, b in zip(g.iters, o.iters):
        assert a["branch"] == b["branch"]
        assert all(same_bits_scalar(a[k], b[k]) for k in ("trX", "trS", "e"))  # bits: NaN-safe
        assert a["width"] == b["width"] and a["required"] == b["required"]
        assert a["products"] == b["products"]  # scalar-product count of the X^2
        assert same_bits_scalar(a["frob2"], b["frob2"])  # T2 of the trace-closest rule (0 otherwise)
        if math.isfinite(b["fnorm"]):
            assert abs(a["fnorm"] - b["fnorm"]) <= 1e-10 * max(b["fnorm"], 1e-300)
        else:  # a diverged run (tau too large for the spectrum): non-finite on both sides (the
            # diagnostic's order is not pinned, c11, so inf - inf may give NaN on one side only)
            assert not math.isfinite(a["fnorm"])
    assert same_bits_scalar(g.trD, o.trD)


@pytest.mark.parametrize("n,seed,tau", [(128, 2, 0.0), (512, 5, 0.0), (1024, 6, 1e-6)])
def test_sp2_iterate_parity(ctx, n, seed, tau):
    H = synth.sym_banded(n, 32, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, seed)
    o = oracle.sp2(H, n // 2, 1e-10, oracle.SP2Opts(threshold=tau, max_iter=100), d_width=n)
    d = eb().Mat.empty(n, n)
    g = ctx.sp2_run(up(H), n // 2, 1e-10, d, threshold=tau, max_iter=100)
    _compare_sp2(g, o)
    assert same_bits(d.to_host(), o.D)
    if tau == 0.0:
        D = o.D.to_dense()
        assert np.linalg.norm(D @ D - D) < 1e-8 and abs(np.trace(D) - n // 2) < 1e-8


@pytest.mark.parametrize("n,seed,tau,shrink", [(48, 0, 0.0, 0.05), (640, 7, 0.0, 0.05), (1024, 8, 1e-6, 0.03),
                                               (512, 3, 1e-7, 0.0)])
def test_sp2_trace_closest_rule_parity(ctx, n, seed, tau, shrink):
    """§8f-f4 (i): the trace-closest branch rule (T2 from X_n, R19), bounds `shrink` inside the
    spectrum so the rule departs from the trace-sign rule; bitwise against the oracle."""
    if n == 48:
        h = np.sort(np.random.default_rng(14).uniform(-2, 2, n))
        H = synth.from_dense(np.diag(h), w=2)
        nocc = 5
    else:
        H = synth.sym_banded(n, 32, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, seed)
        nocc = n // 2 - 5
    lo, hi = oracle.gershgorin(H)
    if shrink:
        lo, hi = lo + shrink * (hi - lo), hi - shrink * (hi - lo)
    o = oracle.sp2(H, nocc, 1e-10, oracle.SP2Opts(threshold=tau, max_iter=100, emin=lo, emax=hi, branch_rule=1),
                   d_width=n)
    d = eb().Mat.empty(n, n)
    g = ctx.sp2_run(up(H), nocc, 1e-10, d, threshold=tau, max_iter=100, bounds=(lo, hi),
                    branch_rule=eb().SP2_RULE_TRACE_CLOSEST)
    _compare_sp2(g, o)
    assert all(it["frob2"] != 0.0 for it in g.iters)
    assert same_bits(d.to_host(), o.D)


SP2_FUZZ = [
    # (n, m, partners, band, seed, tau, rule, width0, nocc_frac)
    (64, 16, 3, 8, 11, 0.0, 0, 0, 0.5),
    (200, 32, 6, 40, 12, 1e-6, 1, 8, 0.3),
    (513, 32, 8, 64, 13, 1e-4, 0, 16, 0.7),
    (600, 64, 10, 100, 14, 1e-4, 1, 0, 0.5),
    (401, 32, 5, 300, 15, 1e-3, 0, 32, 0.25),
    (640, 32, 6, 16, 16, 1e-6, 1, 8, 0.5),
]


@pytest.mark.parametrize("case", SP2_FUZZ, ids=lambda c: f"n{c[0]}tau{c[5]}r{c[6]}")
def test_sp2_fuzz_bitwise(ellpack_lib, case):
    """Seeded SP2 shapes: ragged n, both branch rules, thresholds 0 .. 1e-3, GROW from a narrow
    start (ELLPACK_OPT_SP2_WIDTH0), nocc away from N/2; every iterate record and D bitwise."""
    n, m, partners, band, seed, tau, rule, w0, frac = case
    H = synth.sym_banded(n, m, partners, band, 1, -1.0, 1.0, 0, band / 4.0, 0.0, seed)
    nocc = int(frac * n)
    o = oracle.sp2(H, nocc, 1e-9, oracle.SP2Opts(threshold=tau, max_iter=100, branch_rule=rule,
                                                 initial_width=w0), d_width=n + (n & 1))
    ctx = ellpack_lib.Context(0)
    if w0:
        ctx.set_option(ellpack_lib.OPT_SP2_WIDTH0, w0)
    d = ellpack_lib.Mat.empty(n, n + (n & 1))
    g = ctx.sp2_run(up(H), nocc, 1e-9, d, threshold=tau, max_iter=100, branch_rule=rule)
    assert g.status == o.status  # OK / NOCONV share their codes with the oracle
    _compare_sp2(g, o)
    assert same_bits(d.to_host(), o.D)
    ctx.close()


def test_sp2_grow_fault_injection(ellpack_lib):
    """Start iterates at width 8 (ELLPACK_OPT_SP2_WIDTH0): GROW must reproduce the oracle's widths."""
    ctx = ellpack_lib.Context(0)
    ctx.set_option(ellpack_lib.OPT_SP2_WIDTH0, 8)
    H = synth.sym_banded(768, 32, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, 9)
    o = oracle.sp2(H, 384, 1e-9, oracle.SP2Opts(threshold=1e-7, initial_width=8), d_width=768)
    d = ellpack_lib.Mat.empty(768, 768)
    g = ctx.sp2_run(up(H), 384, 1e-9, d, threshold=1e-7)
    _compare_sp2(g, o)
    assert g.regrows >= 2
    assert same_bits(d.to_host(), o.D)
    ctx.close()


def test_sp2_cfg3_literal_overflow_and_grow_window(ctx):
    """cfg3 (N=12288, M=256): literal FAIL overflows at iteration 0 exactly like the oracle;
    GROW over a 3-iteration window matches iterate by iterate (reading R10)."""
    H = synth.cfg3()
    cf = synth.CFG3
    of = oracle.sp2(H, cf["nocc"], cf["tol"], oracle.SP2Opts(threshold=cf["threshold"], on_overflow=0),
                    d_width=256)
    d = eb().Mat.empty(H.n, 256)
    gf = ctx.sp2_run(up(H), cf["nocc"], cf["tol"], d, threshold=cf["threshold"], on_overflow=eb().SP2_FAIL)
    assert of.status == oracle.OVERFLOW and gf.status == eb().ERR_OVERFLOW
    assert (gf.fail_iter, gf.required_width, gf.overflow_rows) == (of.fail_iter, of.required_width, of.overflow_rows)
    og = oracle.sp2(H, cf["nocc"], cf["tol"], oracle.SP2Opts(threshold=cf["threshold"], max_iter=3), d_width=4096)
    d = eb().Mat.empty(H.n, 4096)
    gg = ctx.sp2_run(up(H), cf["nocc"], cf["tol"], d, threshold=cf["threshold"], max_iter=3)
    _compare_sp2(gg, og)
    assert same_bits(d.to_host(), og.D)


@pytest.mark.parametrize("n,seed,tau,width0", [(1024, 6, 1e-6, 0), (768, 9, 1e-7, 8), (1500, 21, 1e-5, 0)])
def test_sp2_symmetric_step_vs_whole_rows(ellpack_lib, n, seed, tau, width0):
    """§8f-f4 (ii): with H bitwise symmetric the general-path steps compute only the upper
    triangle and mirror it (extra launches: the symmetry check, reach, assembly). Both modes,
    and an H with one asymmetric bit (whole rows), are bitwise the oracle."""
    E = ellpack_lib
    H = synth.sym_banded(n, 32, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, seed)
    o = oracle.sp2(H, n // 2, 1e-10, oracle.SP2Opts(threshold=tau, max_iter=100, initial_width=width0),
                   d_width=n)
    launches = {}
    for sym in (1, 0):
        ctx = E.Context(0)
        ctx.set_option(E.OPT_SP2_DEVICE_LOOP, 1)  # the symmetric step belongs to the host loop
        ctx.set_option(E.OPT_DENSE, 1)  # the sparse kernels' symmetric route (the dense GEMM has its own)
        ctx.set_option(E.OPT_SP2_SYMMETRIC, sym)
        if width0:
            ctx.set_option(E.OPT_SP2_WIDTH0, width0)
        d = E.Mat.empty(n, n)
        k0 = ctx.kernel_launches()
        g = ctx.sp2_run(up(H), n // 2, 1e-10, d, threshold=tau, max_iter=100)
        launches[sym] = ctx.kernel_launches() - k0
        _compare_sp2(g, o)
        assert same_bits(d.to_host(), o.D)
        ctx.close()
    assert launches[1] >= launches[0] + 1  # the symmetry check ran
    if o.final_width > 256:  # wide iterates: general-path steps took the symmetric route
        assert launches[1] > launches[0] + 2
    # one flipped bit in one off-diagonal entry: not symmetric -> whole rows, still bitwise
    Ha = H.copy()
    i = int(np.argmax(Ha.nnz))
    q = int(np.flatnonzero(Ha.col[i, :Ha.nnz[i]] != i)[0])
    Ha.val[i, q] = np.nextafter(Ha.val[i, q], np.inf)
    oa = oracle.sp2(Ha, n // 2, 1e-10, oracle.SP2Opts(threshold=tau, max_iter=100), d_width=n)
    ctx = E.Context(0)
    d = E.Mat.empty(n, n)
    ga = ctx.sp2_run(up(Ha), n // 2, 1e-10, d, threshold=tau, max_iter=100)
    _compare_sp2(ga, oa)
    assert same_bits(d.to_host(), oa.D)
    ctx.close()


# ------------------------------------------------------- multi-rank emulation (1 GPU)

@pytest.mark.parametrize("nranks", [2, 4])
def test_row_block_partition_is_bitwise_invariant(ellpack_lib, nranks):
    """Each 'rank' computes only its 256-aligned row block (ellpack_ctx_set_rows); the union of
    the blocks equals the single-rank product bit for bit (§8c-c12, row independence)."""
    X = synth.cfg5(32768, 64)
    full = ellpack_lib.Context(0)
    y1 = ellpack_lib.Mat.empty(X.n, 1024)
    assert full.multiply_x2(up(X), y1, 1e-5)[0] == ellpack_lib.OK
    yp = ellpack_lib.Mat.empty(X.n, 1024)
    x = up(X)
    for (r0, r1) in ellpack_lib.row_partition(X.n, nranks):
        c = ellpack_lib.Context(0)
        c.set_rows(r0, r1)
        c.multiply_x2(x, yp, 1e-5)
        c.close()
    assert same_bits(yp.to_host(), y1.to_host())
    full.close()


def _corrupt(X, kind):
    Y = X.copy()
    i = int(np.argmax(Y.nnz))  # a row with >= 2 entries
    if kind == "unsorted":
        Y.col[i, 0], Y.col[i, 1] = Y.col[i, 1], Y.col[i, 0]
    elif kind == "duplicate":
        Y.col[i, 1] = Y.col[i, 0]
    elif kind == "col_range":
        Y.col[i, Y.nnz[i] - 1] = Y.n
    elif kind == "negative_col":
        Y.col[i, 0] = -1
    elif kind == "nnz_range":
        Y.nnz[i] = Y.w + 2
    elif kind == "nan":
        Y.val[i, 0] = float("nan")
    return Y


@pytest.mark.parametrize("kind", ["unsorted", "duplicate", "col_range", "negative_col", "nnz_range", "nan"])
def test_validate_option_rejects_non_canonical_inputs(ellpack_lib, kind):
    """ELLPACK_OPT_VALIDATE (§8b: inputs must be canonical D1, checked on request): every entry point
    returns ARG for a non-canonical operand and still computes bitwise for canonical ones."""
    E = ellpack_lib
    ctx = E.Context(0)
    ctx.set_option(E.OPT_VALIDATE, 1)
    X = synth.cfg1()
    Y = synth.Ell.empty(X.n, 256)
    r = oracle.x2(X, Y, 1e-5)
    y = E.Mat.empty(X.n, 256)
    st, tx, tx2 = ctx.multiply_x2(up(X), y, 1e-5)
    assert st == E.OK and (tx, tx2) == (r.trace_x, r.trace_x2) and same_bits(y.to_host(), Y)
    bad = up(_corrupt(X, kind))
    good = up(X)
    calls = [
        lambda: ctx.multiply_x2(bad, E.Mat.empty(X.n, 256), 1e-5, ok=()),
        lambda: ctx.multiply(bad, good, E.Mat.empty(X.n, 256), 1.0, 0.0, 1e-5, ok=()),
        lambda: ctx.multiply(good, bad, E.Mat.empty(X.n, 256), 1.0, 0.0, 1e-5, ok=()),
        lambda: ctx.add(up(X, w=64), bad, 1.0, 1.0, 0.0, ok=()),
        lambda: ctx.add_identity(bad, 1.0, 0.0, ok=()),
        lambda: ctx.trace(bad),
        lambda: ctx.fnorm_diff(good, bad),
        lambda: ctx.gershgorin(bad),
        lambda: ctx.sp2_run(bad, X.n // 2, 1e-8, E.Mat.empty(X.n, X.n), ok=()),
    ]
    for k, call in enumerate(calls):
        with pytest.raises(E.EllpackError) as ei:
            call()
        assert ei.value.status == E.ERR_ARG, (kind, k)
    ctx.close()


def test_nccl_single_rank_communicator_paths(ellpack_lib):
    """The NCCL code paths on one GPU (a 1-rank communicator): status all-reduce, trace-partial
    all-gather, halo exchange (col-range kernel + range all-gather + an empty plan), SP2 with
    halo exchanges and the final all-gather -- all bitwise equal to the oracle."""
    import torch  # noqa: F401  (loads torch's libnccl.so.2 for the library's dlopen)
    E = ellpack_lib
    ctx = E.Context(0)
    uid = E.Context.nccl_unique_id()
    n = 1024
    ctx.attach_nccl(1, 0, uid, 0, n)
    X = synth.cfg5(n, 32)
    Y = synth.Ell.empty(n, 512)
    r = oracle.x2(X, Y, 1e-5)
    x = up(X)
    ctx.halo_rows(x)
    assert same_bits(x.to_host(), X)
    y = E.Mat.empty(n, 512)
    st, tx, tx2 = ctx.multiply_x2(x, y, 1e-5)
    assert st == E.OK and (tx, tx2) == (r.trace_x, r.trace_x2) and same_bits(y.to_host(), Y)
    H = synth.sym_banded(n, 32, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, 3)
    o = oracle.sp2(H, n // 2, 1e-10, oracle.SP2Opts(threshold=1e-7, max_iter=100), d_width=n)
    d = E.Mat.empty(n, n)
    g = ctx.sp2_run(up(H), n // 2, 1e-10, d, threshold=1e-7, max_iter=100)
    _compare_sp2(g, o)
    assert same_bits(d.to_host(), o.D)
    ctx.close()


def test_halo_rows_without_communicator_is_a_no_op(ctx):
    X = synth.cfg5(4096, 32)
    x = up(X)
    ctx.halo_rows(x)
    assert same_bits(x.to_host(), X)


def test_host_buffer_e2e_path(ctx):
    X = synth.cfg1()
    r, Y = ora_x2(X, 256, 1e-5)
    Y2 = Ell.empty(X.n, 256)
    st, tx, tx2 = ctx.multiply_x2_host(X, Y2, 1e-5)
    assert st == eb().OK and same_bits(Y2, Y) and (tx, tx2) == (r.trace_x, r.trace_x2)


def test_kernel_launch_counter(ctx):
    before = ctx.kernel_launches()
    X = synth.cfg1()
    gpu_x2(ctx, X, 256, 1e-5)
    # N = 512 <= 1024: no probe; the small-matrix kernel (rows, status and the canonical sums in
    # one launch)
    assert ctx.kernel_launches() - before == 1
    assert ctx.last_launch()["path"] == "small"
    ctx.set_option(eb().OPT_SMALL_KERNEL, 1)  # the general path: one window covering every column
    before = ctx.kernel_launches()          # (no breakpoints), the row kernel + the one-CTA sums
    gpu_x2(ctx, X, 256, 1e-5)
    assert ctx.kernel_launches() - before == 2
    assert ctx.last_launch()["path"] == "general"
