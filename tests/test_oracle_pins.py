"""Pins of the CPU oracle against things other than itself (CPU only, `-m "not gpu"`).

Each test names the SURVEY.md §8(c) pin it implements (P1..P13), the printed
examples (SPEC) or the hand vectors in tests/golden/.
A plausible oracle mistake -- a dropped term, a wrong sign or index, a
transposed operand, a wrong summation order, a two-stage drop, a wrong tie rule
-- fails at least one of them.
"""
import decimal
import math
from decimal import Decimal as D_

import numpy as np
import pytest

import oracle
import synth
from synth import Ell, from_dense
from tests.helpers import (brute_multiply, ell_from_entries, entries_of, load_golden,
                           random_dense_sparse, same_bits)


# ------------------------------------------------------------------ golden fixtures

def _run_case(case):
    op = case["op"]
    exp = case["expect"]
    if op == "x2":
        X = ell_from_entries(case["X"])
        X2 = Ell.empty(X.n, max(2, X.n + (X.n & 1)))
        r = oracle.x2(X, X2, case["tau"])
        assert r.status == oracle.OK
        assert entries_of(X2) == [tuple(e) for e in exp["X2"]["entries"]]
        assert r.trace_x == exp["trace_x"] and r.trace_x2 == exp["trace_x2"]
    elif op == "multiply":
        A, B = ell_from_entries(case["A"]), ell_from_entries(case["B"])
        C = ell_from_entries(case["C"], w=max(2, A.n + (A.n & 1)))
        r = oracle.multiply(A, B, C, case["alpha"], case["beta"], case["tau"])
        assert r.status == oracle.OK
        assert entries_of(C) == [tuple(e) for e in exp["C"]["entries"]]
    elif op == "trace":
        assert oracle.trace(ell_from_entries(case["A"])) == exp["trace"]
    elif op == "fnorm_diff":
        assert oracle.fnorm_diff(ell_from_entries(case["A"]), ell_from_entries(case["B"])) == exp["fnorm"]
    elif op == "gershgorin":
        assert oracle.gershgorin(ell_from_entries(case["H"])) == (exp["emin"], exp["emax"])
    elif op == "scale_add_identity":
        A = ell_from_entries(case["A"], w=4)
        r = oracle.scale_add_identity(A, case["alpha"], case["beta"], case["tau"])
        assert r.status == oracle.OK
        assert entries_of(A) == [tuple(e) for e in exp["A"]["entries"]]
    elif op == "sp2":
        H = ell_from_entries(case["H"], w=4)
        opts = oracle.SP2Opts(threshold=case["tau"], max_iter=case.get("max_iter", 100),
                              min_iter=case.get("min_iter", 20))
        r = oracle.sp2(H, case["nocc"], case["tol"], opts)
        if "D_dense_within_1e-6" in exp:
            assert np.max(np.abs(r.D.to_dense() - np.array(exp["D_dense_within_1e-6"]))) <= 1e-6
            return
        assert r.iterations == exp["iterations"]
        assert [it["branch"] for it in r.iters] == exp["branches"]
        if "e" in exp:
            assert [it["e"] for it in r.iters] == exp["e"]
            assert (r.emin, r.emax) == (exp["emin"], exp["emax"])
            assert r.stop == exp["stop"]
        if "trD" in exp:
            assert r.trD == exp["trD"]
        assert entries_of(r.D) == [tuple(e) for e in exp["D"]["entries"]]
    else:
        raise AssertionError(op)


@pytest.mark.parametrize("case", load_golden("spec_examples.json"), ids=lambda c: c["id"])
def test_spec_printed_examples(case):
    _run_case(case)


@pytest.mark.parametrize("case", load_golden("hand_vectors.json"), ids=lambda c: c["id"])
def test_hand_vectors(case):
    _run_case(case)


# ------------------------------------------------------- P1: exact brute force, bitwise

@pytest.mark.parametrize("seed", range(40))
def test_p1_bruteforce_exact_fma_bitwise(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 20))
    A = random_dense_sparse(rng, n, rng.uniform(0.1, 0.7))
    B = random_dense_sparse(rng, n, rng.uniform(0.1, 0.7))
    Co = random_dense_sparse(rng, n, rng.uniform(0.0, 0.5))
    alpha = [1.0, 0.5, -1.25, 0.0, 3.0][seed % 5]
    beta = [0.0, 0.5, -2.0, 1.0][seed % 4]
    tau = [0.0, 1e-3, 0.3][seed % 3]
    want = brute_multiply(A, B, Co, alpha, beta, tau)
    Ae, Be, Ce = from_dense(A), from_dense(B), from_dense(Co, w=n + (n & 1) or 2)
    r = oracle.multiply(Ae, Be, Ce, alpha, beta, tau)
    assert r.status == oracle.OK
    got = Ce.to_dense()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert np.array_equal(Ce.nnz, (want != 0).sum(axis=1).astype(np.int32))


# -------------------------------------------------------------- P2: numpy dense GEMM

def test_p2_numpy_gemm_200_instances():
    rng = np.random.default_rng(7)
    for it in range(200):
        n = int(rng.integers(1, 257))
        A = random_dense_sparse(rng, n, rng.uniform(0.005, 0.2))
        B = random_dense_sparse(rng, n, rng.uniform(0.005, 0.2))
        C = Ell.empty(n, n + (n & 1))
        r = oracle.multiply(from_dense(A), from_dense(B), C, 1.0, 0.0, 0.0)
        assert r.status == oracle.OK
        ref = A @ B
        nr = np.linalg.norm(ref)
        err = np.linalg.norm(C.to_dense() - ref)
        assert err <= 1e-12 * max(nr, 1e-300) or (nr == 0 and err == 0), (it, n, err, nr)


# ------------------------------------------------------------------ P3: closed forms

@pytest.mark.parametrize("n", [1, 3, 255, 256, 257, 1000])
def test_p3_closed_forms(n):
    rng = np.random.default_rng(n)
    I = from_dense(np.eye(n), w=2)
    A = synth.random_sparse(n, 8, 0, 6, band=5, seed=n)
    C = Ell.empty(n, 8)
    assert oracle.multiply(I, A, C, 1.0, 0.0, 0.0).status == oracle.OK
    assert same_bits(C, A)  # I.A = A
    Z = Ell.empty(n, 2)
    C2 = Ell.empty(n, 8)
    assert oracle.multiply(A, Z, C2, 1.0, 0.0, 0.0).status == oracle.OK
    assert C2.nnz.sum() == 0  # A.0 = 0
    X2 = Ell.empty(n, 2)
    r = oracle.x2(I, X2, 0.0)
    assert same_bits(X2, I) and r.trace_x == n and r.trace_x2 == n  # I^2 = I, traces (N, N)
    H = from_dense(np.eye(n) * 0.5, w=2)
    r = oracle.x2(H, X2, 0.0)
    assert np.array_equal(X2.to_dense(), np.eye(n) * 0.25)
    assert r.trace_x == n / 2 and r.trace_x2 == n / 4  # (S:L76 generalised)
    del rng


# ----------------------------------------- P4 / P5: symmetry and tr(X^2) = ||X||_F^2

@pytest.mark.parametrize("seed", range(5))
def test_p4_x2_of_symmetric_is_bitwise_symmetric(seed):
    X = synth.sym_banded(700, 24, 8, 40, 2, 0, 0, 0, 12.0, 0.0, seed)
    X2 = Ell.empty(700, 200)
    r = oracle.x2(X, X2, 1e-5)
    assert r.status == oracle.OK
    D = X2.to_dense()
    assert np.array_equal(D.view(np.uint64), D.T.view(np.uint64))


def test_p5_trace_x2_equals_frobenius_squared():
    X = synth.sym_banded(1500, 32, 10, 60, 2, 0, 0, 0, 20.0, 0.0, 11)
    X2 = Ell.empty(1500, 300)
    r = oracle.x2(X, X2, 0.0)
    fro2 = math.fsum(float(v) ** 2 for _, v in ((c, v) for cc, vv in X.rows() for c, v in zip(cc, vv)))
    assert abs(r.trace_x2 - fro2) <= 1e-12 * fro2
    assert r.trace_x == math.fsum(X.to_dense().diagonal()) or abs(r.trace_x - math.fsum(X.to_dense().diagonal())) <= 1e-12


# ------------------------------------------------ P6 / P7: monotone in tau, band bound

def test_p6_threshold_monotone_and_p7_band_bound():
    X = synth.sym_banded(800, 24, 8, 30, 2, 0, 0, 0, 10.0, 0.0, 3)
    prev = None
    for tau in [0.0, 1e-6, 1e-4, 1e-2, 1e-1, 1.0]:
        X2 = Ell.empty(800, 200)
        assert oracle.x2(X, X2, tau).status == oracle.OK
        pat = {(i, j) for i, j, _ in entries_of(X2)}
        if prev is not None:
            assert pat <= prev
        prev = pat
        bw = max((abs(i - j) for i, j in pat), default=0)
        assert bw <= 60  # bw(X) <= 30
    # an unbounded product would violate it: check the bound is attained-ish at tau = 0
    X2 = Ell.empty(800, 200)
    oracle.x2(X, X2, 0.0)
    assert max(abs(i - j) for i, j, _ in entries_of(X2)) > 30


# --------------------------------------------------------------------- P9: add family

def test_p9_add_pins():
    A = synth.random_sparse(300, 16, 0, 12, band=40, seed=5)
    B = synth.random_sparse(300, 16, 0, 12, band=40, seed=6)
    A1 = A.widened(32)
    assert oracle.add(A1, B, 1.0, 0.0, 0.0).status == oracle.OK  # 1.A + 0.B = A
    assert same_bits(A1, A)
    A2 = A.widened(32)
    assert oracle.add(A2, A2, 1.0, -1.0, 0.0).status == oracle.OK  # A - A = 0
    assert A2.nnz.sum() == 0
    A3 = A.widened(32)
    assert oracle.add(A3, B, 0.5, -2.0, 0.0).status == oracle.OK
    ref = 0.5 * A.to_dense() - 2.0 * B.to_dense()
    assert np.max(np.abs(A3.to_dense() - ref)) <= 1e-15 * np.max(np.abs(ref))
    # add_identity inserts beta on a missing diagonal, adds it to a present one (one rounding)
    E = from_dense(np.array([[0.0, 2.0], [0.0, 0.25]]), w=4)
    assert oracle.add_identity(E, 0.5, 0.0).status == oracle.OK
    assert entries_of(E) == [(0, 0, 0.5), (0, 1, 2.0), (1, 1, 0.75)]
    # scale_add_identity: off-diagonal alpha*a, diagonal fma(alpha, a, beta); drop every entry
    F = from_dense(np.array([[1.0, 0.5], [0.5, 3.0]]), w=4)
    assert oracle.scale_add_identity(F, -0.25, 0.75, 0.2).status == oracle.OK
    assert entries_of(F) == [(0, 0, 0.5)]  # (1,1) = 0 dropped, off-diag |-1/8| <= 0.2 dropped


def test_overflow_reporting_matches_dense_counts():
    X = synth.cfg1()
    want = X.to_dense() @ X.to_dense()
    kept = (np.abs(want) > 1e-5).sum(axis=1)
    X2 = Ell.empty(X.n, 32)
    r = oracle.x2(X, X2, 1e-5)
    assert r.status == oracle.OVERFLOW
    # the exact kept count may differ from the dense numpy product only at |c| ~ tau; check both
    assert abs(r.required_width - int(kept.max())) <= 1
    assert abs(r.overflow_rows - int((kept > 32).sum())) <= 1
    X2 = Ell.empty(X.n, 256)
    r2 = oracle.x2(X, X2, 1e-5)
    assert r2.status == oracle.OK and int(X2.nnz.max()) == r.required_width


# ------------------------------------------------------------------- P10: Gershgorin

def test_p10_gershgorin_contains_eigenvalues():
    rng = np.random.default_rng(10)
    for t in range(100):
        n = int(rng.integers(1, 129))
        d = random_dense_sparse(rng, n, rng.uniform(0.02, 0.3), sym=True)
        lo, hi = oracle.gershgorin(from_dense(d, w=max(2, n + (n & 1))))
        ev = np.linalg.eigvalsh(d) if n else np.array([])
        assert lo <= ev.min() + 1e-12 and ev.max() - 1e-12 <= hi
    # diagonal: bounds are the exact extreme eigenvalues
    H = from_dense(np.diag([-3.5, 2.0, 0.25]), w=4)
    assert oracle.gershgorin(H) == (-3.5, 2.0)


# ------------------------------------------------------------- canonical sum (c7) pin

def test_c7_canonical_block_order():
    # Block 0 = [2^53, 1 x 255] -> 2^53 (each +1 is a round-to-even tie); block 1 = 256 ones -> 256.
    # Canonical total = 2^53 + 256. A left-to-right sum gives 2^53; 128-row blocks give 2^53 + 384.
    d = np.ones(512)
    d[0] = 2.0 ** 53
    assert oracle.canonical_sum(d) == 2.0 ** 53 + 256
    X = from_dense(np.diag(d), w=2)
    assert oracle.trace(X) == 2.0 ** 53 + 256
    # integers: exact
    v = np.arange(1, 5001, dtype=np.float64)
    assert oracle.canonical_sum(v) == 5000 * 5001 / 2


def test_fnorm_diff_vs_numpy():
    rng = np.random.default_rng(4)
    for _ in range(30):
        n = int(rng.integers(1, 120))
        a = random_dense_sparse(rng, n, 0.2)
        b = random_dense_sparse(rng, n, 0.2)
        got = oracle.fnorm_diff(from_dense(a, w=n + (n & 1) or 2), from_dense(b, w=n + (n & 1) or 2))
        ref = np.linalg.norm(a - b)
        assert abs(got - ref) <= 1e-12 * max(ref, 1e-300)


# --------------------------------------------------------------------- SP2 pins

def _scalar_sp2_hp(x0, branches):
    """The scalar SP2 maps in 60-digit decimal arithmetic (independent of binary64)."""
    x = list(x0)
    for b in branches:
        x = [xi * xi if b == "SQUARE" else 2 * xi - xi * xi for xi in x]
    return x


def test_p11_diagonal_hamiltonian_scalar_recursion():
    rng = np.random.default_rng(11)
    n = 40
    h = np.sort(rng.uniform(-2, 2, n))
    H = from_dense(np.diag(h), w=2)
    nocc = 17
    r = oracle.sp2(H, nocc, 1e-10, oracle.SP2Opts(max_iter=60))
    assert r.stop in ("CONVERGED", "STAGNATED")
    lo, hi = h.min(), h.max()
    decimal.getcontext().prec = 60
    x0 = [(D_(hi) - D_(hv)) / (D_(hi) - D_(lo)) for hv in h]
    hp = _scalar_sp2_hp(x0, [it["branch"] for it in r.iters])
    got = r.D.to_dense().diagonal()
    assert max(abs(float(e) - g) for e, g in zip(hp, got)) <= 1e-10
    # the limit is the projector on the nocc lowest levels
    assert np.max(np.abs(got - (np.arange(n) < nocc))) <= 1e-6
    # branch rule: SQUARE iff tr(X_n) > nocc (R6)
    for it in r.iters:
        assert (it["branch"] == "SQUARE") == (it["trX"] > nocc)


def test_p12_dimer_closed_form():
    # 2x2 dimer blocks [[eA, t], [t, eB]] (the paper's two-level unit)
    rng = np.random.default_rng(12)
    nb = 64
    blocks = []
    d = np.zeros((2 * nb, 2 * nb))
    for b in range(nb):
        ea, eb, t = rng.uniform(-1, 0), rng.uniform(0, 1), rng.uniform(-1, -0.3)
        d[2 * b, 2 * b], d[2 * b + 1, 2 * b + 1] = ea, eb
        d[2 * b, 2 * b + 1] = d[2 * b + 1, 2 * b] = t
        blocks.append((ea, eb, t))
    H = from_dense(d, w=4)
    r = oracle.sp2(H, nb, 0.0, oracle.SP2Opts(max_iter=80, min_iter=10))
    D = r.D.to_dense()
    for b, (ea, eb, t) in enumerate(blocks):
        m, dd = (ea + eb) / 2, (ea - eb) / 2
        lam = m - math.sqrt(dd * dd + t * t)
        v = np.array([t, lam - ea])
        v /= np.linalg.norm(v)
        ref = np.outer(v, v)
        assert np.max(np.abs(D[2 * b:2 * b + 2, 2 * b:2 * b + 2] - ref)) <= 1e-12
    assert abs(np.trace(D) - nb) <= 1e-12


@pytest.mark.parametrize("n,seed", [(64, 1), (128, 2), (256, 3)])
def test_p13_small_random_vs_eigh_projector(n, seed):
    H = synth.sym_banded(n, n, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, seed)
    d = H.to_dense()
    ev, Q = np.linalg.eigh(d)
    nocc = n // 2
    gap = ev[nocc] - ev[nocc - 1]
    assert gap > 1e-3, "fixture must be gapped"
    Dx = Q[:, :nocc] @ Q[:, :nocc].T
    r = oracle.sp2(H, nocc, 1e-10, oracle.SP2Opts(max_iter=100))
    assert r.status == oracle.OK and r.stop in ("CONVERGED", "STAGNATED")
    D = r.D.to_dense()
    assert np.linalg.norm(D @ D - D) < 1e-8                     # idempotent
    assert abs(np.trace(D) - nocc) < 1e-8                       # occupation
    assert np.linalg.norm(D @ d - d @ D) / np.linalg.norm(d) < 1e-10  # commutes with H
    assert np.linalg.norm(D - Dx) / np.linalg.norm(Dx) < 1e-6   # the eigh projector
    # e_n = sum lambda(1-lambda) >= 0 up to rounding, and the trace identity holds
    for it in r.iters:
        assert it["e"] > -1e-12


# ------------------------------------------- SP2 trace-closest rule (§8f-f4 i, R19)

def test_p14_trace_closest_rule_diagonal_scalar_recursion():
    """Diagonal H with spectral bounds 5% inside the spectrum, so X0 has levels outside [0, 1]:
    every iterate is diagonal, T2 = sum x_i^2 = tr(X_n^2) exactly, and the rule is replayed in
    60-digit arithmetic from the scalar maps alone. Here the trace-sign rule diverges while the
    trace-closest rule recovers the projector (the point of the rule)."""
    rng = np.random.default_rng(14)
    n = 48
    h = np.sort(rng.uniform(-2, 2, n))
    H = from_dense(np.diag(h), w=2)
    nocc = 5
    lo, hi = h.min() + 0.05 * np.ptp(h), h.max() - 0.05 * np.ptp(h)
    r = oracle.sp2(H, nocc, 1e-10, oracle.SP2Opts(max_iter=80, emin=lo, emax=hi, branch_rule=1))
    assert r.stop == "CONVERGED"
    decimal.getcontext().prec = 60
    x = [(D_(hi) - D_(hv)) / (D_(hi) - D_(lo)) for hv in h]
    assert min(x) < 0 and max(x) > 1
    branches = [it["branch"] for it in r.iters]
    differs = 0
    for k, it in enumerate(r.iters):
        tr1, tr2 = sum(x), sum(xi * xi for xi in x)
        # T2 is tr(X_n^2) (binary64 rounding of the exact value)
        assert abs(it["frob2"] - float(tr2)) <= 1e-12 * max(1.0, float(tr2))
        sq, ex = abs(tr2 - nocc), abs(2 * tr1 - tr2 - nocc)
        if abs(sq - ex) > D_("1e-9"):
            assert (branches[k] == "SQUARE") == (sq < ex), k
        differs += (branches[k] == "SQUARE") != (tr1 > nocc)
        x = [xi * xi if branches[k] == "SQUARE" else 2 * xi - xi * xi for xi in x]
    assert differs >= 1
    got = r.D.to_dense().diagonal()
    assert max(abs(float(e) - g) for e, g in zip(x, got)) <= 1e-10
    assert np.max(np.abs(got - (np.arange(n) < nocc))) <= 1e-6
    r0 = oracle.sp2(H, nocc, 1e-10, oracle.SP2Opts(max_iter=80, emin=lo, emax=hi))
    assert r0.stop != "CONVERGED" or abs(r0.trD - nocc) > 1e-6


def test_p14b_rules_coincide_inside_unit_interval():
    """0 <= T2 <= T1 (levels in [0, 1], true bounds): |T2 - nocc| < |2 T1 - T2 - nocc| iff
    T1 > nocc, so both rules take the same branches and give the same bits."""
    for seed in (1, 2):
        H = synth.sym_banded(128, 128, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, seed)
        r0 = oracle.sp2(H, 61, 1e-10, oracle.SP2Opts(max_iter=100))
        r1 = oracle.sp2(H, 61, 1e-10, oracle.SP2Opts(max_iter=100, branch_rule=1))
        assert [it["branch"] for it in r0.iters] == [it["branch"] for it in r1.iters]
        assert np.array_equal(r0.D.val.view(np.uint64), r1.D.val.view(np.uint64))


@pytest.mark.parametrize("n,seed", [(64, 1), (192, 4)])
def test_p15_trace_closest_rule_random_vs_eigh_projector(n, seed):
    """Symmetric banded H: T2 (Frobenius of X_n) agrees with tr(X_n^2) taken from the product's
    diagonal (an independent computation) to rounding, each branch is the trace-closest one, and
    the limit is the eigh projector."""
    H = synth.sym_banded(n, n, 6, 12, 1, -1.0, 1.0, 0, 4.0, 0.0, seed)
    d = H.to_dense()
    ev, Q = np.linalg.eigh(d)
    nocc = n // 2 - 3
    assert ev[nocc] - ev[nocc - 1] > 1e-3, "fixture must be gapped"
    r = oracle.sp2(H, nocc, 1e-10, oracle.SP2Opts(max_iter=100, branch_rule=1))
    assert r.status == oracle.OK and r.stop in ("CONVERGED", "STAGNATED")
    for it in r.iters:
        assert abs(it["frob2"] - it["trS"]) <= 1e-12 * max(1.0, abs(it["trS"]))
        sq, ex = abs(it["trS"] - nocc), abs(2 * it["trX"] - it["trS"] - nocc)
        if abs(sq - ex) > 1e-8:
            assert (it["branch"] == "SQUARE") == (sq < ex)
    D = r.D.to_dense()
    Dx = Q[:, :nocc] @ Q[:, :nocc].T
    assert np.linalg.norm(D @ D - D) < 1e-8 and abs(np.trace(D) - nocc) < 1e-8
    assert np.linalg.norm(D - Dx) / np.linalg.norm(Dx) < 1e-6
    # default rule: frob2 stays 0 (not computed)
    r0 = oracle.sp2(H, nocc, 1e-10, oracle.SP2Opts(max_iter=100))
    assert all(it["frob2"] == 0.0 for it in r0.iters)


def test_sp2_overflow_fail_and_grow_widths():
    H = synth.cfg3(n=2048, m=64)
    opts = oracle.SP2Opts(threshold=1e-5, max_iter=3, on_overflow=0)
    r = oracle.sp2(H, 1024, 1e-8, opts, d_width=2048)
    assert r.status == oracle.OVERFLOW and r.fail_iter == 0 and r.required_width > 64
    opts.on_overflow = 1
    g = oracle.sp2(H, 1024, 1e-8, opts, d_width=2048)
    assert g.status == oracle.NOCONV and g.regrows >= 1
    assert g.iters[0]["width"] == ((r.required_width + 31) // 32) * 32
    assert g.iters[0]["required"] == r.required_width


def test_bounds_error():
    H = from_dense(np.eye(4) * 2.0, w=2)
    r = oracle.sp2(H, 2, 1e-8)
    assert r.status == oracle.BOUNDS
