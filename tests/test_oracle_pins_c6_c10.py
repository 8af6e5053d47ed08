"""Pins of the two oracle parts round 1 left unpinned (CPU only, `-m "not gpu"`).

c6 single rounding: every result entry of add / scale_add_identity is
ONE rounding of the combined value: add v = fma(alpha, a, beta*b), the X0 diagonal
v = fma(alpha, h_ii, beta). The round-1 pins used dyadic alpha/beta only, where the two-rounding
forms alpha*a + beta*b / alpha*a + beta give the same bits. Here an exact-rational brute force
(Fractions: int/int true division is correctly rounded) evaluates the definition with
non-dyadic alpha/beta and planted cancellations and is compared bitwise.

c10 (vi) stop rule ("stagnation", readings R7/R9): CONVERGED if
|e_n| <= tol; STAGNATED if n+1 >= min_iter and e_n <= stag_gate and e_n >= e_{n-2}; NOCONV if
n+1 = max_iter. For a diagonal H every iterate is diagonal and the binary64 SP2 arithmetic
reduces to scalar maps that Python floats replay exactly (x*x and 2x - s are single IEEE
operations; the X0 diagonal is an exact-rational fma). The replay gives the e sequence bit for
bit; the stop iteration the rule implies is then derived here from the rule's text and the
oracle must stop exactly there. The fixtures are chosen so that each plausible misreading
(e_{n-1} for e_{n-2}; n >= min_iter for n+1 >= min_iter; e < stag_gate for e <= stag_gate;
ungated) stops somewhere else.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from synth import Ell, from_dense
from tests.helpers import entries_of, fma_exact

# ------------------------------------------------------------------------ c6 brute force


def _brute_add(A, Am, B, Bm, alpha, beta, tau):
    """Definition c6 add over the union pattern: v = round(alpha*a + round(beta*b)), absent = 0,
    kept iff |v| > tau. Returns {row: [(j, v)]} ascending."""
    n = A.shape[0]
    out = {}
    for i in range(n):
        row = []
        for j in range(n):
            if not (Am[i, j] or Bm[i, j]):
                continue
            a = float(A[i, j]) if Am[i, j] else 0.0
            b = float(B[i, j]) if Bm[i, j] else 0.0
            t = beta * b  # one IEEE multiply (the definition's inner rounding)
            v = float(Fraction(alpha) * Fraction(a) + Fraction(t))
            if abs(v) > tau:
                row.append((j, v))
        out[i] = row
    return out


def _brute_scale_add_identity(A, Am, alpha, beta, tau):
    """Definition c6 scale_add_identity: off-diagonal round(alpha*a), diagonal
    round(alpha*a_ii + beta) (a_ii = 0 if absent, inserted), kept iff |v| > tau."""
    n = A.shape[0]
    out = {}
    for i in range(n):
        row = []
        for j in range(n):
            if j == i:
                a = float(A[i, i]) if Am[i, i] else 0.0
                v = float(Fraction(alpha) * Fraction(a) + Fraction(beta))
            elif Am[i, j]:
                v = float(Fraction(alpha) * Fraction(float(A[i, j])))
            else:
                continue
            if abs(v) > tau:
                row.append((j, v))
        out[i] = row
    return out


def _ell(d, m, w):
    n = d.shape[0]
    e = Ell.empty(n, w)
    for i in range(n):
        cols = np.nonzero(m[i])[0]
        e.col[i, :len(cols)] = cols
        e.val[i, :len(cols)] = d[i, cols]
        e.nnz[i] = len(cols)
    return e


def _rows(e):
    out = {i: [] for i in range(e.n)}
    for i, j, v in entries_of(e):
        out[i].append((j, v))
    return out


def _bits_equal(got, want):
    for i in want:
        if [(j, np.float64(v).view(np.uint64)) for j, v in got[i]] != \
           [(j, np.float64(v).view(np.uint64)) for j, v in want[i]]:
            return False
    return True


# non-dyadic scalars: 1/3, 0.7, the SP2 X0 map of a spectrum [-6.38, 5.09] (BASELINE cfg3-like)
_ALPHAS = [1.0 / 3.0, -0.7, 1.1, -1.0 / 11.47]
_BETAS = [0.7, -1.0 / 3.0, 2.3, 5.09 / 11.47]


@pytest.mark.parametrize("seed", range(12))
def test_c6_add_single_rounding_exact_rational(seed):
    rng = np.random.default_rng(600 + seed)
    n = int(rng.integers(10, 24))
    Am = rng.random((n, n)) < 0.4
    Bm = rng.random((n, n)) < 0.4
    A = np.where(Am, rng.standard_normal((n, n)), 0.0)
    B = np.where(Bm, rng.standard_normal((n, n)), 0.0)
    alpha, beta = _ALPHAS[seed % 4], _BETAS[(seed // 4) % 4]
    # planted cancellations: b = -alpha*a/beta on a third of the shared pattern (v ~ 1 ulp of a)
    both = Am & Bm
    plant = both & (rng.random((n, n)) < 0.5)
    B = np.where(plant, -alpha * A / beta, B)
    tau = [0.0, 1e-15, 1e-3][seed % 3]
    want = _brute_add(A, Am, B, Bm, alpha, beta, tau)
    w = 2 * n + 2
    Ae, Be = _ell(A, Am, w), _ell(B, Bm, w)
    r = oracle.add(Ae, Be, alpha, beta, tau)
    assert r.status == oracle.OK
    got = _rows(Ae)
    assert _bits_equal(got, want)
    # the fixture distinguishes one rounding from two (alpha*a + beta*b) on some entry
    two = 0
    for i in range(n):
        for j in range(n):
            if Am[i, j] or Bm[i, j]:
                a = A[i, j] if Am[i, j] else 0.0
                b = B[i, j] if Bm[i, j] else 0.0
                two += float(Fraction(alpha) * Fraction(a) + Fraction(beta * b)) != float(alpha * a) + float(beta * b)
    assert two > 0


def test_c6_add_alias_same_descriptor():
    """A <- (alpha + beta) A as fma(alpha, a, beta*a) (B is A itself)."""
    rng = np.random.default_rng(61)
    n = 16
    Am = rng.random((n, n)) < 0.5
    A = np.where(Am, rng.standard_normal((n, n)), 0.0)
    alpha, beta = 1.0 / 3.0, 0.7
    want = _brute_add(A, Am, A, Am, alpha, beta, 0.0)
    Ae = _ell(A, Am, n + 2)
    assert oracle.add(Ae, Ae, alpha, beta, 0.0).status == oracle.OK
    assert _bits_equal(_rows(Ae), want)


@pytest.mark.parametrize("seed", range(8))
def test_c6_scale_add_identity_single_rounding(seed):
    """The SP2 X0 map: alpha = -1/(emax - emin), beta = emax/(emax - emin) with
    diagonal entries planted at h_ii ~ emax (alpha*h + beta cancels), some diagonals absent."""
    rng = np.random.default_rng(700 + seed)
    n = int(rng.integers(6, 40))
    Am = rng.random((n, n)) < 0.25
    Am = Am | Am.T
    A = np.where(Am, rng.uniform(-2.0, 0.0, (n, n)), 0.0)
    emin, emax = -6.38 + 0.1 * seed, 5.09 - 0.07 * seed
    dl = emax - emin
    alpha, beta = -1.0 / dl, emax / dl
    diag = np.diag(A).copy()
    for i in range(n):
        if rng.random() < 0.5:
            Am[i, i] = True
            diag[i] = emax * (1.0 + rng.integers(-4, 5) * 2.0 ** -52)  # alpha*h + beta ~ 0
        elif rng.random() < 0.5:
            Am[i, i] = False
            diag[i] = 0.0
    np.fill_diagonal(A, diag)
    tau = [0.0, 1e-17, 1e-5][seed % 3]
    want = _brute_scale_add_identity(A, Am, alpha, beta, tau)
    Ae = _ell(A, Am, n + 2)
    r = oracle.scale_add_identity(Ae, alpha, beta, tau)
    assert r.status == oracle.OK
    assert _bits_equal(_rows(Ae), want)
    # two roundings (alpha*h + beta) differ on a planted diagonal
    diff = sum(float(Fraction(alpha) * Fraction(float(diag[i])) + Fraction(beta)) != float(alpha * diag[i]) + beta
               for i in range(n) if Am[i, i])
    assert diff > 0


def test_c6_add_identity_is_one_rounding_of_a_plus_beta():
    """add_identity: a_ii + beta in one rounding (inserted when absent); off-diagonals untouched."""
    A = np.array([[0.1, 0.2, 0.0], [0.0, 0.0, 0.3], [0.4, 0.0, 1.0 / 3.0]])
    Am = A != 0.0
    beta = 0.7
    want = _brute_scale_add_identity(A, Am, 1.0, beta, 0.0)
    Ae = _ell(A, Am, 4)
    assert oracle.add_identity(Ae, beta, 0.0).status == oracle.OK
    assert _bits_equal(_rows(Ae), want)
    assert want[1][0] == (1, 0.7) and want[0][0] == (0, 0.1 + 0.7)


# ------------------------------------------------------------- c10 (vi): the stop rule


def _canonical(d):
    """§8c-c7: sequential 256-row block sums, then a sequential sum over the blocks."""
    total = 0.0
    for b in range(0, len(d), 256):
        t = 0.0
        for x in d[b:b + 256]:
            t = t + x
        total = total + t
    return total


def replay_diag_sp2(h, nocc, tau, max_iter):
    """SP2 (§8c-c9, c10 (i)-(v)) on H = diag(h) in binary64 scalar operations. Returns the per
    iteration (branch, trX, trS, e) and the final diagonal, WITHOUT any stop rule (runs
    max_iter steps or until the iterate is empty)."""
    emin, emax = min(h), max(h)  # Gershgorin of a diagonal matrix (c8)
    dl = emax - emin
    alpha, beta = -1.0 / dl, emax / dl
    x = []
    for hv in h:
        v = fma_exact(alpha, hv, beta)  # X0 diagonal, one rounding (c6)
        x.append(v if abs(v) > tau else None)
    trX = _canonical([v if v is not None else 0.0 for v in x])
    recs = []
    for _ in range(max_iter):
        sq = trX > float(nocc)  # (i), tie -> EXPAND
        s = [v * v if v is not None else 0.0 for v in x]  # (ii) pre-drop diagonal of X^2
        trS = _canonical(s)
        nx = []
        for v, sv in zip(x, s):
            if v is None:
                nx.append(None)
                continue
            c = sv if sq else 2.0 * v - sv  # (iii) 2x exact: one rounding
            nx.append(c if abs(c) > tau else None)
        e = trX - trS
        recs.append(("SQUARE" if sq else "EXPAND", trX, trS, e))
        x = nx
        trX = _canonical([v if v is not None else 0.0 for v in x])
    return recs


def stop_by_rule(es, tol, min_iter, stag_gate, max_iter):
    """The stop rule as SURVEY §8c-c10 (vi) states it: returns (iterations, reason)."""
    for n, e in enumerate(es):
        if abs(e) <= tol:
            return n + 1, "CONVERGED"
        if n + 1 >= min_iter and e <= stag_gate and n >= 2 and e >= es[n - 2]:
            return n + 1, "STAGNATED"
        if n + 1 == max_iter:
            return n + 1, "NOCONV"
    raise AssertionError("sequence too short")


def _misreadings(es, n, gate, tol):
    """Stop iterations of the plausible misreadings of (vi), for min_iter = n + 1."""
    out = {}
    rules = {
        "e_{n-1}": lambda k, e: k + 1 >= n + 1 and e <= gate and k >= 1 and e >= es[k - 1],
        "k>=min_iter": lambda k, e: k >= n + 1 and e <= gate and k >= 2 and e >= es[k - 2],
        "e<gate": lambda k, e: k + 1 >= n + 1 and e < gate and k >= 2 and e >= es[k - 2],
    }
    for name, rule in rules.items():
        stop = None
        for k, e in enumerate(es):
            if abs(e) <= tol:
                stop = (k + 1, "CONVERGED")
                break
            if rule(k, e):
                stop = (k + 1, "STAGNATED")
                break
        out[name] = stop
    return out


def _find_stagnation_fixture(tau, nlev, seeds):
    """A diagonal H whose replayed e sequence has an index n >= 2 with e_n < e_{n-1} and
    e_n >= e_{n-2} (> 0): with min_iter = n + 1 and stag_gate = e_n the rule stops at n + 1,
    and every misreading stops elsewhere."""
    for seed in seeds:
        rng = np.random.default_rng(seed)
        h = [float(v) for v in np.sort(rng.uniform(-1.0, 1.0, nlev))]
        nocc = int(rng.integers(1, nlev))
        recs = replay_diag_sp2(h, nocc, tau, 60)
        es = [r[3] for r in recs]
        for n in range(2, len(es) - 1):
            e = es[n]
            if e > 0 and e < es[n - 1] and e >= es[n - 2] and all(x > 0 for x in es[:n]):
                mis = _misreadings(es, n, e, 0.0)
                if all(m != (n + 1, "STAGNATED") for m in mis.values()):
                    return h, nocc, recs, n
    raise AssertionError("no fixture found")


@pytest.mark.parametrize("tau,nlev,seeds", [(0.0, 9, range(0, 400)), (1e-3, 12, range(400, 800)),
                                              (0.0, 30, range(800, 1200))])
def test_c10_stagnated_rule_diagonal_replay(tau, nlev, seeds):
    h, nocc, recs, n = _find_stagnation_fixture(tau, nlev, seeds)
    es = [r[3] for r in recs]
    gate = es[n]
    H = from_dense(np.diag(h), w=2)
    opts = oracle.SP2Opts(threshold=tau, max_iter=60, min_iter=n + 1, stag_gate=gate)
    r = oracle.sp2(H, nocc, 0.0, opts)
    assert (r.iterations, r.stop) == stop_by_rule(es, 0.0, n + 1, gate, 60) == (n + 1, "STAGNATED")
    # the e sequence, branches and traces are the replay's, bit for bit
    for k, it in enumerate(r.iters):
        assert (it["branch"], it["trX"], it["trS"], it["e"]) == recs[k]
    # the boundary cases of the rule, each at the same fixture
    assert es[n] < es[n - 1]  # compared with e_{n-1} it would not stagnate here
    r2 = oracle.sp2(H, nocc, 0.0, oracle.SP2Opts(threshold=tau, max_iter=60, min_iter=n + 2, stag_gate=gate))
    assert (r2.iterations, r2.stop) == stop_by_rule(es, 0.0, n + 2, gate, 60)
    assert r2.iterations != n + 1
    below = float(np.nextafter(gate, -np.inf))  # gate one ulp below e_n: not <= gate
    r3 = oracle.sp2(H, nocc, 0.0, oracle.SP2Opts(threshold=tau, max_iter=60, min_iter=n + 1, stag_gate=below))
    assert (r3.iterations, r3.stop) == stop_by_rule(es, 0.0, n + 1, below, 60)
    assert r3.iterations != n + 1


def test_c10_stop_precedence_and_gate():
    """CONVERGED is tested before STAGNATED; the gate keeps stagnation off while e is large
    (R9: an ungated e_n >= e_{n-2} test fires while e is still falling on average)."""
    h, nocc, recs, n = _find_stagnation_fixture(0.0, 9, range(0, 400))
    es = [r[3] for r in recs]
    H = from_dense(np.diag(h), w=2)
    # tol = e_n: CONVERGED at n + 1 even though the stagnation test also holds there
    r = oracle.sp2(H, nocc, es[n], oracle.SP2Opts(max_iter=60, min_iter=n + 1, stag_gate=es[n]))
    assert (r.iterations, r.stop) == stop_by_rule(es, es[n], n + 1, es[n], 60)
    assert r.stop == "CONVERGED" and r.iterations <= n + 1
    # gate below every e: never STAGNATED
    r = oracle.sp2(H, nocc, 0.0, oracle.SP2Opts(max_iter=60, min_iter=3, stag_gate=min(es[:n + 1]) / 2))
    assert (r.iterations, r.stop) == stop_by_rule(es, 0.0, 3, min(es[:n + 1]) / 2, 60)
    # max_iter exactly at n + 1 with the rule off (min_iter beyond): NOCONV with n + 1 iterations
    r = oracle.sp2(H, nocc, 0.0, oracle.SP2Opts(max_iter=n + 1, min_iter=100))
    assert (r.iterations, r.stop, r.status) == (n + 1, "NOCONV", oracle.NOCONV)


# ------------------------------------------------- c4 at X0: the exact overflow-row count


@pytest.mark.parametrize("seed,tau", [(31, 0.0), (32, 0.05)])
def test_c4_sp2_fail_at_x0_counts_rows_over_the_width(seed, tau):
    """SP2 with FAIL whose X0 = drop(alpha H + beta I) overflows the initial width: the report
    carries required_width = max kept count and overflow_rows = #{i : kept_i > W} (§8c-c4), with
    the kept counts of X0 computed here from the definition (c6 diagonal fma, c3 drop)."""
    import synth
    H = synth.sym_banded(300, 40, 10, 30, 1, -1.0, 1.0, 0, 10.0, 0.0, seed)
    d = H.to_dense()
    m = np.zeros_like(d, dtype=bool)
    for i in range(H.n):
        m[i, H.col[i, :H.nnz[i]]] = True
    lo, hi = oracle.gershgorin(H)
    alpha, beta = -1.0 / (hi - lo), hi / (hi - lo)
    kept = np.zeros(H.n, int)
    for i in range(H.n):
        for j in np.nonzero(m[i])[0]:
            if j != i:
                kept[i] += abs(float(Fraction(alpha) * Fraction(float(d[i, j])))) > tau
        a = float(d[i, i]) if m[i, i] else 0.0
        kept[i] += abs(float(Fraction(alpha) * Fraction(a) + Fraction(beta))) > tau
    w = int(np.percentile(kept, 60)) & ~1
    r = oracle.sp2(H, 150, 1e-8, oracle.SP2Opts(threshold=tau, on_overflow=0, initial_width=w), d_width=300)
    assert r.status == oracle.OVERFLOW and r.fail_iter == -1
    assert r.required_width == kept.max()
    assert r.overflow_rows == int((kept > w).sum()) > 0
