"""Full-size SP2 and X^2 checks on the GPU against closed forms and invariants:
no oracle is needed, so N = 65536 runs in seconds.

 * Diagonal H: every iterate is diagonal and SP2 is the scalar recursion x <- x^2 | 2x - x^2 per
   level with the branch sequence the run reports; replayed in extended precision from the
   spectral map x0 = (emax - h)/(emax - emin), and the limit is the projector on the
   nocc lowest levels.
 * 2x2 dimer blocks [[eA, t], [t, eB]] (the paper's two-level unit): D is block-diagonal
   with each block the projector on the block's lower eigenvector when nocc = number of blocks
   and every lower level lies below every upper one.
 * X^2 threshold monotonicity (T5): raising tau only removes entries; the common entries are bitwise
   equal.
"""
import numpy as np
import pytest

import synth
from synth import Ell

pytestmark = pytest.mark.gpu


def eb():
    import paper_2102_08505_b200 as m
    return m


def _diag_ell(h):
    n = len(h)
    E = Ell.empty(n, 2)
    E.val[:, 0] = h
    E.col[:, 0] = np.arange(n, dtype=np.int32)
    E.nnz[:] = 1
    return E


def test_diagonal_h_scalar_recursion_n65536():
    n = 65536
    rng = np.random.default_rng(65536)
    h = np.sort(rng.uniform(-3.0, 2.0, n))
    nocc = 24577
    H = _diag_ell(h)
    ctx = eb().Context(0)
    d = eb().Mat.empty(n, 2)
    g = ctx.sp2_run(eb().Mat.from_host(H), nocc, 1e-9, d, max_iter=80)
    assert g.stop in ("CONVERGED", "STAGNATED")
    lo, hi = h.min(), h.max()  # Gershgorin of a diagonal matrix = its extreme entries
    assert (g.emin, g.emax) == (lo, hi)
    x = (np.longdouble(hi) - h.astype(np.longdouble)) / (np.longdouble(hi) - np.longdouble(lo))
    for it in g.iters:
        x = x * x if it["branch"] == "SQUARE" else 2 * x - x * x
    D = d.to_host()
    assert np.all(D.nnz <= 1) and np.all(D.col[D.nnz == 1, 0] == np.flatnonzero(D.nnz == 1))
    got = np.zeros(n)
    got[D.nnz == 1] = D.val[D.nnz == 1, 0]
    assert np.max(np.abs(got - x.astype(np.float64))) <= 1e-9
    assert np.max(np.abs(got - (np.arange(n) < nocc))) <= 1e-6
    ctx.close()


def test_dimer_blocks_closed_form_n65536():
    nb = 32768
    n = 2 * nb
    rng = np.random.default_rng(2)
    ea = rng.uniform(-1.0, -0.2, nb)
    eB = rng.uniform(0.2, 1.0, nb)
    t = rng.uniform(-0.5, -0.1, nb)
    H = Ell.empty(n, 2)
    r0 = np.arange(0, n, 2)
    H.col[r0, 0], H.col[r0, 1] = r0, r0 + 1
    H.val[r0, 0], H.val[r0, 1] = ea, t
    H.col[r0 + 1, 0], H.col[r0 + 1, 1] = r0, r0 + 1
    H.val[r0 + 1, 0], H.val[r0 + 1, 1] = t, eB
    H.nnz[:] = 2
    ctx = eb().Context(0)
    d = eb().Mat.empty(n, 2)
    g = ctx.sp2_run(eb().Mat.from_host(H), nb, 0.0, d, max_iter=80, min_iter=10)
    assert g.stop in ("CONVERGED", "STAGNATED")
    m, dd = (ea + eB) / 2, (ea - eB) / 2
    lam = m - np.sqrt(dd * dd + t * t)
    v = np.stack([t, lam - ea], axis=1)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    D = d.to_host()
    dense = np.zeros((nb, 2, 2))
    for rr in range(2):
        rows = r0 + rr
        for s in range(2):
            hit = (D.nnz[rows] > s)
            c = D.col[rows, s] - r0
            dense[hit, rr, c[hit]] = D.val[rows[hit], s]
    ref = np.einsum("bi,bj->bij", v, v)
    assert np.max(np.abs(dense - ref)) <= 1e-12
    assert abs(g.trD - nb) <= 1e-9
    ctx.close()


def test_x2_threshold_monotone_cfg5():
    X = synth.cfg5(32768, 64)
    ctx = eb().Context(0)
    x = eb().Mat.from_host(X)
    outs = []
    for tau in (0.0, 1e-5, 1e-3):
        y = eb().Mat.empty(X.n, 2048)
        st, _, _ = ctx.multiply_x2(x, y, tau)
        assert st == eb().OK
        outs.append(y.to_host())
    for lo, hi in zip(outs, outs[1:]):
        assert np.all(hi.nnz <= lo.nnz)
        for i in range(0, X.n, 97):
            a = dict(zip(lo.col[i, :lo.nnz[i]].tolist(), lo.val[i, :lo.nnz[i]].view(np.uint64).tolist()))
            for c, v in zip(hi.col[i, :hi.nnz[i]].tolist(), hi.val[i, :hi.nnz[i]].view(np.uint64).tolist()):
                assert a[c] == v
    ctx.close()
