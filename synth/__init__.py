"""Seeded synthetic ELLPACK inputs (BASELINE.json configs 1..5 + test matrices).

Input synthesis only: this package holds none of the method's arithmetic. It is
the one module both sides may import -- the CPU oracle (``oracle/``) and the
CUDA path (``paper_2102_08505_b200``) consume exactly the bytes it produces.
The generator recipes (reading S14) are documented in
``synth/gen.c`` and DESIGN.md "Input recipe".

Host matrices are :class:`Ell` -- canonical row-major ELLPACK
(``val[n, w]`` float64, ``col[n, w]`` int32, ``nnz[n]`` int32, each row's
columns strictly ascending, padding zeroed).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libsynth.so")


def build(force: bool = False) -> str:
    """Compile gen.c -> libsynth.so with gcc (host code, no GPU needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64, i32, u64, d, i = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double, ctypes.c_int
        _lib.synth_sym_banded.argtypes = [i64, i32, i32, i64, i, d, d, i, d, d, u64, P, P, P]
        _lib.synth_cfg2.argtypes = [i64, i32, i32, i64, d, u64] + [P] * 9
        _lib.synth_lattice.argtypes = [i32, i32, u64, P, P, P]
        _lib.synth_random.argtypes = [i64, i32, i32, i32, i64, d, d, u64, P, P, P]
        _lib.synth_products.argtypes = [i64, i32, P, P, P]
        _lib.synth_products.restype = i64
        for f in ("synth_sym_banded", "synth_cfg2", "synth_lattice", "synth_random"):
            getattr(_lib, f).restype = i
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Ell:
    """Host ELLPACK matrix (canonical form; see module docstring)."""

    val: np.ndarray  # float64 [n, w]
    col: np.ndarray  # int32   [n, w]
    nnz: np.ndarray  # int32   [n]

    @property
    def n(self) -> int:
        return int(self.nnz.shape[0])

    @property
    def w(self) -> int:
        return int(self.val.shape[1])

    @staticmethod
    def empty(n: int, w: int) -> "Ell":
        return Ell(np.zeros((n, w), np.float64), np.zeros((n, w), np.int32), np.zeros(n, np.int32))

    def copy(self) -> "Ell":
        return Ell(self.val.copy(), self.col.copy(), self.nnz.copy())

    def widened(self, w: int) -> "Ell":
        """Same matrix stored at a different width (w >= max nnz)."""
        assert w >= int(self.nnz.max(initial=0))
        out = Ell.empty(self.n, w)
        k = min(w, self.w)
        out.val[:, :k] = self.val[:, :k]
        out.col[:, :k] = self.col[:, :k]
        out.nnz[:] = self.nnz
        return out

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n, self.n), np.float64)
        for i in range(self.n):
            k = int(self.nnz[i])
            d[i, self.col[i, :k]] = self.val[i, :k]
        return d

    def rows(self):
        for i in range(self.n):
            k = int(self.nnz[i])
            yield self.col[i, :k], self.val[i, :k]

    def canonical(self) -> bool:
        """Row invariants: 0<=nnz<=w, cols in [0,n) strictly ascending, finite."""
        if self.nnz.min(initial=0) < 0 or self.nnz.max(initial=0) > self.w:
            return False
        for c, v in self.rows():
            if len(c) and (c[0] < 0 or c[-1] >= self.n or np.any(np.diff(c) <= 0)):
                return False
            if not np.all(np.isfinite(v)):
                return False
        return True


def from_dense(d: np.ndarray, w: int | None = None) -> Ell:
    """Store exactly the nonzero entries of a dense square matrix (format conversion only)."""
    n = d.shape[0]
    counts = (d != 0).sum(axis=1)
    if w is None:
        w = max(1, int(counts.max(initial=0)))
    out = Ell.empty(n, w)
    for i in range(n):
        cols = np.nonzero(d[i])[0]
        if len(cols) > w:
            raise ValueError(f"row {i} has {len(cols)} nonzeros > width {w}")
        out.col[i, : len(cols)] = cols
        out.val[i, : len(cols)] = d[i, cols]
        out.nnz[i] = len(cols)
    return out


def sym_banded(n, w, partners, band, diag_kind, dlo, dhi, off_kind, decay, amp, seed) -> Ell:
    m = Ell.empty(n, w)
    e = _L().synth_sym_banded(n, w, partners, band, diag_kind, dlo, dhi, off_kind, decay, amp, seed,
                              _p(m.val), _p(m.col), _p(m.nnz))
    if e:
        raise ValueError("synth_sym_banded: bad arguments")
    return m


def random_sparse(n, w, kmin, kmax, band=None, p_empty=0.0, scale=1.0, seed=0) -> Ell:
    """Generic seeded non-symmetric test matrix (edge cases: empty / full rows, ragged n)."""
    m = Ell.empty(n, w)
    e = _L().synth_random(n, w, kmin, kmax, n if band is None else band, p_empty, scale, seed,
                          _p(m.val), _p(m.col), _p(m.nnz))
    if e:
        raise ValueError("synth_random: bad arguments")
    return m


def products(a: Ell, b: Ell) -> int:
    """P = sum_i sum_{k in A_i} nnz_B(k): the method's scalar product count (pattern only)."""
    return int(_L().synth_products(a.n, a.w, _p(a.col), _p(a.nnz), _p(b.nnz)))


# ---------------------------------------------------------------- configs
# BASELINE.json "configs" (indices 0..4 = cfg1..cfg5), recipes per SURVEY.md §8d.

def cfg1(seed: int = 0) -> Ell:
    """cfg1: N=512, M=32, symmetric; diag U(-1,1); 15 partners |i-j|<=64; z*exp(-|i-j|/16)."""
    return sym_banded(512, 32, 15, 64, 1, -1.0, 1.0, 0, 16.0, 0.0, seed)


CFG1 = dict(n=512, m=32, threshold=1e-5, alpha=1.0, beta=0.0)


def cfg2(seed: int = 1, n: int = 16384, m: int = 128):
    """cfg2: A, B, C_old from one stream; diag + 47 partners |i-j|<=512; z*exp(-|i-j|/64)."""
    A, B, C = Ell.empty(n, m), Ell.empty(n, m), Ell.empty(n, m)
    e = _L().synth_cfg2(n, m, 47, 512, 64.0, seed, _p(A.val), _p(A.col), _p(A.nnz),
                        _p(B.val), _p(B.col), _p(B.nnz), _p(C.val), _p(C.col), _p(C.nnz))
    if e:
        raise ValueError("synth_cfg2: bad arguments")
    return A, B, C


CFG2 = dict(n=16384, m=128, threshold=1e-6, alpha=1.0, beta=0.5)


def cfg3(seed: int = 3, n: int = 12288, m: int = 256) -> Ell:
    """cfg3 H: diag U(-2,0); 16 partners |i-j|<=1024; 0.5*exp(-|i-j|/128)*sign, mirrored."""
    return sym_banded(n, m, 16, 1024, 1, -2.0, 0.0, 1, 128.0, 0.5, seed)


CFG3 = dict(n=12288, m=256, threshold=1e-5, tol=1e-8, nocc=6144)


def cfg4(seed: int = 4, L: int = 32, m: int = 256) -> Ell:
    """cfg4 H: L^3 lattice, 2 orbitals/site, NN + NNN hoppings U(-1,-0.5), on-site U(-0.5,0.5)."""
    n = 2 * L ** 3
    h = Ell.empty(n, m)
    e = _L().synth_lattice(L, m, seed, _p(h.val), _p(h.col), _p(h.nnz))
    if e:
        raise ValueError("synth_lattice: bad arguments")
    return h


CFG4 = dict(n=65536, m=256, threshold=1e-5, tol=1e-8, nocc=32768)


def cfg5(n: int, m: int, seed: int = 5) -> Ell:
    """cfg5: diag z; M/4 partners |i-j|<=8M; z*exp(-|i-j|/M), mirrored, capped at M."""
    return sym_banded(n, m, m // 4, 8 * m, 2, 0.0, 0.0, 0, float(m), 0.0, seed)


CFG5 = dict(ns=(32768, 131072, 262144), ms=(64, 128, 256), threshold=1e-5)


# ------------------------------------------------------------ paper model Hamiltonian (f2)
# The paper's two-level-system presets. Parameter
# names follow SPEC's ModelParams; unset parameters are 0.0.
MODEL_PRESETS = {
    "metal": dict(d_aa=-1.0, d_bb=-1.0, k=-0.01),
    "semiconductor": dict(d_bb=-1.0, d_ab_intra=-2.0, k=-0.01),
    "soft_matter": dict(d_bb=-1.0, d_ab_intra=-1.0, eps_a=-10.0, k=-0.1, r=1.0),
}


def model_hamiltonian(n: int, kind: str = "soft_matter", tau_store: float = 1e-5, seed: int = 6, **over) -> Ell:
    """Two-level model Hamiltonian (synth_model in gen.c), stored entries |h| > tau_store."""
    prm = dict(eps_a=0.0, eps_b=0.0, d_aa=0.0, d_bb=0.0, d_ab_intra=0.0, d_ab_cross=0.0, k=0.0, r=0.0)
    prm.update(MODEL_PRESETS[kind])
    prm.update(over)
    L = _L()
    f = L.synth_model
    f.restype = ctypes.c_int64
    f.argtypes = [ctypes.c_int64, ctypes.c_int32] + [ctypes.c_double] * 9 + [ctypes.c_uint64] + [ctypes.c_void_p] * 3
    args = (prm["eps_a"], prm["eps_b"], prm["d_aa"], prm["d_bb"], prm["d_ab_intra"], prm["d_ab_cross"], prm["k"],
            prm["r"], tau_store)
    wmax = f(n, 0, *args, seed, None, None, None)
    if wmax < 0:
        raise ValueError("synth_model: bad arguments")
    w = max(2, int(wmax) + (int(wmax) & 1))
    m = Ell.empty(n, w)
    if f(n, w, *args, seed, _p(m.val), _p(m.col), _p(m.nnz)) != 0:
        raise ValueError("synth_model: row wider than the sized width")
    return m
