"""CPU oracle for the ELLPACK multiply / SP2 hot path (arXiv 2102.08505).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package. The product path (``paper_2102_08505_b200``) never imports it and the
two share no code (the seeded generators in ``synth/`` serve both and hold
none of the method's arithmetic).

The arithmetic lives in ``oracle.c`` (plain C99, fp64, explicit ``fma``,
``-ffp-contract=off``), which cites SURVEY.md §8(c) and the SPEC/PAPER lines
for each function. This wrapper only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

from synth import Ell

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, ARG, DIM, OVERFLOW, BOUNDS, NOCONV, NOMEM = range(7)
STOP_NAMES = {0: "CONVERGED", 1: "STAGNATED", 2: "NOCONV", 3: "OVERFLOW"}


def build(force: bool = False) -> str:
    """gcc -O2 -fopenmp -ffp-contract=off (never -ffast-math) -> liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp",
                               "-ffp-contract=off", "-fno-fast-math", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _OMat(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("w", ctypes.c_int32), ("val", ctypes.c_void_p),
                ("col", ctypes.c_void_p), ("nnz", ctypes.c_void_p)]


class _Opts(ctypes.Structure):
    _fields_ = [("threshold", ctypes.c_double), ("max_iter", ctypes.c_int32), ("min_iter", ctypes.c_int32),
                ("stag_gate", ctypes.c_double), ("emin", ctypes.c_double), ("emax", ctypes.c_double),
                ("on_overflow", ctypes.c_int32), ("max_width", ctypes.c_int32),
                ("initial_width", ctypes.c_int32), ("branch_rule", ctypes.c_int32)]


class _Iter(ctypes.Structure):
    _fields_ = [("trX", ctypes.c_double), ("trS", ctypes.c_double), ("e", ctypes.c_double),
                ("fnorm", ctypes.c_double), ("branch", ctypes.c_int32), ("width", ctypes.c_int32),
                ("required", ctypes.c_int32), ("pad", ctypes.c_int32), ("products", ctypes.c_int64),
                ("frob2", ctypes.c_double)]


class _Report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("stop_reason", ctypes.c_int32),
                ("final_width", ctypes.c_int32), ("regrows", ctypes.c_int32),
                ("emin", ctypes.c_double), ("emax", ctypes.c_double), ("trD", ctypes.c_double),
                ("overflow_rows", ctypes.c_int64), ("required_width", ctypes.c_int32),
                ("fail_iter", ctypes.c_int32)]


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P, d, i64, i32 = ctypes.c_void_p, ctypes.c_double, ctypes.c_int64, ctypes.c_int32
        M = ctypes.POINTER(_OMat)
        sig = {
            "oracle_multiply_ex": [M, M, M, d, d, d, P, P, P],
            "oracle_x2": [M, M, d, P, P, P, P],
            "oracle_add": [M, M, d, d, d, P, P],
            "oracle_scale_add_identity": [M, d, d, d, P, P],
            "oracle_add_identity": [M, d, d, P, P],
            "oracle_trace": [M, P],
            "oracle_fnorm_diff": [M, M, P],
            "oracle_gershgorin": [M, P, P],
            "oracle_sp2": [M, i64, d, ctypes.POINTER(_Opts), M, ctypes.POINTER(_Report), P],
            "oracle_set_threads": [ctypes.c_int],
            "oracle_canonical_sum": [P, i64],
            "oracle_block_partials": [P, i64, P],
        }
        for name, args in sig.items():
            f = getattr(_lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        _lib.oracle_canonical_sum.restype = ctypes.c_double
        _lib.oracle_set_threads.restype = None
        _lib.oracle_block_partials.restype = None
        _lib.oracle_num_threads.restype = ctypes.c_int
    return _lib


def _m(e: Ell) -> _OMat:
    for a in (e.val, e.col, e.nnz):
        assert a.flags.c_contiguous
    assert e.val.dtype == np.float64 and e.col.dtype == np.int32 and e.nnz.dtype == np.int32
    return _OMat(e.n, e.w, e.val.ctypes.data, e.col.ctypes.data, e.nnz.ctypes.data)


def _ptr(x):
    return ctypes.cast(ctypes.byref(x), ctypes.c_void_p)


def set_threads(t: int) -> None:
    _L().oracle_set_threads(int(t))


def num_threads() -> int:
    return int(_L().oracle_num_threads())


@dataclass
class Result:
    status: int
    overflow_rows: int = 0
    required_width: int = 0
    trace_x: float = float("nan")
    trace_x2: float = float("nan")
    diag_s: np.ndarray | None = None


def multiply(A: Ell, B: Ell, C: Ell, alpha: float, beta: float, tau: float, want_diag=False) -> Result:
    """C <- drop_tau(alpha*A*B + beta*C) in place (§8c-c2..c4)."""
    ovf, req = ctypes.c_int64(0), ctypes.c_int32(0)
    ds = np.zeros(A.n, np.float64) if want_diag else None
    ma, mb, mc = _m(A), _m(B), _m(C)
    rc = _L().oracle_multiply_ex(ctypes.byref(ma), ctypes.byref(mb), ctypes.byref(mc), alpha, beta, tau,
                                 _ptr(ovf), _ptr(req), None if ds is None else ds.ctypes.data)
    return Result(rc, ovf.value, req.value, diag_s=ds)


def x2(X: Ell, X2: Ell, tau: float) -> Result:
    """X2 <- drop_tau(X*X); returns tr(X), tr(X^2) pre-drop (§8c-c5)."""
    ovf, req = ctypes.c_int64(0), ctypes.c_int32(0)
    tx, tx2 = ctypes.c_double(math.nan), ctypes.c_double(math.nan)
    mx, my = _m(X), _m(X2)
    rc = _L().oracle_x2(ctypes.byref(mx), ctypes.byref(my), tau, _ptr(tx), _ptr(tx2), _ptr(ovf), _ptr(req))
    return Result(rc, ovf.value, req.value, tx.value, tx2.value)


def add(A: Ell, B: Ell, alpha: float, beta: float, tau: float) -> Result:
    """A <- drop_tau(alpha*A + beta*B) (§8c-c6)."""
    ovf, req = ctypes.c_int64(0), ctypes.c_int32(0)
    ma = _m(A)
    mb = ma if B is A else _m(B)
    rc = _L().oracle_add(ctypes.byref(ma), ctypes.byref(mb), alpha, beta, tau, _ptr(ovf), _ptr(req))
    return Result(rc, ovf.value, req.value)


def scale_add_identity(A: Ell, alpha: float, beta: float, tau: float) -> Result:
    ovf, req = ctypes.c_int64(0), ctypes.c_int32(0)
    ma = _m(A)
    rc = _L().oracle_scale_add_identity(ctypes.byref(ma), alpha, beta, tau, _ptr(ovf), _ptr(req))
    return Result(rc, ovf.value, req.value)


def add_identity(A: Ell, beta: float, tau: float) -> Result:
    ovf, req = ctypes.c_int64(0), ctypes.c_int32(0)
    ma = _m(A)
    rc = _L().oracle_add_identity(ctypes.byref(ma), beta, tau, _ptr(ovf), _ptr(req))
    return Result(rc, ovf.value, req.value)


def trace(A: Ell) -> float:
    out = ctypes.c_double(math.nan)
    ma = _m(A)
    rc = _L().oracle_trace(ctypes.byref(ma), _ptr(out))
    assert rc == OK
    return out.value


def fnorm_diff(A: Ell, B: Ell) -> float:
    out = ctypes.c_double(math.nan)
    ma, mb = _m(A), _m(B)
    rc = _L().oracle_fnorm_diff(ctypes.byref(ma), ctypes.byref(mb), _ptr(out))
    assert rc == OK
    return out.value


def gershgorin(H: Ell) -> tuple[float, float]:
    lo, hi = ctypes.c_double(), ctypes.c_double()
    mh = _m(H)
    rc = _L().oracle_gershgorin(ctypes.byref(mh), _ptr(lo), _ptr(hi))
    assert rc == OK
    return lo.value, hi.value


def canonical_sum(d: np.ndarray) -> float:
    d = np.ascontiguousarray(d, np.float64)
    return float(_L().oracle_canonical_sum(d.ctypes.data, d.shape[0]))


def block_partials(d: np.ndarray) -> np.ndarray:
    d = np.ascontiguousarray(d, np.float64)
    out = np.zeros((d.shape[0] + 255) // 256, np.float64)
    _L().oracle_block_partials(d.ctypes.data, d.shape[0], out.ctypes.data)
    return out


@dataclass
class SP2Opts:
    threshold: float = 0.0
    max_iter: int = 100
    min_iter: int = 20
    stag_gate: float = 1e-3
    emin: float = float("nan")
    emax: float = float("nan")
    on_overflow: int = 1  # 0 FAIL, 1 GROW
    max_width: int = 0
    initial_width: int = 0
    branch_rule: int = 0  # 0 trace sign, 1 trace-closest (§8f-f4 i, reading R19)


@dataclass
class SP2Result:
    status: int
    D: Ell
    iterations: int
    stop: str
    final_width: int
    regrows: int
    emin: float
    emax: float
    trD: float
    overflow_rows: int
    required_width: int
    fail_iter: int
    iters: list = field(default_factory=list)


def sp2(H: Ell, nocc: int, tol: float, opts: SP2Opts | None = None, d_width: int | None = None) -> SP2Result:
    """SP2-Basic (§8c-c9, c10). D is returned at width d_width (default n)."""
    o = opts or SP2Opts()
    co = _Opts(o.threshold, o.max_iter, o.min_iter, o.stag_gate, o.emin, o.emax, o.on_overflow,
               o.max_width, o.initial_width, o.branch_rule)
    D = Ell.empty(H.n, d_width or H.n)
    rep = _Report()
    its = (_Iter * max(1, o.max_iter))()
    mh, md = _m(H), _m(D)
    rc = _L().oracle_sp2(ctypes.byref(mh), nocc, tol, ctypes.byref(co), ctypes.byref(md), ctypes.byref(rep),
                         ctypes.cast(its, ctypes.c_void_p))
    iters = [dict(trX=its[k].trX, trS=its[k].trS, e=its[k].e, fnorm=its[k].fnorm,
                  branch="SQUARE" if its[k].branch == 0 else "EXPAND", width=its[k].width,
                  required=its[k].required, products=its[k].products,
                  frob2=its[k].frob2)
             for k in range(min(rep.iterations, o.max_iter))]
    return SP2Result(rc, D, rep.iterations, STOP_NAMES.get(rep.stop_reason, "?"), rep.final_width,
                     rep.regrows, rep.emin, rep.emax, rep.trD, rep.overflow_rows, rep.required_width,
                     rep.fail_iter, iters)
