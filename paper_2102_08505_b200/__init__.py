"""paper_2102_08505_b200 — B200-native ELLPACK SpGEMM + SP2 hot path (arXiv 2102.08505).

Thin ctypes binding over ``libellpack.so`` (C ABI: ``include/ellpack.h``). Every
computation runs in the library's sm_100a CUDA kernels; this module only
marshals arguments. PyTorch provides device memory, streams and
``torch.distributed`` process groups. There is NO CPU fallback: if the shared
library is missing or no CUDA device is present, calls raise.

Names follow the paper / ABI: ``multiply`` (C <- drop(alpha*A*B + beta*C)),
``multiply_x2`` (X^2 with tr(X), tr(X^2)), ``add``, ``add_identity``,
``scale_add_identity``, ``trace``, ``fnorm_diff``, ``gershgorin``, ``sp2_run``.
"""
from __future__ import annotations

import ctypes
import glob
import math
import os
import subprocess
from dataclasses import dataclass, field

_HERE = os.path.dirname(os.path.abspath(__file__))
_REPO = os.path.dirname(_HERE)
_LIB = os.environ.get("ELLPACK_LIB") or os.path.join(_HERE, "libellpack.so")
_SRCS = [os.path.join(_HERE, "csrc", f) for f in ("spgemm.cu", "split.cu", "reduce.cu", "sp2_graph.cu", "dense.cu", "tiny.cu",
                                                          "api.cu")]
_HDRS = [os.path.join(_HERE, "csrc", f) for f in ("internal.cuh", "devutil.cuh", "dense.cuh")] + [os.path.join(_REPO, "include", "ellpack.h")]

OK, ERR_ARG, ERR_DIM, ERR_OVERFLOW, ERR_BOUNDS, ERR_NOCONV, ERR_NOMEM, ERR_CUDA, ERR_NCCL, ERR_STATE = range(10)
OPT_WINDOW, OPT_WARPS, OPT_SP2_WIDTH0, OPT_PROFILE, OPT_ABLATE, OPT_GENERAL_WINDOW, OPT_VALIDATE = 1, 2, 3, 4, 5, 6, 7
OPT_SP2_SYMMETRIC = 8
OPT_SP2_MEM_CAP = 9
OPT_RING_KERNEL = 10
OPT_SP2_DEVICE_LOOP = 11
OPT_DENSE = 12
OPT_DENSE_KERNEL = 13
OPT_SMALL_KERNEL = 14
SP2_FAIL, SP2_GROW = 0, 1
SP2_RULE_TRACE_SIGN, SP2_RULE_TRACE_CLOSEST = 0, 1
STOP_NAMES = {0: "CONVERGED", 1: "STAGNATED", 2: "NOCONV", 3: "OVERFLOW"}

# Every symbol include/ellpack.h declares (checked by tests/test_abi.py).
ABI_SYMBOLS = (
    "ellpack_ctx_create", "ellpack_ctx_destroy", "ellpack_ctx_set_stream", "ellpack_ctx_set_option",
    "ellpack_ctx_kernel_launches", "ellpack_ctx_host_syncs", "ellpack_ctx_last_launch", "ellpack_ctx_kernel_time",
    "ellpack_create", "ellpack_destroy", "ellpack_multiply",
    "ellpack_multiply_x2", "ellpack_add", "ellpack_add_identity", "ellpack_scale_add_identity",
    "ellpack_trace", "ellpack_fnorm_diff", "ellpack_gershgorin", "ellpack_overflow_info", "sp2_run",
    "sp2_opts_default", "ellpack_multiply_x2_host", "ellpack_nccl_unique_id", "ellpack_ctx_attach_nccl",
    "ellpack_ctx_set_rows", "ellpack_allgather_rows", "ellpack_halo_rows", "ellpack_halo_plan",
    "ellpack_multiply_x2_halo", "ellpack_row_split",
    "ellpack_strerror",
)


def _nccl_include() -> str:
    import nvidia.nccl  # torch's bundled NCCL (2.28): header matches the runtime library
    return os.path.join(list(nvidia.nccl.__path__)[0], "include")


def build(force: bool = False, verbose: bool = False, defines=()) -> str:
    """nvcc -gencode arch=compute_100a,code=sm_100a -> libellpack.so (in-tree).
    defines: extra -D tuning macros (tools/variants.py A/B builds only)."""
    stale = force or defines or not os.path.exists(_LIB) or any(
        os.path.getmtime(s) > os.path.getmtime(_LIB) for s in _SRCS + _HDRS)
    if stale:
        import tempfile
        tmp = _LIB + f".tmp{os.getpid()}"
        flags = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
                 "-Xcompiler", "-fPIC", "-I" + os.path.join(_REPO, "include"), "-I" + _nccl_include(),
                 *[f"-D{d}" for d in defines]]
        if verbose:
            flags.insert(0, "-Xptxas=-v")
        with tempfile.TemporaryDirectory(prefix="ellbuild_") as td:
            # one nvcc per translation unit, in parallel, then one link
            objs = [os.path.join(td, os.path.basename(src) + ".o") for src in _SRCS]
            procs = [subprocess.Popen(["nvcc", *flags, "-c", src, "-o", o], cwd=_HERE) for src, o in zip(_SRCS, objs)]
            rcs = [pr.wait() for pr in procs]
            if any(rcs):
                raise subprocess.CalledProcessError(max(rcs), "nvcc")
            subprocess.check_call(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp,
                                   "-ldl"], cwd=_HERE)
        os.replace(tmp, _LIB)
    return _LIB


class EllpackError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {_lib_strerror(status)} (status {status})")


class Desc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("w", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("val", ctypes.c_void_p), ("col", ctypes.c_void_p), ("nnz", ctypes.c_void_p)]


class SP2Opts(ctypes.Structure):
    _fields_ = [("threshold", ctypes.c_double), ("max_iter", ctypes.c_int32), ("min_iter", ctypes.c_int32),
                ("stag_gate", ctypes.c_double), ("emin", ctypes.c_double), ("emax", ctypes.c_double),
                ("on_overflow", ctypes.c_int32), ("max_width", ctypes.c_int32),
                ("initial_width", ctypes.c_int32), ("branch_rule", ctypes.c_int32)]


class SP2IterRec(ctypes.Structure):
    _fields_ = [("trX", ctypes.c_double), ("trS", ctypes.c_double), ("e", ctypes.c_double),
                ("fnorm", ctypes.c_double), ("branch", ctypes.c_int32), ("width", ctypes.c_int32),
                ("required", ctypes.c_int32), ("regime", ctypes.c_int32), ("products", ctypes.c_int64),
                ("frob2", ctypes.c_double), ("products_exec", ctypes.c_int64), ("step_ms", ctypes.c_double)]


class SP2Report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("stop_reason", ctypes.c_int32),
                ("final_width", ctypes.c_int32), ("regrows", ctypes.c_int32),
                ("emin", ctypes.c_double), ("emax", ctypes.c_double), ("trD", ctypes.c_double),
                ("overflow_rows", ctypes.c_int64), ("required_width", ctypes.c_int32),
                ("fail_iter", ctypes.c_int32),
                ("t_read_hamiltonian", ctypes.c_double), ("t_init_misc", ctypes.c_double),
                ("t_sp2_loop_x2", ctypes.c_double), ("t_sp2_loop_norm", ctypes.c_double),
                ("t_sp2_loop_misc", ctypes.c_double), ("iters", ctypes.POINTER(SP2IterRec))]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libellpack.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} not built: run __graft_entry__.build() (nvcc, sm_100a)")
        L = ctypes.CDLL(_LIB)
        P, d, i64, i32, i = ctypes.c_void_p, ctypes.c_double, ctypes.c_int64, ctypes.c_int32, ctypes.c_int
        D = ctypes.POINTER(Desc)
        sig = {
            "ellpack_ctx_create": [i, P, P], "ellpack_ctx_destroy": [P], "ellpack_ctx_set_stream": [P, P],
            "ellpack_ctx_set_option": [P, i, i64], "ellpack_ctx_kernel_launches": [P], "ellpack_ctx_host_syncs": [P], "ellpack_ctx_last_launch": [P, P],
            "ellpack_ctx_kernel_time": [P, P, P],
            "ellpack_create": [P, i64, i32, D], "ellpack_destroy": [P, D],
            "ellpack_multiply": [P, D, D, D, d, d, d], "ellpack_multiply_x2": [P, D, D, d, P, P],
            "ellpack_add": [P, D, D, d, d, d], "ellpack_add_identity": [P, D, d, d],
            "ellpack_scale_add_identity": [P, D, d, d, d], "ellpack_trace": [P, D, P],
            "ellpack_fnorm_diff": [P, D, D, P], "ellpack_gershgorin": [P, D, P, P],
            "ellpack_overflow_info": [P, P, P],
            "sp2_run": [P, D, i64, d, ctypes.POINTER(SP2Opts), D, ctypes.POINTER(SP2Report)],
            "sp2_opts_default": [ctypes.POINTER(SP2Opts)],
            "ellpack_multiply_x2_host": [P, i64, i32, P, P, P, i32, P, P, P, d, P, P],
            "ellpack_nccl_unique_id": [P], "ellpack_ctx_attach_nccl": [P, i, i, P, i64, i64],
            "ellpack_ctx_set_rows": [P, i64, i64], "ellpack_allgather_rows": [P, D],
            "ellpack_halo_rows": [P, D, D], "ellpack_halo_plan": [i64, i32, i32, i64, P, P, P, P, P],
            "ellpack_multiply_x2_halo": [P, D, D, d, P, P], "ellpack_row_split": [i64, i64, i64, P],
            "ellpack_strerror": [i],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.ellpack_ctx_kernel_launches.restype = ctypes.c_int64
        L.ellpack_ctx_host_syncs.restype = ctypes.c_int64
        L.ellpack_strerror.restype = ctypes.c_char_p
        L.sp2_opts_default.restype = None
        _lib = L
    return _lib


def _lib_strerror(s: int) -> str:
    try:
        return lib().ellpack_strerror(s).decode()
    except Exception:  # pragma: no cover
        return "?"


def _chk(status: int, what: str, ok=(OK,)) -> int:
    if status not in ok:
        raise EllpackError(status, what)
    return status


def _torch():
    import torch
    return torch


class Mat:
    """Device ELLPACK matrix backed by torch tensors (val f64 [n,w], col i32 [n,w], nnz i32 [n])."""

    def __init__(self, val, col, nnz):
        torch = _torch()
        assert val.is_cuda and val.dtype == torch.float64 and col.dtype == torch.int32 and nnz.dtype == torch.int32
        assert val.is_contiguous() and col.is_contiguous() and nnz.is_contiguous()
        self.val, self.col, self.nnz = val, col, nnz
        self.desc = Desc(nnz.shape[0], val.shape[1], 0, val.data_ptr(), col.data_ptr(), nnz.data_ptr())

    @property
    def n(self) -> int:
        return int(self.nnz.shape[0])

    @property
    def w(self) -> int:
        return int(self.val.shape[1])

    @staticmethod
    def empty(n: int, w: int, device="cuda") -> "Mat":
        torch = _torch()
        return Mat(torch.zeros((n, w), dtype=torch.float64, device=device),
                   torch.zeros((n, w), dtype=torch.int32, device=device),
                   torch.zeros((n,), dtype=torch.int32, device=device))

    @staticmethod
    def from_host(e, device="cuda", w: int | None = None) -> "Mat":
        """Upload a synth.Ell (numpy) matrix; optional wider storage width."""
        torch = _torch()
        if w is not None and w != e.w:
            e = e.widened(w)
        return Mat(torch.from_numpy(e.val).to(device), torch.from_numpy(e.col).to(device),
                   torch.from_numpy(e.nnz).to(device))

    def to_host(self):
        from synth import Ell
        return Ell(self.val.cpu().numpy(), self.col.cpu().numpy(), self.nnz.cpu().numpy())

    def ref(self):
        return ctypes.byref(self.desc)


@dataclass
class SP2Result:
    status: int
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
    phases: dict
    iters: list = field(default_factory=list)


class Context:
    """One libellpack context bound to a device and a CUDA stream (torch's current one by default)."""

    def __init__(self, device: int = 0, stream=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2102_08505_b200 needs a CUDA device (no CPU fallback)")
        self.device = device
        with torch.cuda.device(device):
            s = stream if stream is not None else torch.cuda.current_stream(device)
        self.stream = s
        self._h = ctypes.c_void_p()
        _chk(lib().ellpack_ctx_create(device, ctypes.c_void_p(s.cuda_stream), ctypes.byref(self._h)),
             "ellpack_ctx_create")

    def close(self):
        if self._h:
            lib().ellpack_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key: int, value: int):
        _chk(lib().ellpack_ctx_set_option(self._h, key, int(value)), "ellpack_ctx_set_option")

    def kernel_launches(self) -> int:
        return int(lib().ellpack_ctx_kernel_launches(self._h))

    def last_launch(self) -> dict:
        """Geometry of the last row-kernel launch (ellpack_ctx_last_launch)."""
        a = (ctypes.c_int32 * 8)()
        _chk(lib().ellpack_ctx_last_launch(self._h, a), "ellpack_ctx_last_launch")
        return dict(path={5: "small", 4: "dense", 3: "ws", 2: "split", 1: "ring", 0: "general"}[a[0]], G=a[1], S=a[2], warps_per_cta=a[3],
                    grid=a[4],
                    smem_bytes=a[5], ctas_per_sm=a[6], hB=a[7])

    def host_syncs(self) -> int:
        """Blocking host synchronisations of the context stream so far (evidence counter)."""
        return int(lib().ellpack_ctx_host_syncs(self._h))

    def kernel_time(self):
        """(accumulated row-kernel ms, launches) since OPT_PROFILE was set."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        _chk(lib().ellpack_ctx_kernel_time(self._h, ctypes.byref(ms), ctypes.byref(n)), "ellpack_ctx_kernel_time")
        return ms.value, n.value

    def set_rows(self, r0: int, r1: int):
        _chk(lib().ellpack_ctx_set_rows(self._h, r0, r1), "ellpack_ctx_set_rows")

    def overflow_info(self):
        rows, req = ctypes.c_int64(), ctypes.c_int32()
        lib().ellpack_overflow_info(self._h, ctypes.byref(rows), ctypes.byref(req))
        return rows.value, req.value

    # ---- ops (return the status; raise on anything but OK / the listed soft statuses)
    def multiply(self, a: Mat, b: Mat, c: Mat, alpha: float, beta: float, threshold: float,
                 ok=(OK, ERR_OVERFLOW)) -> int:
        return _chk(lib().ellpack_multiply(self._h, a.ref(), b.ref(), c.ref(), alpha, beta, threshold),
                    "ellpack_multiply", ok)

    def multiply_x2(self, x: Mat, x2: Mat, threshold: float, ok=(OK, ERR_OVERFLOW)):
        tx, tx2 = ctypes.c_double(math.nan), ctypes.c_double(math.nan)
        st = _chk(lib().ellpack_multiply_x2(self._h, x.ref(), x2.ref(), threshold, ctypes.byref(tx),
                                            ctypes.byref(tx2)), "ellpack_multiply_x2", ok)
        return st, tx.value, tx2.value

    def add(self, a: Mat, b: Mat, alpha: float, beta: float, threshold: float, ok=(OK, ERR_OVERFLOW)) -> int:
        return _chk(lib().ellpack_add(self._h, a.ref(), b.ref(), alpha, beta, threshold), "ellpack_add", ok)

    def add_identity(self, a: Mat, beta: float, threshold: float, ok=(OK, ERR_OVERFLOW)) -> int:
        return _chk(lib().ellpack_add_identity(self._h, a.ref(), beta, threshold), "ellpack_add_identity", ok)

    def scale_add_identity(self, a: Mat, alpha: float, beta: float, threshold: float,
                           ok=(OK, ERR_OVERFLOW)) -> int:
        return _chk(lib().ellpack_scale_add_identity(self._h, a.ref(), alpha, beta, threshold),
                    "ellpack_scale_add_identity", ok)

    def trace(self, a: Mat) -> float:
        out = ctypes.c_double()
        _chk(lib().ellpack_trace(self._h, a.ref(), ctypes.byref(out)), "ellpack_trace")
        return out.value

    def fnorm_diff(self, a: Mat, b: Mat) -> float:
        out = ctypes.c_double()
        _chk(lib().ellpack_fnorm_diff(self._h, a.ref(), b.ref(), ctypes.byref(out)), "ellpack_fnorm_diff")
        return out.value

    def gershgorin(self, h: Mat):
        lo, hi = ctypes.c_double(), ctypes.c_double()
        _chk(lib().ellpack_gershgorin(self._h, h.ref(), ctypes.byref(lo), ctypes.byref(hi)), "ellpack_gershgorin")
        return lo.value, hi.value

    def sp2_run(self, h: Mat, nocc: int, tol: float, d: Mat, threshold: float = 0.0, max_iter: int = 100,
                min_iter: int = 20, stag_gate: float = 1e-3, bounds=None, on_overflow: int = SP2_GROW,
                max_width: int = 0, initial_width: int = 0, branch_rule: int = 0,
                ok=(OK, ERR_NOCONV, ERR_OVERFLOW)) -> SP2Result:
        o = SP2Opts()
        lib().sp2_opts_default(ctypes.byref(o))
        o.threshold, o.max_iter, o.min_iter, o.stag_gate = threshold, max_iter, min_iter, stag_gate
        if bounds is not None:
            o.emin, o.emax = bounds
        o.on_overflow, o.max_width, o.initial_width = on_overflow, max_width, initial_width
        o.branch_rule = branch_rule
        recs = (SP2IterRec * max(1, max_iter))()
        rep = SP2Report()
        rep.iters = ctypes.cast(recs, ctypes.POINTER(SP2IterRec))
        st = _chk(lib().sp2_run(self._h, h.ref(), nocc, tol, ctypes.byref(o), d.ref(), ctypes.byref(rep)),
                  "sp2_run", ok)
        n_rec = min(rep.iterations, max_iter)
        iters = [dict(trX=recs[k].trX, trS=recs[k].trS, e=recs[k].e, fnorm=recs[k].fnorm,
                      branch="SQUARE" if recs[k].branch == 0 else "EXPAND", width=recs[k].width,
                      required=recs[k].required, products=recs[k].products, frob2=recs[k].frob2,
                      products_exec=recs[k].products_exec,
                      regime="dense" if recs[k].regime == 1 else "sparse", step_ms=recs[k].step_ms)
                 for k in range(n_rec)]
        phases = dict(read_hamiltonian=rep.t_read_hamiltonian, init_misc=rep.t_init_misc,
                      sp2_loop_x2=rep.t_sp2_loop_x2, sp2_loop_norm=rep.t_sp2_loop_norm,
                      sp2_loop_misc=rep.t_sp2_loop_misc)
        return SP2Result(st, rep.iterations, STOP_NAMES.get(rep.stop_reason, "?"), rep.final_width, rep.regrows,
                         rep.emin, rep.emax, rep.trD, rep.overflow_rows, rep.required_width, rep.fail_iter,
                         phases, iters)

    def multiply_x2_host(self, x, x2, threshold: float, ok=(OK, ERR_OVERFLOW)):
        """End-to-end X^2 on HOST numpy/pinned-torch arrays (H2D + kernels + D2H inside the call).
        x, x2: objects with .val/.col/.nnz host arrays supporting __array_interface__ or torch CPU tensors."""
        def ptr(a):
            return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
        tx, tx2 = ctypes.c_double(math.nan), ctypes.c_double(math.nan)
        n, wx, wy = x.nnz.shape[0], x.val.shape[1], x2.val.shape[1]
        st = _chk(lib().ellpack_multiply_x2_host(self._h, n, wx, ptr(x.val), ptr(x.col), ptr(x.nnz), wy,
                                                 ptr(x2.val), ptr(x2.col), ptr(x2.nnz), threshold,
                                                 ctypes.byref(tx), ctypes.byref(tx2)),
                  "ellpack_multiply_x2_host", ok)
        return st, tx.value, tx2.value

    # ---- multi-GPU
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _chk(lib().ellpack_nccl_unique_id(buf), "ellpack_nccl_unique_id")
        return bytes(buf)

    def attach_nccl(self, nranks: int, rank: int, uid: bytes, row_begin: int, row_end: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _chk(lib().ellpack_ctx_attach_nccl(self._h, nranks, rank, buf, row_begin, row_end),
             "ellpack_ctx_attach_nccl")

    def multiply_x2_halo(self, x: Mat, x2: Mat, threshold: float, ok=(OK, ERR_OVERFLOW)):
        """X^2 of this rank's rows with the halo exchange of X overlapped with the interior rows (f1)."""
        tx, tx2 = ctypes.c_double(math.nan), ctypes.c_double(math.nan)
        st = _chk(lib().ellpack_multiply_x2_halo(self._h, x.ref(), x2.ref(), threshold, ctypes.byref(tx),
                                                 ctypes.byref(tx2)), "ellpack_multiply_x2_halo", ok)
        return st, tx.value, tx2.value

    def allgather_rows(self, m: Mat):
        _chk(lib().ellpack_allgather_rows(self._h, m.ref()), "ellpack_allgather_rows")

    def halo_rows(self, a: Mat, b: Mat | None = None):
        """Band-aware halo exchange (f1): the rows of b that this rank's rows of a reference."""
        _chk(lib().ellpack_halo_rows(self._h, a.ref(), (b or a).ref()), "ellpack_halo_rows")


def halo_plan(n: int, nranks: int, rank: int, per: int, need):
    """ellpack_halo_plan (host only): need = [(lo_q, hi_q)] per rank (inclusive) ->
    (sends, recvs), lists of (peer, row_begin, row_end)."""
    import numpy as np
    nd = np.ascontiguousarray(np.asarray(need, dtype=np.int64).reshape(-1))
    snd = np.zeros(3 * nranks, np.int64)
    rcv = np.zeros(3 * nranks, np.int64)
    ns, nr = ctypes.c_int32(), ctypes.c_int32()
    _chk(lib().ellpack_halo_plan(n, nranks, rank, per, nd.ctypes.data, ctypes.byref(ns), snd.ctypes.data,
                                 ctypes.byref(nr), rcv.ctypes.data), "ellpack_halo_plan")
    return ([tuple(int(x) for x in snd[3 * k:3 * k + 3]) for k in range(ns.value)],
            [tuple(int(x) for x in rcv[3 * k:3 * k + 3]) for k in range(nr.value)])


def row_split(r0: int, r1: int, h: int):
    """ellpack_row_split (host only): (interior, lower boundary, upper boundary) row ranges."""
    out = (ctypes.c_int64 * 6)()
    _chk(lib().ellpack_row_split(r0, r1, h, out), "ellpack_row_split")
    return (out[0], out[1]), (out[2], out[3]), (out[4], out[5])


def row_partition(n: int, nranks: int, align: int = 256):
    """Contiguous, equal, 256-aligned row blocks [r0, r1) per rank.
    Requires n % (align * nranks) == 0 for nranks > 1 (equal NCCL all-gather counts)."""
    if nranks == 1:
        return [(0, n)]
    if n % (align * nranks):
        raise ValueError(f"n={n} must be a multiple of {align}*{nranks} for a {nranks}-rank partition")
    per = n // nranks
    return [(r * per, (r + 1) * per) for r in range(nranks)]
