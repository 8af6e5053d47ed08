"""CPU-side checks of the C ABI boundary (no GPU compute calls).

* libellpack.so builds for sm_100a and loads on a machine without a GPU;
* it exports every function include/ellpack.h declares, and the Python binding's
  symbol list is exactly that set;
* the ctypes struct layouts match the C header (sizes/offsets via a tiny C probe);
* without a device, creating a context fails loudly (no CPU fallback);
* the row partition used by the multi-GPU path is 256-aligned and contiguous.
"""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ellpack.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s+\**([a-z_0-9]+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol(ellpack_lib):
    names = declared_functions()
    assert len(names) >= 20, names
    lib = ctypes.CDLL(ellpack_lib.build())
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(ellpack_lib.ABI_SYMBOLS) == names


def test_struct_layouts_match_header(ellpack_lib):
    probe = r"""
#include <stdio.h>
#include <stddef.h>
#include "ellpack.h"
int main(void) {
  printf("%zu %zu %zu %zu\n", sizeof(ellpack_desc), offsetof(ellpack_desc, val), offsetof(ellpack_desc, nnz), sizeof(sp2_opts));
  printf("%zu %zu %zu\n", sizeof(sp2_iter_rec), sizeof(sp2_report), offsetof(sp2_report, iters));
  printf("%zu %zu\n", offsetof(sp2_opts, on_overflow), offsetof(sp2_report, t_read_hamiltonian));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "p.c"), os.path.join(d, "p")
        open(src, "w").write(probe)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe])
        out = subprocess.check_output([exe]).decode().split()
    got = list(map(int, out))
    E = ellpack_lib
    want = [ctypes.sizeof(E.Desc), E.Desc.val.offset, E.Desc.nnz.offset, ctypes.sizeof(E.SP2Opts),
            ctypes.sizeof(E.SP2IterRec), ctypes.sizeof(E.SP2Report), E.SP2Report.iters.offset,
            E.SP2Opts.on_overflow.offset, E.SP2Report.t_read_hamiltonian.offset]
    assert got == want


def test_strerror_and_no_cpu_fallback(ellpack_lib):
    lib = ellpack_lib.lib()
    assert lib.ellpack_strerror(3).decode() == "output row exceeds ELLPACK width"
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(RuntimeError):
            ellpack_lib.Context(0)
        h = ctypes.c_void_p()
        assert lib.ellpack_ctx_create(0, None, ctypes.byref(h)) != 0


def test_row_partition(ellpack_lib):
    rp = ellpack_lib.row_partition
    assert rp(1000, 1) == [(0, 1000)]
    parts = rp(262144, 8)
    assert parts[0] == (0, 32768) and parts[-1][1] == 262144
    assert all(b0 % 256 == 0 for b0, _ in parts)
    assert all(p[1] == q[0] for p, q in zip(parts, parts[1:]))
    with pytest.raises(ValueError):
        rp(512, 8)
