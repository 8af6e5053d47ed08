#!/usr/bin/env python
"""A/B compile-time variants of the dense GEMM (dense.cu macros): rebuild, dense parity subset, GEMM time
(tools/dense_time.py). Variants: "base" or NAME=VALUE[,NAME=VALUE]. The default build is restored."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2102_08505_b200 as eb  # noqa: E402

sizes = os.environ.get("SIZES", "4096 8192 12288").split()
for v in sys.argv[1:]:
    defs = () if v == "base" else tuple(v.split(","))
    eb.build(force=True, defines=defs)
    chk = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                          os.path.join(ROOT, "tests", "test_gpu_dense.py"), "-k", "x2_dense"],
                         capture_output=True, text=True, cwd=ROOT)
    ok = chk.stdout.strip().splitlines()[-1] if chk.stdout.strip() else chk.stderr[-200:]
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "dense_time.py"), *sizes],
                         capture_output=True, text=True, cwd=ROOT)
    for line in out.stdout.strip().splitlines():
        print(f"[{v}] {line}", flush=True)
    if out.returncode:
        print(f"[{v}] error {out.stderr[-300:]}", flush=True)
    print(f"[{v}] parity: {ok}", flush=True)
eb.build(force=True)
