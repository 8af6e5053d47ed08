#!/usr/bin/env python
"""A/B compile-time variants of the split-row ring kernel (split.cu macros) on the GPU box: for each
variant ("base" or NAME=VALUE[,NAME=VALUE]) rebuild, check bitwise parity on the ring-kernel tests,
time cfg5 X^2 (tools/ab_ring.py, ELLPACK_OPT_RING_KERNEL=2). The default build is restored at the end.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2102_08505_b200 as eb  # noqa: E402

sizes = os.environ.get("SIZES", "262144:256 262144:128").split()
for v in sys.argv[1:]:
    defs = () if v == "base" else tuple(v.split(","))
    eb.build(force=True, defines=defs)
    chk = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                          os.path.join(ROOT, "tests", "test_gpu_ring_kernels.py"), "-k", "split_w1"],
                         capture_output=True, text=True, cwd=ROOT)
    ok = chk.stdout.strip().splitlines()[-1] if chk.stdout.strip() else chk.stderr[-200:]
    for sz in sizes:
        n, m = sz.split(":")
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ab_ring.py"), "--n", n, "--m", m,
                              "--kernels", "2", "--reps", "10"], capture_output=True, text=True, cwd=ROOT).stdout
        for line in out.strip().splitlines():
            try:
                d = json.loads(line)
                print(f"[{v}] n={n} m={m} kernel {d['kernel_ms']:.3f} ms step {d['step_ms']:.3f} ms "
                      f"S={d['launch']['S']} ctas/SM={d['launch']['ctas_per_sm']}", flush=True)
            except Exception:
                print(f"[{v}] {line}", flush=True)
    print(f"[{v}] parity: {ok}", flush=True)
eb.build(force=True)
