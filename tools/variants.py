#!/usr/bin/env python
"""A/B the row kernel's compile-time tuning macros on the GPU box: for each variant
(a comma-separated list of NAME=VALUE defines, "base" = none) rebuild libellpack.so
with those -D flags, run a bitwise spot check against the in-tree oracle, and time
cfg5 X^2 with tools/sweep.py. The default build is restored at the end.
Usage: python tools/variants.py base ELL_STAGE_F=256 "ELL_STAGE_F=192,ELL_ROW_CHUNK=2"
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2102_08505_b200 as eb  # noqa: E402

sizes = os.environ.get("SIZES", "262144:256 131072:128").split()
sp2 = os.environ.get("SP2", "")  # e.g. "3 4:6": also time bench.py --workload sp2 --sp2-cfg C [--sp2-iters K]
tests_k = os.environ.get("TESTS_K", "x2 or multiply")
for v in sys.argv[1:]:
    defs = () if v == "base" else tuple(v.split(","))
    eb.build(force=True, defines=defs)
    chk = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                          "-k", tests_k], capture_output=True, text=True, cwd=ROOT)
    ok = chk.stdout.strip().splitlines()[-1] if chk.stdout.strip() else chk.stderr[-200:]
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sweep.py"), "--sizes", *sizes],
                         capture_output=True, text=True, cwd=ROOT).stdout
    for line in out.strip().splitlines():
        print(f"[{v}] {line}", flush=True)
    print(f"[{v}] parity: {ok}", flush=True)
    for spec in sp2.split():  # "C" or "C:K" (K = SP2 window)
        c, _, k = spec.partition(":")
        o = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "sp2", "--sp2-cfg", c,
                            "--steps", "2", "--warmup", "1"] + (["--sp2-iters", k] if k else [])
                           + (["--general-window", os.environ["GW"]] if os.environ.get("GW") else []),
                           capture_output=True, text=True, cwd=ROOT).stdout
        line = o.strip().splitlines()[-1] if o.strip() else "?"
        try:
            import json
            d = json.loads(line)
            line = f"sp2 cfg{c}: {d['value']:.2f} it/s  {d['config'].get('gflops', 0):.0f} GFLOP/s"
        except Exception:
            pass
        print(f"[{v}] {line}", flush=True)
eb.build(force=True)
