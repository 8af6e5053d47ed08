#!/usr/bin/env python
"""Dense-regime measurements (csrc/dense.cu):
  1. X^2 of a filled symmetric matrix (N = 4096, 8192) forced dense: ms per call and GEMM TFLOP/s
     (N^3 / 2 FMAs for the symmetric tiles), beside torch.matmul float64 (cuBLAS DGEMM) of the same size;
  2. SP2 on cfg1's X as H (N = 512) to the stop rule: automatic regime vs dense off (host and device loop);
  3. SP2 cfg3 (N = 12288) to the stop rule (max 100 iterations): automatic regime, per-iteration regime.
One JSON line per measurement."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2102_08505_b200 as eb  # noqa: E402
import synth  # noqa: E402

eb.build()
dev = torch.device("cuda:0")


def filled_sym(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)) * 0.01
    a = (a + a.T) * 0.5
    return synth.from_dense(a)


for n in (4096, 8192):
    X = filled_sym(n, n)
    ctx = eb.Context(0)
    ctx.set_option(eb.OPT_DENSE, 2)
    x = eb.Mat.from_host(X)
    y = eb.Mat.empty(n, n)
    for _ in range(2):
        st, _, _ = ctx.multiply_x2(x, y, 0.0)
    torch.cuda.synchronize()
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        ctx.multiply_x2(x, y, 0.0)
    dt = (time.perf_counter() - t0) / reps
    path = ctx.last_launch()["path"]
    ctx.close()
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(a, a)
    e1.record()
    torch.cuda.synchronize()
    tm = e0.elapsed_time(e1) / reps * 1e-3
    print(json.dumps({"what": "x2 dense forced, filled symmetric", "n": n, "status": st, "path": path,
                      "ms_per_call": dt * 1e3, "gemm_tflops_sym": n ** 3 / dt / 1e12,
                      "gemm_tflops_equiv_full": 2 * n ** 3 / dt / 1e12,
                      "cublas_dgemm_ms": tm * 1e3, "cublas_dgemm_tflops": 2 * n ** 3 / tm / 1e12}), flush=True)
    del x, y, a
    torch.cuda.empty_cache()


def run_sp2(H, nocc, tol, tau, dense, loop, max_iter=100):
    ctx = eb.Context(0)
    ctx.set_option(eb.OPT_DENSE, dense)
    ctx.set_option(eb.OPT_SP2_DEVICE_LOOP, loop)
    h = eb.Mat.from_host(H)
    d = eb.Mat.empty(H.n, H.n)
    ctx.sp2_run(h, nocc, tol, d, threshold=tau, max_iter=max_iter)  # warm-up (graphs, workspace)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = ctx.sp2_run(h, nocc, tol, d, threshold=tau, max_iter=max_iter)
    dt = time.perf_counter() - t0
    D = d.to_host()
    ctx.close()
    return r, dt, D


H = synth.cfg1()
ref = None
for dense, loop, name in ((0, 0, "auto"), (1, 1, "sparse host loop"), (1, 2, "sparse device loop")):
    r, dt, D = run_sp2(H, 256, 1e-8, 1e-5, dense, loop)
    same = None
    if ref is None:
        ref = D
    else:
        same = bool(np.array_equal(ref.nnz, D.nnz) and all(
            np.array_equal(ref.val[i, :ref.nnz[i]].view(np.uint64), D.val[i, :D.nnz[i]].view(np.uint64))
            for i in range(D.n)))
    print(json.dumps({"what": f"SP2 cfg1 X as H N=512, {name}", "iterations": r.iterations, "stop": r.stop,
                      "ms_per_run": dt * 1e3, "us_per_iteration": dt / r.iterations * 1e6,
                      "dense_iterations": sum(it["regime"] == "dense" for it in r.iters),
                      "same_D_as_auto": same}), flush=True)

H3 = synth.cfg3()
r, dt, D = run_sp2(H3, H3.n // 2, 1e-8, 1e-5, 0, 0)
print(json.dumps({"what": "SP2 cfg3 N=12288 to the stop rule, auto regime", "iterations": r.iterations,
                  "stop": r.stop, "seconds": dt, "iterations_per_s": r.iterations / dt,
                  "final_width": r.final_width,
                  "regimes": "".join("D" if it["regime"] == "dense" else "s" for it in r.iters),
                  "phases": r.phases}), flush=True)
