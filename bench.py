#!/usr/bin/env python
"""bench.py -- ELLPACK X^2 multiply + SP2 on B200 (BASELINE.json metric), one JSON line.

Headline (BASELINE.json configs[4], the largest single-GPU multiply, on which the north star's
">= 50% of HBM peak" target is stated):
    cfg5: X^2 of a random banded symmetric X, N=262144, M=256, tau=1e-5, FP64.
A "step" = one ellpack_multiply_x2 call (fused row kernel: window pre-pass, gather-accumulate,
drop/compact/write, trace partials; canonical trace reduction; status read-back) -- SURVEY §8a
rows a0..a4. With N > 1 ranks a step is ellpack_multiply_x2_halo: the band-aware halo exchange of
X's rows (NCCL send/recv of exactly the rows the rank's own rows reference, §8f-f1; BJ north_star
(3)) on a second stream while the rank's interior rows are computed, then its boundary rows
(strong scaling: total work fixed).

The same line carries the rest of BASELINE.json's metric ("SP2 iterations/sec at 1/2/4/8") and the
other configs' timings as sub-objects: "sp2" (cfg3 K = 10 and cfg4 K = 10 windows, SURVEY §8d "SP2
protocol"), "cfg1" (us per ABI call, launch-latency bound) and "cfg2" (C = alpha A B + beta C).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload x2|sp2] [--n N --m M] [--quick]

--gpus N without a launcher re-executes itself under torch.distributed.run with N ranks (one per
GPU); under a launcher WORLD_SIZE must equal N. --impl reference times the CPU oracle (oracle/, the
reference arm of this tier) on the host cores, on a bounded row sample of the same workload (rank 0
only under a launcher).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

HBM_FALLBACK_GBS = 6650.0
TAU5 = 1e-5


def workload_name(n: int, m: int, tau: float) -> str:
    """The one workload string both arms print (the driver compares them)."""
    return f"cfg5 X^2 N={n} M={m} tau={tau:g}"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def kernel_src_sha() -> str:
    """Hash of the row-kernel source: an ncu capture is only quoted for the kernel it measured."""
    h = hashlib.sha256()
    for f in ("spgemm.cu", "split.cu", "internal.cuh", "devutil.cuh"):
        h.update(open(os.path.join(ROOT, "paper_2102_08505_b200", "csrc", f), "rb").read())
    return h.hexdigest()[:16]


def ncu_capture(key: str):
    """DRAM bytes / L2 hit rates per launch of the row kernel from the committed ncu --set full
    capture (profiles/ncu_traffic.json), or (None, why) when that capture is of another kernel
    source than the one that just ran."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, "no capture"
    d = json.load(open(p)).get(key)
    if not d:
        return None, "no capture of this workload"
    if not isinstance(d, dict):
        return None, "capture predates kernel-source hashing"
    if d.get("src_sha") != kernel_src_sha():
        return None, f"capture {d.get('source')} is of kernel source {d.get('src_sha')}, not the current one"
    return d, d.get("source")


def microbench(name: str):
    """Measured co-bound peaks (tools/microbench.cu on a B200, profiles/r02_microbench.json)."""
    p = os.path.join(ROOT, "profiles", "r02_microbench.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get(name)


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML every 10 ms (the timed
    region of a default run is ~0.1 s), nvidia-smi every 0.2 s if NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, {reason names})
        self._stop = threading.Event()
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nvml = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        self.rows.append((float(sm), float(mx), {n for n, b in zip(self.NAMES, bits) if r & b}))

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        if out:
            r = [x.strip() for x in out.split(",")]
            num = lambda x: float(x) if x.replace(".", "").isdigit() else None  # noqa: E731
            self.rows.append((num(r[0]), num(r[1]),
                              {self.NAMES[k] for k in range(4) if len(r) > 3 + k and r[3 + k] == "Active"}))

    def _run(self):
        while not self._stop.wait(0.01 if self._nvml else 0.0):
            self._sample()
            if not self._nvml:
                self._stop.wait(0.2)

    def _sample(self):
        try:
            self._sample_nvml() if self._nvml else self._sample_smi()
        except Exception:
            pass

    def __enter__(self):
        if self._nvml:
            self._sample()  # the region's first instant (NVML is ~5 us a query)
        self._t.start()
        return self

    def __exit__(self, *a):
        if self._nvml:
            self._sample()  # and its last
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clocks unavailable"], "samples": 0}
        sm = [r[0] for r in self.rows if r[0] is not None]
        mx = [r[1] for r in self.rows if r[1] is not None]
        reasons = sorted(set().union(*[r[2] for r in self.rows]))
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml" if self._nvml else "nvidia-smi"}




def live_entries(e) -> int:
    return int(e.nnz.sum())


def x2_bytes(nnz_x: int, nnz_c: int, n: int) -> int:
    """Compulsory HBM bytes of one X^2: 12 B per stored input entry read once,
    12 B per kept output entry written once, 4 B per row_nnz read and written."""
    return 12 * (nnz_x + nnz_c) + 8 * n


def lsu_floor(X, P: int, nnz_c: int, sm_mhz, num_sms: int = 148, slot_bytes: int = 4) -> dict:
    """The ring kernel's L1/LSU data-pipe floor, in SM-cycles: per product a 64-bit
    LDS + STS on the ring -- a conflict-free 32-lane STS.64 takes 2 cycles, an LDS.64 1 (loads are
    served at 256 B/clk: tools/bank_model.cu, profiles/r02_bank_model.log), so 3 cycles per 32
    products -- and a (8 + slot_bytes)-byte B record gather (one 128-byte wavefront per cycle);
    per output-span column one read-and-clear (2 per 32); per kept entry 12 bytes stored.
    Conflict-free, unpadded counts: the floor a perfect schedule would meet."""
    nnz = X.nnz.astype(np.int64)
    live = nnz > 0
    rows = np.flatnonzero(live)
    first = X.col[rows, 0].astype(np.int64)
    last = X.col[rows, nnz[rows] - 1].astype(np.int64)
    hB = int(max((rows - first).max(initial=0), (last - rows).max(initial=0)))
    lo = np.maximum(0, first - hB) & ~31
    hi = (np.minimum(X.n - 1, last + hB) + 32) & ~31
    cols = int((hi - lo).sum())
    wf = P * (3 / 32 + (8 + slot_bytes) / 128) + cols * (2 / 32) + nnz_c * (12 / 128)
    if not sm_mhz:
        return {"wavefronts": wf, "floor_ms": None}
    return {"wavefronts": wf, "output_span_columns": cols, "sm_mhz": sm_mhz,
            "floor_ms": wf / (num_sms * sm_mhz * 1e6) * 1e3}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def round_up32(x: int) -> int:
    return ((x + 31) // 32) * 32


# ---------------------------------------------------------------------------- oracle arm

def oracle_sample(X, tau: float, budget_s: float):
    """Choose a bounded row sample of the X^2 workload for the oracle (as it stands): uniformly
    sampled rows of X, grown until one oracle call takes about budget_s / 4 seconds. The sample's
    output is stored at its required width (every kept entry is written, as in the GPU step).
    Returns (run, products, description, cores): run() executes the sample once (seconds)."""
    import oracle
    from synth import Ell
    n = X.n
    rows = 256
    rng = np.random.default_rng(0)
    while True:
        idx = np.sort(rng.choice(n, size=min(rows, n), replace=False))
        A = Ell.empty(n, X.w)
        A.val[idx] = X.val[idx]
        A.col[idx] = X.col[idx]
        A.nnz[idx] = X.nnz[idx]
        P = synth.products(A, X)
        t0 = time.perf_counter()
        r = oracle.multiply(A, X, Ell.empty(n, 2), 1.0, 0.0, tau)  # sizing call: required width
        dt = time.perf_counter() - t0
        if dt > budget_s / 5 or rows >= n:
            Y = Ell.empty(n, max(2, round_up32(r.required_width)))

            def run(A=A, Y=Y):
                t0 = time.perf_counter()
                rr = oracle.multiply(A, X, Y, 1.0, 0.0, tau)
                assert rr.status == oracle.OK
                return time.perf_counter() - t0

            desc = (f"{len(idx)} uniformly sampled rows of the same X^2 ({P} products per sample, output at "
                    f"the sample's required width {Y.w})")
            return run, P, desc, oracle.num_threads()
        rows = min(n, int(rows * max(2.0, (budget_s / 5) / max(dt, 1e-3))))


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    X = synth.cfg5(args.n, args.m)
    run, P, desc, cores = oracle_sample(X, TAU5, args.ref_budget)
    for _ in range(args.warmup):
        run()
    times = [run() for _ in range(args.steps)]
    dt = statistics.median(times)
    gflops = 2.0 * P / dt / 1e9
    line = {
        "impl": "reference", "metric": "ELLPACK X^2 multiply GFLOP/s", "value": gflops, "unit": "GFLOP/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (synth.cfg5, seed 5)",
        "config": {"workload": workload_name(args.n, args.m, TAU5), "sample_products": P},
        "cpu_baseline": {"value": gflops, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": gflops, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm

def _init(args):
    """Process group (N > 1), device, context, NCCL communicator over the given rows."""
    import torch

    import paper_2102_08505_b200 as eb
    from paper_2102_08505_b200 import multirank as mr

    ws, rank, local = mr.dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        mr.init_process_group("nccl", device=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    eb.build()
    return ws, rank, torch.cuda.current_device()


def _comm_ctx(eb, mr, dev, ws, rank, n):
    ctx = eb.Context(dev)
    if ws > 1:
        uid = mr.broadcast_bytes(eb.Context.nccl_unique_id() if rank == 0 else None)
        r0, r1 = mr.rank_rows(n, ws, rank)
        ctx.attach_nccl(ws, rank, uid, r0, r1)
    return ctx


def check_ranks_bitwise(eb, mr, dev, ws, rank):
    """N > 1: before timing, the rank's rows of a small cfg5 X^2 computed through the communicator
    (halo exchange + own rows) must equal a one-rank computation bit for bit (§8c-c12)."""
    import torch
    import torch.distributed as dist
    X = synth.cfg5(32768, 64)
    solo = eb.Context(dev)
    x1 = eb.Mat.from_host(X)
    y1 = eb.Mat.empty(X.n, 832)
    st1, tx1, tx21 = solo.multiply_x2(x1, y1, TAU5)
    solo.close()
    ctx = _comm_ctx(eb, mr, dev, ws, rank, X.n)
    x = eb.Mat.from_host(X)
    r0, r1 = mr.rank_rows(X.n, ws, rank)
    keep = torch.zeros(X.n, dtype=torch.bool, device="cuda")
    keep[r0:r1] = True
    x.nnz.masked_fill_(~keep, 0)  # this rank holds only its own rows; the halo brings the rest
    ctx.halo_rows(x)
    y = eb.Mat.empty(X.n, 832)
    st, tx, tx2 = ctx.multiply_x2(x, y, TAU5)
    live = torch.arange(832, device="cuda")[None, :] < y1.nnz[r0:r1, None]
    ok = (st == st1 == eb.OK and (tx, tx2) == (tx1, tx21) and torch.equal(y.nnz[r0:r1], y1.nnz[r0:r1])
          and torch.equal(y.col[r0:r1][live], y1.col[r0:r1][live])
          and torch.equal(y.val[r0:r1][live].view(torch.int64), y1.val[r0:r1][live].view(torch.int64)))
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(flag)
    ctx.close()
    if int(flag.item()):
        raise SystemExit(f"bench.py: P={ws} result differs from P=1 on cfg5 N=32768 M=64 (rank {rank}: ok={ok})")
    return True


def time_sp2(eb, mr, dev, ws, rank, cfg: int, K: int, steps: int, warmup: int):
    """SP2 iterations/sec over a fixed K-iteration GROW window (SURVEY §8d "SP2 protocol"): one timed
    call = one sp2_run of K iterations, CUDA events on the context stream, max over ranks."""
    import torch
    H, cf = (synth.cfg3(), synth.CFG3) if cfg == 3 else (synth.cfg4(), synth.CFG4)
    n = H.n
    torch.cuda.empty_cache()  # (the dense regime's arrays are sized against the free memory)
    ctx = _comm_ctx(eb, mr, dev, ws, rank, n)
    h = eb.Mat.from_host(H)
    d = eb.Mat.empty(n, min(n + (n & 1), 8192))
    stream = torch.cuda.current_stream()
    run = lambda: ctx.sp2_run(h, cf["nocc"], cf["tol"], d, threshold=cf["threshold"], max_iter=K)  # noqa: E731
    for _ in range(max(1, warmup)):
        r = run()
    torch.cuda.synchronize()
    s0, l0 = ctx.host_syncs(), ctx.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        r = run()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if ws > 1:
        ms = mr.max_over_ranks(ms, device="cuda")
    syncs = (ctx.host_syncs() - s0) / steps
    launches = (ctx.kernel_launches() - l0)
    ctx.close()
    P = sum(it["products"] for it in r.iters)
    out = {"workload": f"cfg{cfg} SP2 N={n} tau={cf['threshold']:g} window K={K} GROW", "iterations": r.iterations,
           "stop": r.stop, "final_width": r.final_width, "ms_per_window": ms, "iterations_per_s": r.iterations / (ms * 1e-3),
           "products": P, "gflops_effective": 2.0 * P / (ms * 1e-3) / 1e9,
           "host_syncs_per_iteration": syncs / max(r.iterations, 1), "gpu_launches": launches,
           "symmetric_step": True,
           "regimes": "".join("D" if it["regime"] == "dense" else "s" for it in r.iters),
           "per_iteration": sp2_per_iteration(r.iters)}
    out.update(sp2_rooflines(r.iters))
    return out


def sp2_per_iteration(iters):
    """SURVEY §8d "SP2 protocol": per iteration the width, P_n, the step's device time, GFLOP/s, e_n,
    the branch and the regime (compact arrays)."""
    return {"width": [it["width"] for it in iters], "products": [it["products"] for it in iters],
            "step_ms": [round(it["step_ms"], 4) if it["step_ms"] == it["step_ms"] else None for it in iters],
            "gflops": [round(2.0 * it["products"] / (it["step_ms"] * 1e-3) / 1e9, 1)
                       if it["step_ms"] == it["step_ms"] and it["step_ms"] > 0 else None for it in iters],
            "e": [it["e"] for it in iters], "branch": "".join("S" if it["branch"] == "SQUARE" else "E" for it in iters),
            "regime": "".join("D" if it["regime"] == "dense" else "s" for it in iters)}


def sp2_rooflines(iters):
    """Per-regime rooflines of an SP2 run from its per-step device times (sp2_iter_rec.step_ms): the
    sparse steps' executed products against the measured random FP64 shared-RMW peak (the
    accumulator's bound), the dense steps' GEMM FMAs against the measured FP64 FMA peak; "roofline"
    is the regime that took more of the time."""
    rmw, fma = microbench("smem_rmw_f64_random_peak"), microbench("fp64_fma")
    sp = [it for it in iters if it["regime"] != "dense"]
    de = [it for it in iters if it["regime"] == "dense"]
    sp_ms = sum(it["step_ms"] for it in sp)
    de_ms = sum(it["step_ms"] for it in de)
    out = {"products_executed": sum(it["products_exec"] for it in sp), "dense_fmas_executed":
           sum(it["products_exec"] for it in de), "sparse_step_ms": sp_ms, "dense_step_ms": de_ms}
    r_s = r_d = None
    if sp and sp_ms > 0:
        a = out["products_executed"] / (sp_ms * 1e-3) / 1e9
        r_s = {"bound": "smem_rmw", "achieved": a, "unit": "Gupd/s", "peak": rmw["Gupd_per_s"] if rmw else None,
               "frac": a / rmw["Gupd_per_s"] if rmw else None, "steps": len(sp),
               "peak_source": "tools/microbench.cu random-address FP64 smem RMW, best occupancy "
                              "(profiles/r02_microbench.json)"}
    if de and de_ms > 0:
        a = 2.0 * out["dense_fmas_executed"] / (de_ms * 1e-3) / 1e12
        r_d = {"bound": "fp64", "achieved": a, "unit": "TFLOP/s", "peak": fma["TFLOPs"] if fma else None,
               "frac": a / fma["TFLOPs"] if fma else None, "steps": len(de),
               "note": "step time includes densify and epilogue; FMAs of the occupied k blocks",
               "peak_source": "tools/microbench.cu FP64 FMA throughput (profiles/r02_microbench.json)"}
    out["roofline_sparse_steps"] = r_s
    out["roofline_dense_steps"] = r_d
    out["roofline"] = r_d if (r_d and de_ms >= sp_ms) else r_s
    return out


def time_sp2_full(eb, dev, cfg: int = 3, max_iter: int = 100):
    """BASELINE configs[2] as named: SP2 on cfg3 to the stop rule (GROW, max_iter 100), one GPU, the
    automatic regime -- sparse row kernels while the iterates are narrow, the dense GEMM once they fill
    in (ELLPACK_OPT_DENSE 0). One warm-up run of 30 iterations (workspace, dense buffers), then one
    timed run, CUDA events on the context stream."""
    import torch
    H, cf = synth.cfg3(), synth.CFG3
    n = H.n
    ctx = eb.Context(dev)
    h = eb.Mat.from_host(H)
    d = eb.Mat.empty(n, n + (n & 1))
    ctx.sp2_run(h, cf["nocc"], cf["tol"], d, threshold=cf["threshold"], max_iter=30)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0 = ctx.host_syncs()
    e0.record(stream)
    r = ctx.sp2_run(h, cf["nocc"], cf["tol"], d, threshold=cf["threshold"], max_iter=max_iter)
    e1.record(stream)
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) * 1e-3
    syncs = ctx.host_syncs() - s0
    ctx.close()
    dense = [it for it in r.iters if it["regime"] == "dense"]
    out = {"workload": f"cfg3 SP2 N={n} tau={cf['threshold']:g} tol={cf['tol']:g} to the stop rule "
                       f"(max_iter {max_iter}), GROW, automatic regime",
           "iterations": r.iterations, "stop": r.stop, "final_width": r.final_width, "seconds": sec,
           "iterations_per_s": r.iterations / sec, "host_syncs_per_iteration": syncs / max(r.iterations, 1),
           "regimes": "".join("D" if it["regime"] == "dense" else "s" for it in r.iters),
           "dense_iterations": len(dense), "products": sum(it["products"] for it in r.iters),
           "round1_seconds": 51.18, "round1_source": "profiles/r01_sp2_full_cfg3.json (sparse kernels only)",
           "per_iteration": sp2_per_iteration(r.iters)}
    out.update(sp2_rooflines(r.iters))
    return out


def time_dense_gemm(eb, dev, n: int = 8192, reps: int = 5):
    """The dense regime's GEMM (csrc/dense.cu) on its own: X^2 of a filled, bitwise-symmetric N x N
    matrix (seeded N(0, 0.01)), ELLPACK_OPT_DENSE 2: symmetric tiles (T (T + 1) / 2 of 128 x 128,
    every k block non-empty), the GEMM's device time by CUDA events around its launch
    (ELLPACK_OPT_PROFILE), against the measured FP64 FMA peak (profiles/r02_microbench.json)."""
    import numpy as np
    import torch
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) * 0.01
    a = (a + a.T) * 0.5
    X = synth.Ell(val=np.ascontiguousarray(a), col=np.tile(np.arange(n, dtype=np.int32), (n, 1)),
                  nnz=np.full(n, n, dtype=np.int32))
    del a
    ctx = eb.Context(dev)
    ctx.set_option(eb.OPT_DENSE, 2)
    x = eb.Mat.from_host(X)
    y = eb.Mat.empty(n, n)
    for _ in range(2):
        ctx.multiply_x2(x, y, 0.0)
    torch.cuda.synchronize()
    ctx.set_option(eb.OPT_DENSE, 2)
    ctx.set_option(eb.OPT_PROFILE, 1)
    t0 = time.perf_counter()
    for _ in range(reps):
        st, _, _ = ctx.multiply_x2(x, y, 0.0)
    dt = (time.perf_counter() - t0) / reps
    kms, kn = ctx.kernel_time()
    path = ctx.last_launch()["path"]
    ctx.close()
    T = n // 128
    fmas = T * (T + 1) // 2 * 128 * 128 * n
    tf = 2.0 * fmas / (kms / kn * 1e-3) / 1e12
    mb = microbench("fp64_fma")
    return {"workload": f"X^2 of a filled symmetric N={n} matrix, dense regime forced (symmetric tiles)",
            "status": st, "path": path, "ms_per_call": dt * 1e3, "gemm_ms": kms / kn, "fmas": fmas,
            "roofline": {"bound": "fp64", "achieved": tf, "unit": "TFLOP/s",
                         "peak": mb["TFLOPs"] if mb else None, "frac": tf / mb["TFLOPs"] if mb else None,
                         "peak_source": "tools/microbench.cu FP64 FMA throughput (profiles/r02_microbench.json)"},
            "full_product_equivalent_tflops": 2.0 * n ** 3 / (kms / kn * 1e-3) / 1e12}


def time_sp2_small(eb, dev, reps: int, which: str = "cfg1"):
    """SP2 on a cfg1-sized H, to the stop rule (nocc = N/2, tau = 1e-5, tol = 1e-8): us per iteration
    with the host loop (one host synchronisation per iteration) and with the device-resident loop
    (one CUDA-graph launch per run), the same bits either way. which = "cfg1":
    BASELINE configs[0]'s matrix (N = 512) as H -- gapless, its iterates fill the 512 x 512 matrix, so
    an iteration is a dense-ish 512^3 product; "soft_matter": the paper's gapped soft-matter model H
    at N = 512, whose iterates stay sparse -- the launch-latency-bound case."""
    import torch
    if which == "cfg1":
        H = synth.cfg1()
        out = {"workload": "SP2 on cfg1's X as H: N=512 nocc=256 tau=1e-05 tol=1e-08, to the stop rule"}
    else:
        H = synth.model_hamiltonian(512, "soft_matter", tau_store=1e-5)
        out = {"workload": "SP2 on the soft-matter model H: N=512 nocc=256 tau=1e-05 tol=1e-08, to the stop rule"}
    n = H.n
    ref = None
    # automatic regime (dense GEMM steps once filled: the host loop switches per step, the device loop
    # runs every step dense at N <= 1024), and the device loop on the sparse kernels only (round 2's first)
    for name, loop, dense in (("host_loop", 1, 0), ("device_loop", 2, 0), ("device_loop_sparse_only", 2, 1)):
        ctx = eb.Context(dev)
        ctx.set_option(eb.OPT_SP2_DEVICE_LOOP, loop)
        ctx.set_option(eb.OPT_DENSE, dense)
        h = eb.Mat.from_host(H)
        d = eb.Mat.empty(n, n)
        run = lambda: ctx.sp2_run(h, n // 2, 1e-8, d, threshold=1e-5, max_iter=100)  # noqa: E731
        for _ in range(3):
            r = run()
        torch.cuda.synchronize()
        s0 = ctx.host_syncs()
        t0 = time.perf_counter()
        for _ in range(reps):
            r = run()
        dt = (time.perf_counter() - t0) / reps
        out[name] = {"us_per_iteration": dt * 1e6 / r.iterations, "us_per_run": dt * 1e6, "iterations": r.iterations,
                     "stop": r.stop, "host_syncs_per_run": (ctx.host_syncs() - s0) / reps,
                     "dense_iterations": sum(it["regime"] == "dense" for it in r.iters)}
        key = (r.iterations, r.trD, tuple(it["e"] for it in r.iters))
        out[name]["same_as_host_loop"] = None if ref is None else key == ref
        ref = ref or key
        ctx.close()
    return out


def time_sweep(eb, dev, reps: int):
    """BASELINE configs[4]'s sweep, N in {32768, 131072, 262144} x M in {64, 128, 256} (one GPU): per
    point the X^2 step time (CUDA events around the ABI call), the row kernel's time and its HBM
    roofline fraction (compulsory bytes / kernel time / measured peak)."""
    import torch
    hbm_peak, _ = peaks()
    out = []
    for n in (32768, 131072, 262144):
        for m in (64, 128, 256):
            X = synth.cfg5(n, m)
            ctx = eb.Context(dev)
            x = eb.Mat.from_host(X)
            y = eb.Mat.empty(n, m)
            st, _, _ = ctx.multiply_x2(x, y, TAU5)
            w = round_up32(ctx.overflow_info()[1]) if st == eb.ERR_OVERFLOW else m
            del y
            y = eb.Mat.empty(n, w)
            for _ in range(2):
                ctx.multiply_x2(x, y, TAU5)
            torch.cuda.synchronize()
            ctx.set_option(eb.OPT_PROFILE, 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                ctx.multiply_x2(x, y, TAU5)
            e1.record()
            torch.cuda.synchronize()
            kms, kn = ctx.kernel_time()
            kms /= max(kn, 1)
            ms = e0.elapsed_time(e1) / reps
            P = synth.products(X, X)
            Bc = x2_bytes(live_entries(X), int(y.nnz.sum().item()), n)
            launch = ctx.last_launch()
            out.append({"n": n, "m": m, "out_width": w, "ms_per_step": ms, "kernel_ms": kms,
                        "gflops": 2.0 * P / (ms * 1e-3) / 1e9, "hbm_frac": Bc / (kms * 1e-3) / 1e9 / hbm_peak,
                        "path": launch["path"], "G": launch["G"], "S": launch["S"], "rows_per_sm": launch["ctas_per_sm"]})
            ctx.close()
            del x, y
            torch.cuda.empty_cache()
    return out


def time_cfg1(eb, dev, reps: int):
    """cfg1 (N = 512): us per ellpack_multiply_x2 call (incl. its status read-back), host clock over
    back-to-back calls, plus the device time of the same calls by CUDA events."""
    import torch
    X = synth.cfg1()
    ctx = eb.Context(dev)
    x = eb.Mat.from_host(X)
    y = eb.Mat.empty(X.n, 256)
    for _ in range(20):
        assert ctx.multiply_x2(x, y, TAU5)[0] == eb.OK
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0, s0 = ctx.kernel_launches(), ctx.host_syncs()
    e0.record()
    t0 = time.perf_counter()
    for _ in range(reps):
        ctx.multiply_x2(x, y, TAU5)
    dt = (time.perf_counter() - t0) / reps
    e1.record()
    torch.cuda.synchronize()
    out = {"workload": "cfg1 X^2 N=512 M=32 tau=1e-05 (out width 256)", "us_per_call": dt * 1e6,
           "device_us_per_call": e0.elapsed_time(e1) * 1e3 / reps, "calls": reps,
           "gpu_launches_per_call": (ctx.kernel_launches() - l0) / reps,
           "host_syncs_per_call": (ctx.host_syncs() - s0) / reps,
           "gflops": 2.0 * synth.products(X, X) / dt / 1e9}
    ctx.close()
    return out


def time_cfg2(eb, mr, dev, ws, rank, reps: int):
    """cfg2: C <- drop(alpha A B + beta C) in place, N = 16384, M = 128, at the required width;
    C_old is restored (outside the timed region) before every call."""
    import torch
    A, B, C = synth.cfg2()
    cf = synth.CFG2
    ctx = _comm_ctx(eb, mr, dev, ws, rank, A.n)
    a, b = eb.Mat.from_host(A), eb.Mat.from_host(B)
    c = eb.Mat.from_host(C)
    st = ctx.multiply(a, b, c, cf["alpha"], cf["beta"], cf["threshold"])
    assert st == eb.ERR_OVERFLOW
    w = round_up32(ctx.overflow_info()[1])
    c0 = eb.Mat.from_host(C, w=w)
    c = eb.Mat.from_host(C, w=w)
    ms = []
    for k in range(reps + 3):
        c.val.copy_(c0.val), c.col.copy_(c0.col), c.nnz.copy_(c0.nnz)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert ctx.multiply(a, b, c, cf["alpha"], cf["beta"], cf["threshold"]) == eb.OK
        e1.record()
        torch.cuda.synchronize()
        if k >= 3:
            ms.append(e0.elapsed_time(e1))
    t = statistics.median(ms)
    if ws > 1:
        t = mr.max_over_ranks(t, device="cuda")
    P = synth.products(A, B)
    ctx.close()
    return {"workload": f"cfg2 C=aAB+bC N=16384 M=128 a=1 b=0.5 tau=1e-06 (out width {w})", "ms_per_call": t,
            "gflops": 2.0 * P / (t * 1e-3) / 1e9, "calls": reps}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2102_08505_b200 as eb
    from paper_2102_08505_b200 import multirank as mr

    ws, rank, dev = _init(args)
    ranks_checked = check_ranks_bitwise(eb, mr, dev, ws, rank) if ws > 1 else None
    ctx = _comm_ctx(eb, mr, dev, ws, rank, args.n)
    if args.window:
        ctx.set_option(eb.OPT_WINDOW, args.window)
    if args.warps:
        ctx.set_option(eb.OPT_WARPS, args.warps)
    tau = TAU5
    X = synth.cfg5(args.n, args.m)
    n = X.n
    P = synth.products(X, X)
    x = eb.Mat.from_host(X)
    # reading R2: the literal width M overflows; the first call reports the required width
    y = eb.Mat.empty(n, args.m)
    st, _, _ = ctx.multiply_x2(x, y, tau)
    assert st == eb.ERR_OVERFLOW
    _, req = ctx.overflow_info()
    w_out = round_up32(req)
    del y
    y = eb.Mat.empty(n, w_out)
    stream = torch.cuda.current_stream()

    def step():
        if ws > 1:
            # the rows of X this rank's rows reference travel by NCCL on a second stream while the
            # interior rows are computed (band-aware halo overlapped, §8f-f1)
            return ctx.multiply_x2_halo(x, y, tau)
        return ctx.multiply_x2(x, y, tau)

    for _ in range(max(3, args.warmup)):
        s, tx, tx2 = step()
        assert s == eb.OK
    nnz_c = int(y.nnz.sum().item())
    launch = ctx.last_launch()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.kernel_launches()
    ctx.set_option(eb.OPT_PROFILE, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms_total = e0.elapsed_time(e1)
    kern_ms, kern_n = ctx.kernel_time()
    ctx.set_option(eb.OPT_PROFILE, 0)
    launches = ctx.kernel_launches() - launches0
    if ws > 1:
        ms_total = mr.max_over_ranks(ms_total, device="cuda")
        dist.barrier()
    ms_step = ms_total / args.steps
    gflops = 2.0 * P / (ms_step * 1e-3) / 1e9
    Bc = x2_bytes(live_entries(X), nnz_c, n)
    hbm_peak, peak_src = peaks()
    kern_avg = kern_ms / max(kern_n, 1)
    # with N > 1 ranks, exchange-inclusive (the step: halo + every launch, max over ranks)
    # and multiply-only (the row kernels alone, max over ranks) reported separately
    multi = None
    if ws > 1:
        multi = {"exchange_inclusive_ms_per_step": ms_step,
                 "row_kernels_ms_per_step_max_over_ranks": mr.max_over_ranks(kern_ms / args.steps, device="cuda"),
                 "halo": "band-aware, ncclSend/ncclRecv on a second stream, overlapped with the interior rows"}
    bytes_launch = Bc / ws  # equal row blocks: the rank's share of the compulsory bytes
    achieved = bytes_launch / (kern_avg * 1e-3) / 1e9
    cap, cap_src = ncu_capture(f"x2_n{n}_m{args.m}")
    kname = {"ws": f"ell::row_ws_kernel<G={launch['G']}> (accumulator + emitter warps, ring S={launch['S']}, "
                   f"{launch['ctas_per_sm']} rows/SM)",
             "split": f"ell::row_split_kernel<W={launch['warps_per_cta']},G={launch['G']}> (ring S={launch['S']}, "
                      f"{launch['ctas_per_sm']} rows/SM)",
             "ring": f"ell::row_fast_kernel<G={launch['G']}> (ring S={launch['S']}, {launch['ctas_per_sm']} CTAs/SM)",
             "general": "ell::row_general_kernel"}[launch["path"]]

    # ---- end to end through the host-buffer ABI call (H2D of X + kernels + D2H of the rank's X^2 rows)
    e2e = None
    del y
    torch.cuda.empty_cache()
    if not args.no_e2e:
        hx = {k: torch.from_numpy(getattr(X, k)).pin_memory() for k in ("val", "col", "nnz")}
        hy = {"val": torch.empty((n, w_out), dtype=torch.float64).pin_memory(),
              "col": torch.empty((n, w_out), dtype=torch.int32).pin_memory(),
              "nnz": torch.empty((n,), dtype=torch.int32).pin_memory()}

        class _H:
            pass
        hxo, hyo = _H(), _H()
        for k in hx:
            setattr(hxo, k, hx[k])
            setattr(hyo, k, hy[k])
        ctx.multiply_x2_host(hxo, hyo, tau)  # warm (allocates the device scratch)
        torch.cuda.synchronize()
        k_e2e = max(1, min(args.steps, 3))
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            ctx.multiply_x2_host(hxo, hyo, tau)
        dt = (time.perf_counter() - t0) / k_e2e
        if ws > 1:
            dt = mr.max_over_ranks(dt, device="cuda")
        h2d = sum(t.numel() * t.element_size() for t in hx.values()) * ws
        d2h = sum(t.numel() * t.element_size() for t in hy.values())  # every rank brings back its rows
        e2e = {"value": 2.0 * P / dt / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3,
               "what": "ellpack_multiply_x2_host: pinned host X -> device, X^2, padded X^2 rows -> pinned host"}
        del hx, hy, hxo, hyo
    clocks = clk.summary()
    ctx.close()
    del x
    torch.cuda.empty_cache()

    # ---- the rest of the metric: SP2 windows, cfg1 latency, cfg2
    sp2 = cfg1 = cfg2 = sweep = dense_gemm = None
    if not args.quick:
        sp2 = {"cfg3": time_sp2(eb, mr, dev, ws, rank, 3, 10, 3, 1),
               "cfg4": time_sp2(eb, mr, dev, ws, rank, 4, 10, 2, 1)}
        if ws == 1:
            sp2["cfg3_full"] = time_sp2_full(eb, dev)
            sp2["cfg1_sized"] = time_sp2_small(eb, dev, 20, "cfg1")
            sp2["soft_matter_512"] = time_sp2_small(eb, dev, 50, "soft_matter")
        cfg1 = time_cfg1(eb, dev, 300) if ws == 1 else {"skipped": "N=512 is not divisible into 256-row blocks (R17)"}
        sweep = time_sweep(eb, dev, 5) if ws == 1 else None
        dense_gemm = time_dense_gemm(eb, dev) if ws == 1 else None
        cfg2 = time_cfg2(eb, mr, dev, ws, rank, 10)

    # ---- CPU oracle beside it (rank 0, N=1 only, bounded sample)
    cpu = None
    if not args.no_cpu_baseline and ws == 1 and rank == 0:
        run, Ps, desc, cores = oracle_sample(X, tau, args.ref_budget)
        dt = statistics.median([run() for _ in range(3)])
        cpu = {"value": 2.0 * Ps / dt / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "sample": desc}

    lsu_pipe = None
    if ws == 1 and launch["path"] in ("ring", "split", "ws"):
        lsu_pipe = lsu_floor(X, P, nnz_c, clocks.get("sm_mhz"), torch.cuda.get_device_properties(dev).multi_processor_count,
                             slot_bytes=2 if launch["path"] in ("split", "ws") else 4)
        if lsu_pipe.get("floor_ms"):
            lsu_pipe["frac"] = lsu_pipe["floor_ms"] / kern_avg
    if rank == 0:
        line = {
            "metric": "ELLPACK X^2 multiply GFLOP/s", "value": gflops, "unit": "GFLOP/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (synth.cfg5, seed 5; BASELINE configs[4] recipe, SURVEY §8d)",
            "config": {"workload": workload_name(n, args.m, tau), "products": P,
                       "out_width": w_out, "nnz_x": live_entries(X), "nnz_x2": nnz_c,
                       "l2": "inputs larger than L2 (X 0.8 GB padded, X^2 16 GB)",
                       "parallelism": f"row-blocks x{ws} + band-aware halo" if ws > 1 else "1 GPU"},
            "hbm_gbs_algorithmic": Bc / (ms_step * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": (cap or {}).get("dram_bytes"),
                         "traffic_source": cap_src, "peak_source": peak_src,
                         "l2_hit_pct": (cap or {}).get("l2_hit_pct"),
                         "kernel": kname, "launch": launch, "kernel_ms_avg": kern_avg,
                         "algorithmic_bytes_per_launch": bytes_launch,
                         "lsu_pipe": lsu_pipe},
            "sp2": sp2, "cfg1": cfg1, "cfg2": cfg2, "cfg5_sweep": sweep, "dense_gemm": dense_gemm,
            "multi_gpu": multi,
            "ranks_bitwise_vs_1": ranks_checked,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------------- SP2 window

def run_sp2(args):
    """SP2 iterations/sec (BASELINE metric, second half) on cfg3 or cfg4 over a fixed window of K
    iterations, or on the paper's model Hamiltonian to the stop rule (GROW policy; SURVEY §8d "SP2
    protocol"): one step = one sp2_run call, timed with CUDA events on the context stream; the CPU
    oracle runs the same window beside it (rank 0, N = 1)."""
    import torch

    import paper_2102_08505_b200 as eb
    from paper_2102_08505_b200 import multirank as mr

    ws, rank, dev = _init(args)
    if args.sp2_model:
        # the paper's own gapped SP2 workloads, run to the stop rule
        H = synth.model_hamiltonian(args.sp2_n, args.sp2_model, tau_store=1e-5)
        cf = dict(nocc=args.sp2_n // 2, tol=1e-8, threshold=1e-5)
    elif args.sp2_cfg == 3:
        H, cf = synth.cfg3(), synth.CFG3
    else:
        H, cf = synth.cfg4(), synth.CFG4
    n = H.n
    ctx = _comm_ctx(eb, mr, dev, ws, rank, n)
    if args.general_window:
        ctx.set_option(eb.OPT_GENERAL_WINDOW, args.general_window)
    if args.no_sp2_symmetric:
        ctx.set_option(eb.OPT_SP2_SYMMETRIC, 0)
    ctx.set_option(eb.OPT_DENSE, args.dense)
    K = args.sp2_iters
    h = eb.Mat.from_host(H)
    d = eb.Mat.empty(n, min(n + (n & 1), 8192))
    stream = torch.cuda.current_stream()

    def step():
        return ctx.sp2_run(h, cf["nocc"], cf["tol"], d, threshold=cf["threshold"], max_iter=K)

    for _ in range(max(1, args.warmup)):
        r = step()
    prods = sum(it["products"] for it in r.iters)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0, syncs0 = ctx.kernel_launches(), ctx.host_syncs()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            r = step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if ws > 1:
        ms = mr.max_over_ranks(ms, device="cuda")
    its = r.iterations
    syncs = (ctx.host_syncs() - syncs0) / args.steps
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        import oracle
        t0 = time.perf_counter()
        o = oracle.sp2(H, cf["nocc"], cf["tol"], oracle.SP2Opts(threshold=cf["threshold"], max_iter=K),
                       d_width=min(n + (n & 1), 8192))
        dt = time.perf_counter() - t0
        cpu = {"value": o.iterations / dt, "unit": "iterations/s", "cores": oracle.num_threads(), "kind": "oracle",
               "sample": f"the same {K}-iteration window (stop {o.stop}, width {o.final_width})"}
    roof = sp2_rooflines(r.iters)
    if rank == 0:
        line = {
            "metric": "SP2 iterations/sec", "value": its / (ms * 1e-3), "unit": "iterations/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": (f"synthetic (synth.model_hamiltonian {args.sp2_model}, P:L419-433)" if args.sp2_model
                     else f"synthetic (synth.cfg{args.sp2_cfg}, SURVEY §8d)"),
            "config": {"workload": (f"{args.sp2_model} SP2 N={n} tau={cf['threshold']:g} max_iter={K} GROW"
                                    if args.sp2_model else
                                    f"cfg{args.sp2_cfg} SP2 N={n} tau={cf['threshold']:g} window K={K} GROW"),
                       "iterations": its, "stop": r.stop, "final_width": r.final_width, "regrows": r.regrows,
                       "products": prods, "gflops_effective": 2.0 * prods / (ms * 1e-3) / 1e9,
                       "regimes": "".join("D" if it["regime"] == "dense" else "s" for it in r.iters),
                       "host_syncs_per_iteration": syncs / max(its, 1), "phases_s": r.phases,
                       "per_iteration": sp2_per_iteration(r.iters)},
            "roofline": roof["roofline"], "roofline_sparse_steps": roof["roofline_sparse_steps"],
            "roofline_dense_steps": roof["roofline_dense_steps"],
            "cpu_baseline": cpu, "gpu_launches": ctx.kernel_launches() - launches0, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=262144)
    ap.add_argument("--m", type=int, default=256)
    ap.add_argument("--window", type=int, default=0, help="dense-window doubles per row (0 = auto)")
    ap.add_argument("--warps", type=int, default=0, help="warps per CTA (0 = auto)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="headline only (no sp2 / cfg1 / cfg2 sub-objects)")
    ap.add_argument("--ref-budget", type=float, default=20.0, help="seconds of oracle work per sample")
    ap.add_argument("--workload", default="x2", choices=["x2", "sp2"],
                    help="x2: the headline cfg5 X^2 line (default); sp2: one SP2 line on cfg3/cfg4/a model H")
    ap.add_argument("--sp2-cfg", type=int, default=3, choices=[3, 4])
    ap.add_argument("--sp2-iters", type=int, default=10, help="SP2 window (max_iter)")
    ap.add_argument("--sp2-model", default=None, choices=["metal", "semiconductor", "soft_matter"],
                    help="SP2 on the paper's model Hamiltonian instead of cfg3/cfg4")
    ap.add_argument("--sp2-n", type=int, default=16384)
    ap.add_argument("--general-window", type=int, default=0, help="general-path window (0 = auto)")
    ap.add_argument("--dense", type=int, default=0, choices=(0, 1, 2),
                    help="SP2 workload: ELLPACK_OPT_DENSE (0 automatic regime, 1 sparse kernels only, 2 every step dense)")
    ap.add_argument("--no-sp2-symmetric", action="store_true",
                    help="SP2: compute whole rows even when H is symmetric (A/B of §8f-f4 ii)")
    args = ap.parse_args()
    if args.workload == "sp2" and args.impl == "reference":
        print(json.dumps({"impl": "reference", "unavailable": "--workload sp2 reports the oracle inline "
                          "(cpu_baseline); the reference arm is the x2 workload"}))
        return 0
    env_ws = os.environ.get("WORLD_SIZE")
    if env_ws is None and args.gpus > 1:
        # one process per GPU: re-execute under torch.distributed.run (rendezvous on 127.0.0.1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
               *sys.argv[1:]]
        return subprocess.call(cmd)
    if env_ws is not None and int(env_ws) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_ws}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    import torch
    if torch.cuda.device_count() < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} CUDA device(s) visible",
              file=sys.stderr)
        return 2
    if args.workload == "sp2":
        return run_sp2(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
