// sp2_graph.cu -- device-resident SP2 control ("no extra pass"; P:L494-495
// "SP2 Loop Misc."): the per-iteration decisions of sp2_run (api.cu) made on the device, so that a
// whole SP2 loop is ONE launch of a CUDA graph with a conditional WHILE node and the host waits
// once per run instead of once per iteration.
//
// The control kernel applies exactly the host loop's rules, in the same binary64 expressions
// (reading R6/R19 branch rules, c10 (iv) GROW/FAIL, c10 (vi) stop rule), so the iterates, traces,
// branches and the stop iteration are bitwise those of the host loop and of the oracle.
#include "internal.cuh"
#include <math_constants.h>
#include "../../include/ellpack.h"

#include <cmath>

namespace ell {

__global__ void count_over_dev_kernel(const int32_t* nnz, int64_t n, const Sp2Dev* dev, int32_t* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t w = dev->wy;
    const unsigned m = __ballot_sync(FULL, i < n && nnz[i] > w);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(out, __popc(m));
}

cudaError_t launch_count_over_dev(const int32_t* nnz, int64_t n, const Sp2Dev* dev, int32_t* out, cudaStream_t s) {
    count_over_dev_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(nnz, n, dev, out);
    return cudaGetLastError();
}

__global__ void sp2_ctl_kernel(Sp2Dev* dev, const double* sums, const int32_t* status, int32_t* ovf,
                               unsigned long long* prod, sp2_iter_rec* rec, cudaGraphConditionalHandle cond) {
    Sp2Dev& d = *dev;
    const int it = d.it;
    const double trS = sums[0], trY = sums[1], nsq = sums[2];
    const int32_t kept = status[1];
    const int64_t products = (int64_t)*prod;
    const int32_t over = *ovf;
    *ovf = 0;
    *prod = 0ull;
    if (kept > d.wy) {
        // c10 (iv): FAIL, or GROW past max_width -> OVERFLOW(n); else the logical width grows
        if (d.on_overflow == SP2_FAIL || kept > d.maxw) {
            d.stop = SP2_OVERFLOWED;
            d.overflow_rows = over;
            d.required = kept;
            d.fail_iter = it;
            cudaGraphSetConditional(cond, 0u);
            return;
        }
        const int32_t r32 = (int32_t)((kept + 31) & ~31);
        d.wy = r32 < d.maxw ? r32 : d.maxw;
        d.regrows++;
    }
    const double e = __dsub_rn(d.trX, trS);
    sp2_iter_rec& r = rec[it];
    r.trX = d.trX;
    r.trS = trS;
    r.e = e;
    r.fnorm = sqrt(nsq);
    r.branch = d.branch;
    r.width = d.wy;
    r.required = kept;
    r.regime = dev->pad0;  // pad0: the regime of every step of this loop (1 dense), set by the host
    r.products = products;
    r.frob2 = d.closest ? d.t2 : 0.0;
    r.products_exec = products;
    r.step_ms = CUDART_NAN;  // one graph launch: no per-iteration timing
    if (d.closest) d.t2 = sums[3];
    d.trX = trY;
    int stop = -1;
    if (fabs(e) <= d.tol) stop = SP2_CONVERGED;
    else if (it + 1 >= d.min_iter && e <= d.stag_gate && !isnan(d.e2) && e >= d.e2) stop = SP2_STAGNATED;
    else if (it + 1 == d.max_iter) stop = SP2_MAXITER;
    d.e2 = d.e1;
    d.e1 = e;
    d.it = it + 1;
    if (stop >= 0) {
        d.stop = stop;
        cudaGraphSetConditional(cond, 0u);
        return;
    }
    // the next step's branch (same expressions as the host loop / oracle; tie -> EXPAND)
    int branch = (d.trX > d.nocc) ? SP2_SQUARE : SP2_EXPAND;
    if (d.closest)
        branch = (fabs(__dsub_rn(d.t2, d.nocc)) < fabs(__dsub_rn(__dsub_rn(__dmul_rn(2.0, d.trX), d.t2), d.nocc)))
                     ? SP2_SQUARE : SP2_EXPAND;
    d.branch = branch;
    d.dyn[0] = branch == SP2_SQUARE ? 1.0 : -1.0;
    d.dyn[1] = branch == SP2_SQUARE ? 0.0 : 2.0;
    d.dyn[2] = branch == SP2_SQUARE ? 2.0 : 1.0;
    cudaGraphSetConditional(cond, 1u);
}

cudaError_t launch_sp2_ctl(Sp2Dev* dev, const double* sums, const int32_t* status, int32_t* ovf,
                           unsigned long long* prod, void* rec, unsigned long long cond_handle, cudaStream_t s) {
    sp2_ctl_kernel<<<1, 1, 0, s>>>(dev, sums, status, ovf, prod, (sp2_iter_rec*)rec,
                                   (cudaGraphConditionalHandle)cond_handle);
    return cudaGetLastError();
}

}  // namespace ell
