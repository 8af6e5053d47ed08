// tiny.cu — the small-matrix row kernel of libellpack (sm_100a, FP64 CUDA cores).
//
// Same method as the general path of spgemm.cu for one window that covers every column (N <= 1024,
// one rank, no Old operand: the cfg1-sized X^2 call of SURVEY §8d, BASELINE configs[0]):
//   s_j = fma chain over k ascending in A_i of a_ik * b_kj   (§8a-a2, reading R12),
//   c_j = alpha * s_j, kept iff |c_j| > tau, written ascending (§8a-a3, R3),
//   tr X from the stored a_ii, tr X^2 from the pre-drop s_ii (§8a-a4, R5), canonical sums (c7).
// What differs is latency, not arithmetic. Such a launch has one row per warp and a few warps per
// SM, so nothing hides a load: the general kernel spends its time waiting for one B row's gathers
// at a time (ncu: long-scoreboard stalls on every round). Here a warp issues the gathers of 16 B
// rows at once (columns and values up to the ELLPACK width, masked by nnz afterwards, so no load
// waits for another), then applies the 16 rows in k order; the per-CTA status partials and the
// canonical sums of tr X and tr X^2 are finished by the last CTA (one launch instead of a
// status memset, a ticket memset, the row kernel and the canonical-sum kernel).
#include "internal.cuh"
#include "devutil.cuh"

#include <climits>

namespace ell {

constexpr int kTinyWarps = 4;
constexpr int kTinyKB = 16;  // B rows whose gathers are in flight together

template <int UT, bool A1>
__global__ void __launch_bounds__(kTinyWarps * 32) row_tiny_kernel(const RowOpParams p, int Np,
                                                                   unsigned int* __restrict__ counter,
                                                                   int32_t* __restrict__ part,
                                                                   int32_t* __restrict__ status,
                                                                   double* __restrict__ sums) {
    extern __shared__ __align__(16) double tw[];  // [kTinyWarps][Np] windows (all columns)
    __shared__ int32_t cta_kept[kTinyWarps], cta_ovf[kTinyWarps];
    __shared__ unsigned int ticket;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t acc = (uint32_t)__cvta_generic_to_shared(tw + (size_t)wid * Np);
    for (int j = lane; j < Np; j += 32) sts64(acc + 8u * (uint32_t)j, 0.0);
    __syncwarp();
    const int64_t i = p.row_begin + (int64_t)blockIdx.x * kTinyWarps + wid;
    int32_t kept = 0, ovf = 0;
    if (i < p.row_end) {
        const int32_t* __restrict__ a_col = p.A.col + (size_t)i * p.A.w;
        const double* __restrict__ a_val = p.A.val + (size_t)i * p.A.w;
        const int nA = p.alpha != 0.0 ? p.A.nnz[i] : 0;
        const int nAs = p.A.nnz[i];  // the stored diagonal is looked up even when alpha = 0
        int lo = INT_MAX, hi = -1;
        for (int kb = 0; kb < nA; kb += 32) {
            const int q = kb + lane;
            const int kq = q < nA ? __ldg(a_col + q) : 0;
            const double aq = q < nA ? __ldg(a_val + q) : 0.0;
            const int cnt = min(32, nA - kb);
            for (int e0 = 0; e0 < cnt; e0 += kTinyKB) {
                int J[kTinyKB][UT], nb[kTinyKB];
                double V[kTinyKB][UT];
#pragma unroll
                for (int e = 0; e < kTinyKB; ++e) {  // every load of the batch before any use
                    const int k = __shfl_sync(FULL, kq, e0 + e);
                    const bool live = e0 + e < cnt;
                    const int32_t* __restrict__ bc = p.B.col + (size_t)k * p.B.w;
                    const double* __restrict__ bv = p.B.val + (size_t)k * p.B.w;
                    nb[e] = live ? __ldg(p.B.nnz + k) : 0;
#pragma unroll
                    for (int u = 0; u < UT; ++u) {
                        const int idx = 32 * u + lane;
                        const bool in = live && idx < p.B.w;  // the row's slots, padding masked below
                        J[e][u] = in ? __ldg(bc + idx) : -1;
                        V[e][u] = in ? __ldg(bv + idx) : 0.0;
                    }
                }
#pragma unroll
                for (int e = 0; e < kTinyKB; ++e) {  // k ascending (the oracle's fma chain per column)
                    const double a = __shfl_sync(FULL, aq, e0 + e);
#pragma unroll
                    for (int u = 0; u < UT; ++u) {
                        if (32 * u + lane < nb[e]) {
                            const int j = J[e][u];
                            const uint32_t ad = acc + 8u * (uint32_t)j;
                            sts64(ad, __fma_rn(a, V[e][u], lds64(ad)));
                            lo = min(lo, j);
                            hi = max(hi, j);
                        }
                    }
                    __syncwarp();
                }
            }
        }
        lo = warp_min(lo);
        hi = warp_max(hi);
        // pre-drop s_ii (R5): the accumulated value of column i (+0 when no product reaches it)
        const double ds = lds64(acc + 8u * (uint32_t)i);
        double dc = 0.0;
        double* __restrict__ crow_v = p.C.val + (size_t)i * p.C.w;
        int32_t* __restrict__ crow_c = p.C.col + (size_t)i * p.C.w;
        const int cw = p.C.w;
        if (hi >= lo) {
            for (int j0 = lo & ~31; j0 <= hi; j0 += 32) {  // Np is a multiple of 32 > hi
                const int j = j0 + lane;
                const uint32_t ad = acc + 8u * (uint32_t)j;
                const double v = lds64(ad);
                sts64(ad, 0.0);
                const double x = A1 ? v : __dmul_rn(p.alpha, v);
                const bool keep = fabs(x) > p.tau;
                const unsigned m = __ballot_sync(FULL, keep);
                const uint32_t pos = (uint32_t)kept + (uint32_t)__popc(m & lt);
                st_entry(keep && pos < (uint32_t)cw, crow_v + pos, crow_c + pos, x, j);
                if ((int64_t)j == i) dc = keep ? x : 0.0;
                kept += __popc(m);
            }
        }
        // stored a_ii
        double dA = 0.0;
        bool has = false;
        for (int q = lane; q < nAs; q += 32)
            if (a_col[q] == (int)i) { dA = a_val[q]; has = true; }
        const unsigned hm = __ballot_sync(FULL, has);
        dA = hm ? __shfl_sync(FULL, dA, __ffs(hm) - 1) : 0.0;
        dc = warp_sum(dc);  // one lane holds it, the others +0: x + 0 = x exactly
        if (lane == 0) {
            p.C.nnz[i] = kept < cw ? kept : cw;
            if (p.diag_a) p.diag_a[i] = dA;
            if (p.diag_s) p.diag_s[i] = ds;
            if (p.diag_c) p.diag_c[i] = dc;
        }
        ovf = kept > cw ? 1 : 0;
    }
    if (lane == 0) {
        cta_kept[wid] = kept;
        cta_ovf[wid] = ovf;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t mk = 0, ov = 0;
        for (int w = 0; w < kTinyWarps; ++w) {
            mk = max(mk, cta_kept[w]);
            ov += cta_ovf[w];
        }
        part[2 * blockIdx.x] = mk;
        part[2 * blockIdx.x + 1] = ov;
        __threadfence();  // this CTA's rows, diagonals and partials before its ticket
        ticket = atomicAdd(counter, 1u);
    }
    __syncthreads();
    if (ticket != gridDim.x - 1) return;
    // last CTA: status (rows over the width, max kept) and the canonical sums (c7) of tr X, tr X^2
    __threadfence();
    if (threadIdx.x == 0) {
        int32_t mk = 0, ov = 0;
        for (unsigned b = 0; b < gridDim.x; ++b) {
            mk = max(mk, __ldcg(part + 2 * b));
            ov += __ldcg(part + 2 * b + 1);
        }
        status[0] = ov;
        status[1] = mk;
        *counter = 0u;  // ready for the next launch (graph replays)
    }
    if (sums) {
        // (array, 256-row block) chains, one warp each (n <= 1024: <= 8 chains), then block order
        const int64_t n = p.row_end;  // one rank: rows [0, n)
        const int nbk = (int)((n + kTraceBlock - 1) / kTraceBlock);
        __shared__ double bpart[2][4];
        double* stage = tw + (size_t)wid * Np;  // this warp's window, now all zero and unused
        for (int t = wid; t < 2 * nbk; t += kTinyWarps) {
            const int a = t / nbk, b = t % nbk;
            const double* __restrict__ d = a == 0 ? p.diag_a : p.diag_s;
            const int64_t r0 = (int64_t)b * kTraceBlock;
            const int cnt = (int)(min((int64_t)kTraceBlock, n - r0));
            double v[kTraceBlock / 32];
#pragma unroll
            for (int u = 0; u < kTraceBlock / 32; ++u) {
                const int q = lane + 32 * u;
                v[u] = q < cnt ? __ldcg(d + r0 + q) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kTraceBlock / 32; ++u) {
                const int q = lane + 32 * u;
                if (q < cnt) stage[q] = v[u];
            }
            __syncwarp();
            if (lane == 0) {
                double s = 0.0;
#pragma unroll 16
                for (int q = 0; q < cnt; ++q) s = __dadd_rn(s, stage[q]);
                bpart[a][b] = s;
            }
            __syncwarp();
        }
        __syncthreads();
        if (threadIdx.x < 2) {
            double s = 0.0;
            for (int b = 0; b < nbk; ++b) s = __dadd_rn(s, bpart[threadIdx.x][b]);
            sums[threadIdx.x] = s;
        }
    }
    __threadfence_system();  // status / sums may live in mapped host memory
}

bool tiny_eligible(const RowOpParams& p, int64_t n) {
    return n <= 1024 && p.row_begin == 0 && p.row_end == n && p.old_mode == 0 && !p.upper && !p.dyn &&
           !p.stash_a && !p.stash_old && p.B.w <= 64 && p.diag_a && p.diag_s;
}

size_t tiny_smem(int64_t n) { return (size_t)kTinyWarps * (size_t)((n + 31) & ~int64_t(31)) * 8; }

// The counter (zero; the kernel leaves it zero) and part (2 ints per CTA) are the caller's scratch;
// status[0..1] (rows over C.w, max kept) and sums (nullable: tr X, tr X^2 by the canonical sums of
// p.diag_a, p.diag_s) may be device or mapped pinned host addresses.
cudaError_t launch_tiny(const RowOpParams& p, int64_t n, unsigned int* counter, int32_t* part, int32_t* status,
                        double* sums, cudaStream_t s) {
    const int Np = (int)((n + 31) & ~int64_t(31));
    const unsigned grid = (unsigned)((p.row_end - p.row_begin + kTinyWarps - 1) / kTinyWarps);
    if (grid == 0) return cudaSuccess;
    const size_t smem = tiny_smem(n);
    const bool a1 = p.alpha == 1.0;  // smem <= 32 KB: within the default dynamic limit
    if (p.B.w <= 32) {
        if (a1) row_tiny_kernel<1, true><<<grid, kTinyWarps * 32, smem, s>>>(p, Np, counter, part, status, sums);
        else row_tiny_kernel<1, false><<<grid, kTinyWarps * 32, smem, s>>>(p, Np, counter, part, status, sums);
    } else {
        if (a1) row_tiny_kernel<2, true><<<grid, kTinyWarps * 32, smem, s>>>(p, Np, counter, part, status, sums);
        else row_tiny_kernel<2, false><<<grid, kTinyWarps * 32, smem, s>>>(p, Np, counter, part, status, sums);
    }
    return cudaGetLastError();
}

}  // namespace ell
