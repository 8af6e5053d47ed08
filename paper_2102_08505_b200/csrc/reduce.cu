// reduce.cu — canonical reductions and small per-row kernels of libellpack.
//
//  * canonical sums (reading R12): the per-row inputs d_i (stored
//    diagonals, pre-drop diagonals, row norms) are summed sequentially inside
//    256-row blocks (one thread per block), then sequentially over blocks (one
//    thread). This fixed tree makes every trace bitwise reproducible, equal to the
//    oracle's, and identical for any row partition over ranks whose blocks start
//    on multiples of 256 (§8c-c12): the block partials are exchanged, never
//    re-associated.
//  * Gershgorin bounds (§8c-c8): thread per row, sequential in slot
//    order; min/max are exact, so any combine order gives the same bits.
//  * fnorm_diff rows: warp per row, binary search of the partner row.
#include <climits>
#include "internal.cuh"

namespace ell {

// The sequential sum over the block partials (c7 second level), one array at a time: the whole CTA
// stages the partials in shared memory (independent coalesced loads, all of a thread's loads issued
// before its stores: a generic load may alias shared memory, so a load-store-load sequence would
// wait out every load), then one thread adds them in block order -- the dependent chain runs on
// shared-memory operands, not on global-load latency.
__global__ void __launch_bounds__(256) final_sums_kernel(const double* __restrict__ partials, int narr,
                                                         int64_t nblocks, double* out) {
    __shared__ double sp[2048];
    for (int a = 0; a < narr; ++a) {
        double s = 0.0;
        for (int64_t b0 = 0; b0 < nblocks; b0 += 2048) {
            const int cnt = (int)(nblocks - b0 < 2048 ? nblocks - b0 : 2048);
            __syncthreads();
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = (int)threadIdx.x + 256 * u;
                v[u] = t < cnt ? __ldg(partials + (size_t)a * nblocks + b0 + t) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = (int)threadIdx.x + 256 * u;
                if (t < cnt) sp[t] = v[u];
            }
            __syncthreads();
            if (threadIdx.x == 0) {
#pragma unroll 16
                for (int t = 0; t < cnt; ++t) s = __dadd_rn(s, sp[t]);
            }
        }
        if (threadIdx.x == 0) out[a] = s;
    }
}

struct PtrPack { const double* p[8]; };

// array a of the pack by selects (an indexed param array would be copied to local memory)
__device__ __forceinline__ const double* pick_array(const PtrPack& pk, int a) {
    const double* d = pk.p[0];
#pragma unroll
    for (int q = 1; q < 8; ++q) d = a == q ? pk.p[q] : d;
    return d;
}

// a 256-row block's values d[0, cnt) into shared sv by one warp: every load in flight before the
// first store (see final_sums_kernel)
__device__ __forceinline__ void stage_block(const double* __restrict__ d, int cnt, int lane, double* sv) {
    double v[kTraceBlock / 32];
#pragma unroll
    for (int u = 0; u < kTraceBlock / 32; ++u) {
        const int q = lane + 32 * u;
        v[u] = q < cnt ? __ldg(d + q) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kTraceBlock / 32; ++u) {
        const int q = lane + 32 * u;
        if (q < cnt) sv[q] = v[u];
    }
}

// lane 0: the block's values in row order (c7 first level)
__device__ __forceinline__ double block_chain(const double* sv, int cnt) {
    double s = 0.0;
#pragma unroll 16
    for (int q = 0; q < cnt; ++q) s = __dadd_rn(s, sv[q]);
    return s;
}

// One 256-row block of one array per 32-thread group: the lanes stage the block's values in shared
// memory with coalesced loads, then lane 0 adds them in row order (c7 first level: the dependent
// chain runs on shared-memory operands, not on global-load latency).
__global__ void block_partials_pack_kernel(PtrPack arrays, int narr, int64_t b0, int64_t b1,
                                           int64_t row_end, double* partials, int64_t nblocks_total) {
    __shared__ double sv[8][kTraceBlock];
    const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + g;
    const int64_t nb = b1 - b0;
    if (t >= nb * narr) return;
    const int a = (int)(t / nb);
    const int64_t b = b0 + t % nb;
    const int64_t r0 = b * kTraceBlock;
    const int cnt = (int)(min(r0 + kTraceBlock, row_end) - r0);
    stage_block(pick_array(arrays, a) + r0, cnt, lane, sv[g]);
    __syncwarp();
    if (lane == 0) partials[(size_t)a * nblocks_total + b] = block_chain(sv[g], cnt);
}

// Both levels in one CTA for a small matrix (narr * nblocks <= 16, one rank): warp t sums (array,
// block) t as block_partials_pack_kernel does, then thread a adds array a's partials in block order
// as final_sums_kernel does -- the same two sequential chains, one launch instead of two.
__global__ void canonical_small_kernel(PtrPack arrays, int narr, int64_t n, double* out) {
    __shared__ double sv[16][kTraceBlock];
    __shared__ double sp[16];
    const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nb = (int)((n + kTraceBlock - 1) / kTraceBlock);
    if (g < narr * nb) {
        const int a = g / nb, b = g % nb;
        const int64_t r0 = (int64_t)b * kTraceBlock;
        const int cnt = (int)(min(r0 + kTraceBlock, n) - r0);
        stage_block(pick_array(arrays, a) + r0, cnt, lane, sv[g]);
        __syncwarp();
        if (lane == 0) sp[g] = block_chain(sv[g], cnt);
    }
    __syncthreads();
    if ((int)threadIdx.x < narr) {
        double s = 0.0;
        for (int b = 0; b < nb; ++b) s = __dadd_rn(s, sp[threadIdx.x * nb + b]);
        out[threadIdx.x] = s;
    }
}

cudaError_t launch_canonical_small(const double* const* arrays, int narr, int64_t n, double* out, cudaStream_t s) {
    if (narr < 1 || narr > 8 || narr * ((n + kTraceBlock - 1) / kTraceBlock) > 16) return cudaErrorInvalidValue;
    PtrPack pk{};
    for (int a = 0; a < narr; ++a) pk.p[a] = arrays[a];
    canonical_small_kernel<<<1, 512, 0, s>>>(pk, narr, n, out);
    return cudaGetLastError();
}

// partials layout: [narr][nblocks(n)], only blocks of [row_begin,row_end) written.
cudaError_t launch_block_partials(const double* const* arrays, int narr, int64_t row_begin,
                                  int64_t row_end, int64_t n, double* partials, cudaStream_t s) {
    if (narr < 1 || narr > 8) return cudaErrorInvalidValue;
    PtrPack pk{};
    for (int a = 0; a < narr; ++a) pk.p[a] = arrays[a];
    const int64_t nbt = (n + kTraceBlock - 1) / kTraceBlock;
    const int64_t b0 = row_begin / kTraceBlock;
    const int64_t b1 = (row_end + kTraceBlock - 1) / kTraceBlock;
    const int64_t work = (b1 - b0) * narr;  // (array, block) pairs, one warp each
    if (work <= 0) return cudaSuccess;
    block_partials_pack_kernel<<<(unsigned)((work + 7) / 8), 256, 0, s>>>(pk, narr, b0, b1, row_end, partials, nbt);
    return cudaGetLastError();
}

cudaError_t launch_final_sums(const double* partials, int narr, int64_t nblocks, double* out,
                              cudaStream_t s) {
    final_sums_kernel<<<1, 256, 0, s>>>(partials, narr, nblocks, out);
    return cudaGetLastError();
}

// stored diagonal a_ii (0 if absent): warp per row, lanes scan the sorted row.
__global__ void stored_diag_kernel(KMat a, int64_t r0, int64_t r1, double* out) {
    const int lane = threadIdx.x & 31;
    const int64_t i = r0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (i >= r1) return;
    const int32_t* c = a.col + (size_t)i * a.w;
    const double* v = a.val + (size_t)i * a.w;
    const int n = a.nnz[i];
    double d = 0.0;
    for (int q = lane; q < n; q += 32)
        if (c[q] == (int)i) d = v[q];
    const unsigned m = __ballot_sync(FULL, d != 0.0);
    d = m ? __shfl_sync(FULL, d, __ffs(m) - 1) : 0.0;
    if (lane == 0) out[i] = d;
}

cudaError_t launch_stored_diag(KMat a, int64_t r0, int64_t r1, double* out, cudaStream_t s) {
    const int64_t rows = r1 - r0;
    if (rows <= 0) return cudaSuccess;
    stored_diag_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, s>>>(a, r0, r1, out);
    return cudaGetLastError();
}

// Gershgorin: keys[0] = min key of lo_i, keys[1] = max key of hi_i (dkey order).
__global__ void gershgorin_kernel(KMat h, int64_t r0, int64_t r1, unsigned long long* keys) {
    const int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long kmin = ~0ull, kmax = 0ull;
    if (i < r1) {
        const int32_t* c = h.col + (size_t)i * h.w;
        const double* v = h.val + (size_t)i * h.w;
        const int n = h.nnz[i];
        double r = 0.0, d = 0.0;
        for (int q = 0; q < n; ++q) {
            if (c[q] == (int)i) d = v[q];
            else r = __dadd_rn(r, fabs(v[q]));
        }
        kmin = dkey(__dsub_rn(d, r));
        kmax = dkey(__dadd_rn(d, r));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(FULL, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(FULL, kmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(keys + 0, kmin);
        atomicMax(keys + 1, kmax);
    }
}

cudaError_t launch_gershgorin(KMat h, int64_t r0, int64_t r1, unsigned long long* keys,
                              cudaStream_t s) {
    const int64_t rows = r1 - r0;
    if (rows <= 0) return cudaSuccess;
    gershgorin_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, s>>>(h, r0, r1, keys);
    return cudaGetLastError();
}

__device__ __forceinline__ int lower_bound(const int32_t* c, int n, int key) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (c[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// out[i] = sum over the union of (a_ij - b_ij)^2 (order: lanes then butterfly; deterministic)
__global__ void fnorm_rows_kernel(KMat a, KMat b, int64_t r0, int64_t r1, double* out) {
    const int lane = threadIdx.x & 31;
    const int64_t i = r0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (i >= r1) return;
    const int32_t* ca = a.col + (size_t)i * a.w;
    const double* va = a.val + (size_t)i * a.w;
    const int32_t* cb = b.col + (size_t)i * b.w;
    const double* vb = b.val + (size_t)i * b.w;
    const int na = a.nnz[i], nb = b.nnz[i];
    double s = 0.0;
    for (int q = lane; q < na; q += 32) {
        const int j = ca[q];
        const int pb = lower_bound(cb, nb, j);
        const double bj = (pb < nb && cb[pb] == j) ? vb[pb] : 0.0;
        const double d = __dsub_rn(va[q], bj);
        s = __fma_rn(d, d, s);
    }
    for (int q = lane; q < nb; q += 32) {
        const int j = cb[q];
        const int pa = lower_bound(ca, na, j);
        if (!(pa < na && ca[pa] == j)) s = __fma_rn(vb[q], vb[q], s);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(FULL, s, o));
    if (lane == 0) out[i] = s;
}

cudaError_t launch_fnorm_rows(KMat a, KMat b, int64_t r0, int64_t r1, double* out, cudaStream_t s) {
    const int64_t rows = r1 - r0;
    if (rows <= 0) return cudaSuccess;
    fnorm_rows_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, s>>>(a, b, r0, r1, out);
    return cudaGetLastError();
}

// q_i = fma chain over the stored slots of row i, ascending, q <- fma(x, x, q) from +0
// (the T2 of the trace-closest SP2 branch rule, include/ellpack.h SP2_RULE_TRACE_CLOSEST).
// One thread per row: the chain order is the definition. Consecutive threads read consecutive
// rows, so every 128-byte line a warp touches is reused by the next slots from L1.
__global__ void sumsq_rows_kernel(KMat a, int64_t r0, int64_t r1, double* out) {
    const int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= r1) return;
    const double* v = a.val + (size_t)i * a.w;
    const int n = a.nnz[i];
    double q = 0.0;
    for (int p = 0; p < n; ++p) q = __fma_rn(v[p], v[p], q);
    out[i] = q;
}

cudaError_t launch_sumsq_rows(KMat a, int64_t r0, int64_t r1, double* out, cudaStream_t s) {
    const int64_t rows = r1 - r0;
    if (rows <= 0) return cudaSuccess;
    sumsq_rows_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, s>>>(a, r0, r1, out);
    return cudaGetLastError();
}

__global__ void col_range_kernel(KMat a, int64_t r0, int64_t r1, long long* out) {
    const int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    long long lo = LLONG_MAX, hi = -1;
    if (i < r1) {
        const int nz = a.nnz[i];
        if (nz > 0) {
            lo = a.col[(size_t)i * a.w];
            hi = a.col[(size_t)i * a.w + nz - 1];
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(FULL, lo, o));
        hi = max(hi, __shfl_xor_sync(FULL, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (lo != LLONG_MAX) atomicMin(out, lo);
        if (hi >= 0) atomicMax(out + 1, hi);
    }
}

cudaError_t launch_col_range(KMat a, int64_t r0, int64_t r1, long long* out, cudaStream_t s) {
    const int64_t rows = r1 - r0;
    if (rows <= 0) return cudaSuccess;
    col_range_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(a, r0, r1, out);
    return cudaGetLastError();
}

// Canonical-form check (D1, §8c-c1): 0 <= nnz <= w, columns in [0, n) strictly ascending, values
// finite. Thread per row; any violation sets *bad (ELLPACK_OPT_VALIDATE).
__global__ void validate_kernel(KMat a, int64_t n, int32_t* bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int nz = a.nnz[i];
    bool ok = nz >= 0 && nz <= a.w;
    if (ok) {
        const int32_t* c = a.col + (size_t)i * a.w;
        const double* v = a.val + (size_t)i * a.w;
        int prev = -1;
        for (int p = 0; p < nz && ok; ++p) {
            const int j = c[p];
            ok = j > prev && (int64_t)j < n && isfinite(v[p]);
            prev = j;
        }
    }
    if (!ok) atomicOr(bad, 1);
}

cudaError_t launch_validate(KMat a, int64_t n, int32_t* bad, cudaStream_t s) {
    validate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, n, bad);
    return cudaGetLastError();
}

__global__ void identity_kernel(int64_t n, KOut id) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    id.val[(size_t)i * id.w] = 1.0;
    id.col[(size_t)i * id.w] = (int32_t)i;
    id.nnz[i] = 1;
}

cudaError_t launch_identity(int64_t n, KOut id, cudaStream_t s) {
    identity_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, id);
    return cudaGetLastError();
}

// dst row i <- src row i (truncated to dst.w; status[0] += overflow rows, status[1] max nnz)
__global__ void copy_rows_kernel(KMat src, KOut dst, int64_t r0, int64_t r1, int32_t* status) {
    const int lane = threadIdx.x & 31;
    const int64_t i = r0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (i >= r1) return;
    const int n = src.nnz[i];
    const int m = n < dst.w ? n : dst.w;
    const size_t so = (size_t)i * src.w, d_o = (size_t)i * dst.w;
    // pairs of entries per lane (widths are even: 16-byte value pairs, 8-byte column pairs)
    const double2* sv = reinterpret_cast<const double2*>(src.val + so);
    const int2* sc = reinterpret_cast<const int2*>(src.col + so);
    double2* dv = reinterpret_cast<double2*>(dst.val + d_o);
    int2* dc = reinterpret_cast<int2*>(dst.col + d_o);
    for (int q = lane; 2 * q < m; q += 32) {
        dv[q] = sv[q];  // (a row's slot m of an odd count is padding: copying it is harmless)
        dc[q] = sc[q];
    }
    if (lane == 0) {
        dst.nnz[i] = m;
        if (n > dst.w) atomicAdd(status, 1);
        atomicMax(status + 1, n);
    }
}

cudaError_t launch_copy_rows(KMat src, KOut dst, int64_t r0, int64_t r1, int32_t* status,
                             cudaStream_t s) {
    const int64_t rows = r1 - r0;
    if (rows <= 0) return cudaSuccess;
    copy_rows_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, s>>>(src, dst, r0, r1, status);
    return cudaGetLastError();
}

__global__ void max_nnz_kernel(const int32_t* nnz, int64_t r0, int64_t r1, int32_t* out) {
    const int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int v = (i < r1) ? nnz[i] : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
    if ((threadIdx.x & 31) == 0 && v) atomicMax(out, v);
}

// out[0] += #rows r in [r0, r1) with nnz[r] > w (the exact overflow-row count of a kept-count array)
__global__ void count_over_kernel(const int32_t* nnz, int64_t r0, int64_t r1, int32_t w, int32_t* out) {
    const int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned m = __ballot_sync(FULL, i < r1 && nnz[i] > w);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(out, __popc(m));
}

cudaError_t launch_count_over(const int32_t* nnz, int64_t r0, int64_t r1, int32_t w, int32_t* out,
                              cudaStream_t s) {
    const int64_t rows = r1 - r0;
    if (rows <= 0) return cudaSuccess;
    count_over_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(nnz, r0, r1, w, out);
    return cudaGetLastError();
}

cudaError_t launch_max_nnz(const int32_t* nnz, int64_t r0, int64_t r1, int32_t* out, cudaStream_t s) {
    const int64_t rows = r1 - r0;
    if (rows <= 0) return cudaSuccess;
    max_nnz_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(nnz, r0, r1, out);
    return cudaGetLastError();
}

}  // namespace ell

namespace ell {
// P = sum_i sum_{k in A_i} nnz_B(k), rows [r0, r1): the scalar-product count of A x B
// (SURVEY §8d "P"), reported per SP2 iteration. Warp per row, exact int64 atomics.
__global__ void products_kernel(KMat a, const int32_t* __restrict__ nnz_b, int64_t r0, int64_t r1,
                                unsigned long long* out) {
    const int lane = threadIdx.x & 31;
    const int64_t i = r0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    unsigned long long s = 0;
    if (i < r1) {
        const int na = a.nnz[i];
        const int32_t* ac = a.col + (size_t)i * a.w;
        for (int q = lane; q < na; q += 32) s += (unsigned long long)nnz_b[ac[q]];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane == 0 && s) atomicAdd(out, s);
}

cudaError_t launch_products(KMat a, const int32_t* nnz_b, int64_t r0, int64_t r1, unsigned long long* out,
                            cudaStream_t s) {
    const int64_t rows = r1 - r0;
    if (rows <= 0) return cudaSuccess;
    products_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(a, nnz_b, r0, r1, out);
    return cudaGetLastError();
}
}  // namespace ell
