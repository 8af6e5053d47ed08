// spgemm.cu — the fused ELLPACK row kernel of libellpack (sm_100a, FP64 CUDA cores).
//
// One warp owns one output row i (BJ north_star (1): "a warp or small CTA owns each
// output row"); a persistent grid strides over rows [row_begin, row_end).
// Per row:
//   a1  span pre-pass: lo = min over k in A_i of col_B[k][0], hi = max of the last
//       column (plus Old_i's extent); the row's column window [lo, hi] is processed
//       in ceil(span / S) passes of an S-double dense-window accumulator in shared
//       memory (single pass whenever the span fits).
//   a2  gather + accumulate: for k in A_i ascending, the warp's lanes take the
//       entries of B row k (distinct columns, so no two lanes collide inside one k)
//       and do acc[j] = fma(a_ik, b_kj, acc[j]); a __syncwarp between consecutive
//       k orders the read-modify-writes, so every output entry is the fma chain in
//       ascending k (reading R12 -> bitwise equal to the oracle). B rows are
//       prefetched D steps ahead into registers (R slots of 32 entries per step)
//       with read-only (ld.global.nc) loads, hiding the L2 latency of the gather.
//   a3  combine + drop + compact: Old_i entries (C_old / the SP2 iterate) are merged
//       into the window with c = fma(alpha, s, beta*old); a window scan keeps
//       |c| > tau, compacts with ballot/popc and writes the row contiguously in
//       ascending column order (coalesced stores), counting overflow past C.w.
//   a4  per-row trace / norm inputs (stored a_ii, pre-drop s_ii, stored c_ii,
//       ||S - Old||^2), reduced later in canonical order (reduce.cu).
// With A = B = Old = X this single kernel is the fused SP2 step (BJ north_star (2)):
// SQUARE = (alpha 1, old_mode 2), EXPAND = (alpha -1, beta 2, old_mode 1) since
// fma(-1, s, 2x) = round(2x - s) exactly (2x is exact).
#include "internal.cuh"
#include <climits>

namespace ell {

__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(FULL, v, o));
    return v;
}
__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

template <int R, int D>
__global__ void __launch_bounds__(128) row_op_kernel(const RowOpParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int wpc = blockDim.x >> 5;
    const int S = p.S;
    double* acc = reinterpret_cast<double*>(smem_raw) + (size_t)wid * S;
    unsigned char* flg = smem_raw + (size_t)wpc * S * sizeof(double) + (size_t)wid * S;
    const bool has_old = p.old_mode != 0;
    for (int j = lane; j < S; j += 32) acc[j] = 0.0;
    if (has_old)
        for (int j = lane; j < S; j += 32) flg[j] = 0;
    __syncwarp();

    const unsigned lt_mask = (1u << lane) - 1u;
    const int64_t gw = (int64_t)blockIdx.x * wpc + wid;
    const int64_t nwarps = (int64_t)gridDim.x * wpc;
    int32_t my_max_kept = 0, my_ovf = 0;

    for (int64_t i = p.row_begin + gw; i < p.row_end; i += nwarps) {
        const double* a_val = p.A.val + (size_t)i * p.A.w;
        const int32_t* a_col = p.A.col + (size_t)i * p.A.w;
        const int32_t nA = (p.alpha != 0.0) ? p.A.nnz[i] : 0;
        const double* o_val = nullptr;
        const int32_t* o_col = nullptr;
        int32_t nOld = 0;
        if (has_old) {
            o_val = p.Old.val + (size_t)i * p.Old.w;
            o_col = p.Old.col + (size_t)i * p.Old.w;
            nOld = p.Old.nnz[i];
        }

        // ---- a1: span pre-pass (+ stored diagonal of A)
        int lo = INT_MAX, hi = -1;
        double dA = 0.0;
        bool hasdA = false;
        for (int q = lane; q < nA; q += 32) {
            const int k = a_col[q];
            if (k == (int)i) { dA = a_val[q]; hasdA = true; }
            const int nb = __ldg(p.B.nnz + k);
            if (nb > 0) {
                const int32_t* bc = p.B.col + (size_t)k * p.B.w;
                lo = min(lo, __ldg(bc));
                hi = max(hi, __ldg(bc + nb - 1));
            }
        }
        if (nOld > 0 && lane == 0) {
            lo = min(lo, o_col[0]);
            hi = max(hi, o_col[nOld - 1]);
        }
        lo = warp_min(lo);
        hi = warp_max(hi);
        if (p.diag_a) {
            const unsigned m = __ballot_sync(FULL, hasdA);
            dA = m ? __shfl_sync(FULL, dA, __ffs(m) - 1) : 0.0;
        }

        int32_t kept = 0;
        double ds = 0.0, dc = 0.0, nrm = 0.0;
        const size_t c_off = (size_t)i * p.C.w;
        if (hi >= lo) {
            const int span = hi - lo + 1;
            const int npass = (span + S - 1) / S;
            const bool multi = npass > 1;
            int32_t* cur = p.cursors + gw * p.cur_stride;
            if (multi && (p.stash_a || p.stash_old)) {
                // C aliases an input: copy the input rows aside before pass 0 writes.
                double* sv = p.st_val + gw * p.st_stride;
                int32_t* sc = p.st_col + gw * p.st_stride;
                if (p.stash_a) {
                    for (int q = lane; q < nA; q += 32) { sv[q] = a_val[q]; sc[q] = a_col[q]; }
                    a_val = sv; a_col = sc;
                    sv += p.A.w; sc += p.A.w;
                }
                if (p.stash_old) {
                    for (int q = lane; q < nOld; q += 32) { sv[q] = o_val[q]; sc[q] = o_col[q]; }
                    o_val = sv; o_col = sc;
                }
                __syncwarp();
            }
            int old_cur = 0;
            for (int pass = 0; pass < npass; ++pass) {
                const int c0 = lo + pass * S;
                const int c1 = min(c0 + S, hi + 1);

                // ---- a2: gather + accumulate, k ascending
                for (int p0 = 0; p0 < nA; p0 += 32) {
                    const int cnt = min(32, nA - p0);
                    int mk = 0, mnb = 0, mst = 0;
                    double ma = 0.0;
                    if (lane < cnt) {
                        mk = a_col[p0 + lane];
                        ma = a_val[p0 + lane];
                        mnb = __ldg(p.B.nnz + mk);
                        if (multi && pass > 0) mst = cur[p0 + lane];
                    }
                    int rj[D][R];
                    double rv[D][R];
                    // prologue: steps 0..D-1
#pragma unroll
                    for (int d = 0; d < D; ++d) {
                        if (d < cnt) {
                            const int k = __shfl_sync(FULL, mk, d);
                            const int nb = __shfl_sync(FULL, mnb, d);
                            const int st = __shfl_sync(FULL, mst, d);
                            const int32_t* bc = p.B.col + (size_t)k * p.B.w;
                            const double* bv = p.B.val + (size_t)k * p.B.w;
#pragma unroll
                            for (int r = 0; r < R; ++r) {
                                const int q = st + lane + 32 * r;
                                rj[d][r] = INT_MAX;
                                rv[d][r] = 0.0;
                                if (q < nb) { rj[d][r] = __ldg(bc + q); rv[d][r] = __ldg(bv + q); }
                            }
                        }
                    }
                    for (int t0 = 0; t0 < cnt; t0 += D) {
#pragma unroll
                        for (int d = 0; d < D; ++d) {
                            const int t = t0 + d;
                            if (t < cnt) {
                                const double a = __shfl_sync(FULL, ma, t);
                                int n_in = 0;
#pragma unroll
                                for (int r = 0; r < R; ++r) {
                                    const int j = rj[d][r];
                                    const bool inr = j < c1;
                                    if (inr) {
                                        double* ap = acc + (j - c0);
                                        *ap = __fma_rn(a, rv[d][r], *ap);
                                    }
                                    n_in += __popc(__ballot_sync(FULL, inr));
                                }
                                if (n_in == 32 * R) {
                                    // B row longer than the prefetched slots: finish it directly.
                                    const int k = __shfl_sync(FULL, mk, t);
                                    const int nb = __shfl_sync(FULL, mnb, t);
                                    const int st = __shfl_sync(FULL, mst, t);
                                    const int32_t* bc = p.B.col + (size_t)k * p.B.w;
                                    const double* bv = p.B.val + (size_t)k * p.B.w;
                                    int q = st + 32 * R + lane;
                                    while (true) {
                                        const bool v = q < nb;
                                        const int j = v ? __ldg(bc + q) : INT_MAX;
                                        const bool inr = j < c1;
                                        if (inr) {
                                            double* ap = acc + (j - c0);
                                            *ap = __fma_rn(a, __ldg(bv + q), *ap);
                                        }
                                        const int n = __popc(__ballot_sync(FULL, inr));
                                        n_in += n;
                                        if (n < 32) break;
                                        q += 32;
                                    }
                                }
                                if (multi && lane == t) mst += n_in;
                                // refill this slot with step t + D
                                if (t + D < cnt) {
                                    const int k = __shfl_sync(FULL, mk, t + D);
                                    const int nb = __shfl_sync(FULL, mnb, t + D);
                                    const int st = __shfl_sync(FULL, mst, t + D);
                                    const int32_t* bc = p.B.col + (size_t)k * p.B.w;
                                    const double* bv = p.B.val + (size_t)k * p.B.w;
#pragma unroll
                                    for (int r = 0; r < R; ++r) {
                                        const int q = st + lane + 32 * r;
                                        rj[d][r] = INT_MAX;
                                        rv[d][r] = 0.0;
                                        if (q < nb) { rj[d][r] = __ldg(bc + q); rv[d][r] = __ldg(bv + q); }
                                    }
                                }
                                __syncwarp();
                            }
                        }
                    }
                    if (multi && lane < cnt) cur[p0 + lane] = mst;
                }
                __syncwarp();

                // ---- a4: pre-combine diagonal s_ii
                if ((int64_t)c0 <= i && i < (int64_t)c1) ds = acc[i - c0];

                // ---- a3: combine with Old entries in [c0, c1)
                if (has_old) {
                    while (old_cur < nOld) {
                        const int q = old_cur + lane;
                        const bool v = q < nOld;
                        const int j = v ? o_col[q] : INT_MAX;
                        const bool inr = j < c1;
                        if (inr) {
                            const double x = o_val[q];
                            double* ap = acc + (j - c0);
                            const double s = *ap;
                            if (p.normsq) {
                                const double df = __dsub_rn(s, x);
                                nrm = __fma_rn(df, df, nrm);
                            }
                            const double tt = (p.old_mode == 1) ? __dmul_rn(p.beta, x) : 0.0;
                            *ap = __fma_rn(p.alpha, s, tt);
                            flg[j - c0] = 1;
                        }
                        const int n = __popc(__ballot_sync(FULL, inr));
                        old_cur += n;
                        if (n < 32) break;
                    }
                    __syncwarp();
                }

                // ---- a3: drop + compact + write (ascending columns)
                const int width = c1 - c0;
                for (int b = 0; b < width; b += 32) {
                    const int jj = b + lane;
                    const bool in = jj < width;
                    double v = 0.0;
                    bool f = false;
                    if (in) {
                        v = acc[jj];
                        acc[jj] = 0.0;
                        if (has_old) { f = flg[jj] != 0; flg[jj] = 0; }
                    }
                    double c;
                    if (f) {
                        c = v;
                    } else {
                        c = __fma_rn(p.alpha, v, 0.0);
                        if (p.normsq) nrm = __fma_rn(v, v, nrm);
                    }
                    const bool keep = in && fabs(c) > p.tau;
                    const unsigned m = __ballot_sync(FULL, keep);
                    if (keep) {
                        const int pos = kept + __popc(m & lt_mask);
                        if (pos < p.C.w) {
                            p.C.val[c_off + pos] = c;
                            p.C.col[c_off + pos] = c0 + jj;
                        }
                        if ((int64_t)(c0 + jj) == i) dc = c;
                    }
                    kept += __popc(m);
                }
                __syncwarp();
            }
        }
        // ---- row epilogue
        if (lane == 0) p.C.nnz[i] = kept < p.C.w ? kept : p.C.w;
        my_max_kept = max(my_max_kept, kept);
        if (kept > p.C.w) ++my_ovf;
        if (p.diag_c) {
            dc = warp_sum(dc);  // at most one lane holds c_ii != 0; x + 0 = x exactly
            if (lane == 0) p.diag_c[i] = dc;
        }
        if (p.diag_s && lane == 0) p.diag_s[i] = ds;
        if (p.diag_a && lane == 0) p.diag_a[i] = dA;
        if (p.normsq) {
            nrm = warp_sum(nrm);
            if (lane == 0) p.normsq[i] = nrm;
        }
    }
    if (lane == 0) {
        if (my_ovf) atomicAdd(p.status + 0, my_ovf);
        if (my_max_kept) atomicMax(p.status + 1, my_max_kept);
    }
}

template <int R, int D>
static cudaError_t config_kernel(size_t smem) {
    return cudaFuncSetAttribute(row_op_kernel<R, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem);
}

static int pick_R(int wb) { return wb <= 32 ? 1 : (wb <= 64 ? 2 : 4); }

cudaError_t plan_row_op(const RowOpParams& p, int window_opt, int warps_opt, int num_sms,
                        LaunchCfg* cfg) {
    int S = window_opt > 0 ? window_opt : 4096;
    S = (S + 31) & ~31;
    int wpc = warps_opt > 0 ? warps_opt : 4;
    if (wpc > 4) wpc = 4;  // __launch_bounds__(128)
    cfg->S = S;
    cfg->warps_per_cta = wpc;
    cfg->R = pick_R(p.B.w);
    cfg->smem = (size_t)wpc * S * (sizeof(double) + (p.old_mode ? 1 : 0));
    if (cfg->smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    cudaError_t e;
    int blocks_per_sm = 0;
    switch (cfg->R) {
        case 1:
            if ((e = config_kernel<1, 8>(cfg->smem))) return e;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, row_op_kernel<1, 8>,
                                                              wpc * 32, cfg->smem);
            break;
        case 2:
            if ((e = config_kernel<2, 8>(cfg->smem))) return e;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, row_op_kernel<2, 8>,
                                                              wpc * 32, cfg->smem);
            break;
        default:
            if ((e = config_kernel<4, 4>(cfg->smem))) return e;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, row_op_kernel<4, 4>,
                                                              wpc * 32, cfg->smem);
            break;
    }
    if (e) return e;
    if (blocks_per_sm < 1) return cudaErrorInvalidConfiguration;
    const int64_t rows = p.row_end - p.row_begin;
    int64_t need = (rows + wpc - 1) / wpc;
    int64_t full = (int64_t)blocks_per_sm * num_sms;
    cfg->grid = (int)(need < full ? (need > 0 ? need : 1) : full);
    return cudaSuccess;
}

cudaError_t launch_row_op(const RowOpParams& p, const LaunchCfg& cfg, cudaStream_t s) {
    dim3 block(cfg.warps_per_cta * 32), grid(cfg.grid);
    switch (cfg.R) {
        case 1: row_op_kernel<1, 8><<<grid, block, cfg.smem, s>>>(p); break;
        case 2: row_op_kernel<2, 8><<<grid, block, cfg.smem, s>>>(p); break;
        default: row_op_kernel<4, 4><<<grid, block, cfg.smem, s>>>(p); break;
    }
    return cudaGetLastError();
}

}  // namespace ell
