// spgemm.cu — the fused ELLPACK row kernel of libellpack (sm_100a, FP64 CUDA cores).
//
// One warp owns one output row i (BJ north_star (1): "a warp or small CTA owns each
// output row"); a persistent grid strides over rows [row_begin, row_end).
// Per row:
//   a1  window: the host probes the bandwidths of A, B (and Old) once per launch, so
//       every row's products fall in the row-centred window [i - h, i + h]; the
//       window (S doubles, S >= 2h+1) is a dense accumulator in shared memory and
//       the row needs no span pre-pass ("fast path"). Rows whose span does not fit
//       (S capped by shared memory, e.g. dense SP2 iterates) take the general path:
//       a span pre-pass and ceil(span/S) passes with per-k cursors.
//   a2  gather + accumulate: A's row is staged in shared memory (B-row offset,
//       a_ik, nnz_B(k)); for k ascending the warp's lanes take the entries of B row k
//       (distinct columns, so no two lanes collide inside one k) and do
//       acc[j] = fma(a_ik, b_kj, acc[j]); a __syncwarp between consecutive k orders
//       the read-modify-writes, so every output entry is the fma chain in ascending
//       k (reading R12 -> bitwise equal to the oracle). B rows are prefetched D
//       steps ahead into registers (up to R groups of 32 entries per step; groups
//       beyond nnz_B(k) are skipped warp-uniformly) with read-only loads, hiding the
//       L2 latency of the gather; a step's R shared loads, fmas and shared stores
//       are issued as batches on 32-bit shared addresses.
//   a3  combine + drop + compact: Old_i entries (C_old / the SP2 iterate) are merged
//       into the window with c = fma(alpha, s, beta*old); a window scan (two slots
//       per lane, 16-byte shared loads) keeps |c| > tau, compacts with ballot/popc
//       and writes the row contiguously in ascending column order with predicated
//       stores, counting overflow past C.w.
//   a4  per-row trace / norm inputs (stored a_ii, pre-drop s_ii, stored c_ii,
//       ||S - Old||^2), reduced later in canonical order (reduce.cu).
// With A = B = Old = X this single kernel is the fused SP2 step (BJ north_star (2)):
// SQUARE = (alpha 1, old_mode 2), EXPAND = (alpha -1, beta 2, old_mode 1) since
// fma(-1, s, 2x) = round(2x - s) exactly (2x is exact).
//
// Template parameters: R (B groups of 32 per prefetched step), D (prefetch depth),
// MODE (0: no Old operand; 1: Old operand; 2: Old operand + ||S - Old||^2 norm). Whether
// Old enters the value (beta*old, p.old_mode == 1) or only the union (p.old_mode == 2)
// is a runtime, warp-uniform choice.
#include "internal.cuh"
#include <climits>

namespace ell {

constexpr int kStage = 128;  // A-row entries staged in shared memory per piece

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

// 32-bit shared-window accesses (no generic->shared conversion per access)
__device__ __forceinline__ double lds64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts64(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void lds128(uint32_t a, double& x, double& y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, double x, double y) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds16u(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts16u(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Branch-free predicated store of one output entry (value + column).
__device__ __forceinline__ void st_entry(bool pred, double* pv, int32_t* pc, double x, int32_t c) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t"
        "@q st.global.f64 [%1], %2;\n\t@q st.global.b32 [%3], %4;\n\t}" ::"r"((int)pred),
        "l"(pv), "d"(x), "l"(pc), "r"(c)
        : "memory");
}

// Per-warp shared layout: acc[S + 2] f64 | stage: boff[kStage] i64, aa[kStage] f64,
// anb[kStage] i32, ast[kStage] i32, ak[kStage] i32 | flags[S] u8 (MODE != 0 only)
struct WarpSmem {
    uint32_t acc;  // shared address of acc[0]
    uint32_t flg;  // shared address of flags[0]
    uint32_t stg;  // shared address of the stage (explicit 32-bit shared accesses: the
                   // generic path would route these through L1TEX with long-scoreboard waits)
};

// stage field accessors (boff | aa | anb | ast | ak, kStage entries each)
__device__ __forceinline__ long long stg_boff(const WarpSmem& w, int t) {
    long long v;
    asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(w.stg + 8u * t) : "memory");
    return v;
}
__device__ __forceinline__ double stg_aa(const WarpSmem& w, int t) { return lds64(w.stg + 8u * (kStage + t)); }
__device__ __forceinline__ int lds32i(uint32_t a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts32i(uint32_t a, int v) {
    asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t stg_anb_a(const WarpSmem& w, int t) { return w.stg + 16u * kStage + 4u * t; }
__device__ __forceinline__ uint32_t stg_ast_a(const WarpSmem& w, int t) { return w.stg + 20u * kStage + 4u * t; }
__device__ __forceinline__ uint32_t stg_ak_a(const WarpSmem& w, int t) { return w.stg + 24u * kStage + 4u * t; }
__device__ __forceinline__ int stg_anb(const WarpSmem& w, int t) { return lds32i(stg_anb_a(w, t)); }
__device__ __forceinline__ int stg_ast(const WarpSmem& w, int t) { return lds32i(stg_ast_a(w, t)); }
__device__ __forceinline__ int stg_ak(const WarpSmem& w, int t) { return lds32i(stg_ak_a(w, t)); }

// acc has S + 2 slots: acc[S] is the trash slot of padded lanes (16-byte aligned pair).
__host__ __device__ inline size_t warp_smem_bytes(int S, bool has_old) {
    return (size_t)(S + 2) * 8 + (size_t)kStage * 28 + (has_old ? (size_t)S : 0);
}

// Stage A-row entries [p0, p0 + cnt): B-row offset k*B.w, a_ik, nnz_B(k), cursor.
__device__ __forceinline__ void stage_piece(const RowOpParams& p, const WarpSmem& w, int lane,
                                            const int32_t* a_col, const double* a_val, int p0, int cnt,
                                            const int32_t* cur) {
    for (int q = lane; q < cnt; q += 32) {
        const int k = a_col[p0 + q];
        const long long bo = (long long)k * p.B.w;
        asm volatile("st.shared.s64 [%0], %1;" ::"r"(w.stg + 8u * q), "l"(bo) : "memory");
        sts64(w.stg + 8u * (kStage + q), a_val[p0 + q]);
        sts32i(stg_anb_a(w, q), __ldg(p.B.nnz + k));
        sts32i(stg_ast_a(w, q), cur ? cur[p0 + q] : 0);
        sts32i(stg_ak_a(w, q), k);
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------- fast path

// Accumulate the staged steps [0, cnt) into the window [c0, c0 + S). The host's probe
// guarantees (i) every product column lies inside the window and (ii) every B row has at
// most 64*G entries, so a step is a fixed, branch-free block: each lane takes entries
// 2*lane, 2*lane+1 of each 64-entry group (8/16-byte vector loads), forms the shared
// address acc + 8*(j - c0) with one IMAD from a per-row base (entries past nnz_B(k) are
// sent to a per-warp trash slot acc[S] instead of being predicated), then issues all 2G
// shared loads, all 2G FMAs and all 2G shared stores of the step. Ring slots hold raw
// loaded registers and are not read until the step is consumed D steps later.
template <int G, int D>
__device__ __forceinline__ void accumulate_fast(const RowOpParams& p, const WarpSmem& w, int lane, int cnt,
                                                int c0, int S) {
    int2 rc[D][G];
    double2 rv[D][G];
    double ra[D];
    int rnb[D];
    const int32_t* __restrict__ bcol = p.B.col;
    const double* __restrict__ bval = p.B.val;
    const int trash = c0 + S;                          // column that maps to acc[S]
    const uint32_t abase = w.acc - 8u * (uint32_t)c0;  // acc + 8*(j - c0) = abase + 8*j (mod 2^32)
    auto load = [&](int d, int t) {
        const long long bo = stg_boff(w, t);
        const int nb = stg_anb(w, t);
        ra[d] = stg_aa(w, t);
        rnb[d] = nb;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int q = 64 * g + 2 * lane;
            if (q < nb) {
                rc[d][g] = __ldg(reinterpret_cast<const int2*>(bcol + bo + q));
                rv[d][g] = __ldg(reinterpret_cast<const double2*>(bval + bo + q));
            }
        }
    };
#pragma unroll
    for (int d = 0; d < D; ++d)
        if (d < cnt) load(d, d);
    for (int t0 = 0; t0 < cnt; t0 += D) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const int t = t0 + d;
            if (t < cnt) {
                const double a = ra[d];
                const int nb = rnb[d];
                uint32_t ad[G][2];
                double old[G][2];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const int q = 64 * g + 2 * lane;
                    const int j0 = q < nb ? rc[d][g].x : trash;
                    const int j1 = q + 1 < nb ? rc[d][g].y : trash;
                    ad[g][0] = abase + 8u * (uint32_t)j0;
                    ad[g][1] = abase + 8u * (uint32_t)j1;
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    old[g][0] = lds64(ad[g][0]);
                    old[g][1] = lds64(ad[g][1]);
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    sts64(ad[g][0], __fma_rn(a, rv[d][g].x, old[g][0]));
                    sts64(ad[g][1], __fma_rn(a, rv[d][g].y, old[g][1]));
                }
                if (t + D < cnt) load(d, t + D);
                __syncwarp();
            }
        }
    }
}

// ------------------------------------------------------------------------- general path

// Multi-pass accumulate: entries at or beyond c0 + width are left for later passes; the
// staged cursor ast[t] advances by the in-range count.
__device__ __forceinline__ void accumulate_multi(const RowOpParams& p, const WarpSmem& w, int lane, int cnt,
                                                 int c0, int width) {
    const int32_t* __restrict__ bcol = p.B.col;
    const double* __restrict__ bval = p.B.val;
    for (int t = 0; t < cnt; ++t) {
        const long long bo = stg_boff(w, t);
        const int nb = stg_anb(w, t);
        const int st = stg_ast(w, t);
        const double a = stg_aa(w, t);
        int q0 = st, n_in = 0;
        while (q0 < nb) {
            const int qa = q0 + lane, qb = q0 + 32 + lane;
            const int ja = qa < nb ? __ldg(bcol + bo + qa) : INT_MAX;
            const int jb = qb < nb ? __ldg(bcol + bo + qb) : INT_MAX;
            const unsigned oa = (unsigned)(ja - c0), ob = (unsigned)(jb - c0);
            const bool ia = oa < (unsigned)width, ib = ob < (unsigned)width;
            const double va = ia ? __ldg(bval + bo + qa) : 0.0;
            const double vb = ib ? __ldg(bval + bo + qb) : 0.0;
            double xa = 0.0, xb = 0.0;
            if (ia) xa = lds64(w.acc + oa * 8u);
            if (ib) xb = lds64(w.acc + ob * 8u);
            if (ia) sts64(w.acc + oa * 8u, __fma_rn(a, va, xa));
            if (ib) sts64(w.acc + ob * 8u, __fma_rn(a, vb, xb));
            const int n = __popc(__ballot_sync(FULL, ia)) + __popc(__ballot_sync(FULL, ib));
            n_in += n;
            if (n < 64) break;
            q0 += 64;
        }
        if (lane == 0) sts32i(stg_ast_a(w, t), st + n_in);
        __syncwarp();
    }
}

// --------------------------------------------------------------------- combine and emit

// Combine Old entries with columns in [c0, c0 + width): acc <- fma(alpha, s, beta*old), flag.
// Returns false (fast path) if an Old entry lies outside the window.
template <int MODE>
__device__ __forceinline__ bool combine_old(const RowOpParams& p, const WarpSmem& w, int lane,
                                            const int32_t* o_col, const double* o_val, int nOld,
                                            int& old_cur, int c0, int width, bool multi, double& nrm) {
    bool ok = true;
    while (old_cur < nOld) {
        const int q = old_cur + lane;
        const bool v = q < nOld;
        const int j = v ? o_col[q] : INT_MAX;
        const unsigned off = (unsigned)(j - c0);
        const bool inr = v && off < (unsigned)width;
        if (v && !inr && !multi) ok = false;
        if (inr) {
            const double x = o_val[q];
            const double s = lds64(w.acc + off * 8u);
            if (MODE == 2) {
                const double df = __dsub_rn(s, x);
                nrm = __fma_rn(df, df, nrm);
            }
            const double tt = (p.old_mode == 1) ? __dmul_rn(p.beta, x) : 0.0;
            sts64(w.acc + off * 8u, __fma_rn(p.alpha, s, tt));
            sts8(w.flg + off, 1u);
        }
        const int n = __popc(__ballot_sync(FULL, inr));
        old_cur += n;
        if (n < 32) break;
    }
    __syncwarp();
    return __all_sync(FULL, ok);
}

// Emit window slots [0, width) (columns c0 + jj): drop, compact, write into the C row at
// `kept`; clears the window (and flags). One slot per lane per sub-step (four sub-steps per
// iteration), so every ballot-compacted run is a contiguous, coalesced store. Slots for
// columns >= N hold +0 and are never kept (tau >= 0). The stored diagonal c_ii is read by
// the caller before the emit (window_diag).
template <int MODE, bool A1>
__device__ __forceinline__ void emit_window_t(const RowOpParams& p, const WarpSmem& w, int lane,
                                              double* __restrict__ crow_v, int32_t* __restrict__ crow_c,
                                              int c0, int width, int& kept, double& nrm) {
    const unsigned lt_mask = (1u << lane) - 1u;
    const int cw = p.C.w;
    const double tau = p.tau, alpha = p.alpha;
    for (int b = 0; b < width; b += 128) {
        double v[4];
        uint32_t f[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int jj = b + 32 * s + lane;
            v[s] = 0.0;
            f[s] = 0;
            if (jj < width) {
                const uint32_t ad = w.acc + (uint32_t)jj * 8u;
                v[s] = lds64(ad);
                sts64(ad, 0.0);
                if (MODE != 0) {
                    f[s] = lds8(w.flg + jj);
                    sts8(w.flg + jj, 0u);
                }
            }
        }
        double x[4];
        unsigned m[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            x[s] = v[s];
            if (MODE == 0 || !f[s]) {
                if (!A1) x[s] = __dmul_rn(alpha, v[s]);
                if (MODE == 2) nrm = __fma_rn(v[s], v[s], nrm);
            }
            m[s] = __ballot_sync(FULL, fabs(x[s]) > tau);
        }
        // positions of the four runs are independent: no serial dependence on `kept`
        int before = kept;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int pos = before + __popc(m[s] & lt_mask);
            st_entry(((m[s] >> lane) & 1u) && pos < cw, crow_v + pos, crow_c + pos, x[s], c0 + b + 32 * s + lane);
            before += __popc(m[s]);
        }
        kept = before;
    }
    __syncwarp();
}

template <int MODE>
__device__ __forceinline__ void emit_window(const RowOpParams& p, const WarpSmem& w, int lane,
                                            double* __restrict__ crow_v, int32_t* __restrict__ crow_c,
                                            int c0, int width, int& kept, double& nrm) {
    if (p.alpha == 1.0) emit_window_t<MODE, true>(p, w, lane, crow_v, crow_c, c0, width, kept, nrm);
    else emit_window_t<MODE, false>(p, w, lane, crow_v, crow_c, c0, width, kept, nrm);
}

// Stored (post-combine, post-drop) value of window slot jd, or 0 (read before the emit).
template <int MODE>
__device__ __forceinline__ double window_diag(const RowOpParams& p, const WarpSmem& w, int jd, int width) {
    if (jd < 0 || jd >= width) return 0.0;
    double x = lds64(w.acc + (uint32_t)jd * 8u);
    const bool flagged = MODE != 0 && lds8(w.flg + jd) != 0;
    if (!flagged && p.alpha != 1.0) x = __dmul_rn(p.alpha, x);
    return fabs(x) > p.tau ? x : 0.0;
}

// Zero the window (after an abandoned fast-path attempt / at start).
template <int MODE>
__device__ __forceinline__ void clear_window(const WarpSmem& w, int lane, int S) {
    for (int jj = 2 * lane; jj < S; jj += 64) {
        sts128(w.acc + (uint32_t)jj * 8u, 0.0, 0.0);
        if (MODE != 0) sts16u(w.flg + jj, 0u);
    }
    __syncwarp();
}

// ------------------------------------------------------------------- ring fast path
//
// Row-centred windows need 2(hA + hB) + 1 doubles per row. The k-sweep is ascending, and
// step k touches only columns [k - hB, k + hB], so once step k starts every column below
// k - hB is final. The fast path therefore keeps a RING of S >= 2 hB + 33 slots (column j
// lives in slot j mod S, S a multiple of 32) and emits finished 32-column chunks as the
// sweep advances ("progressive emission"): before step k, chunks below floor32(k - hB) are
// combined with Old, dropped, compacted and written, and their slots cleared, so the live
// span never exceeds S. Half the shared memory of a full window for X^2 (hA = hB), hence
// twice the rows in flight per SM. Each step is software-pipelined over a (D+1)-slot
// register ring: the gathers for step t + D are issued before step t's FMAs.

// Emit NCH consecutive 32-column chunks [F, F + 32 NCH) (column j lives in ring slot
// j - baseF, minus S past the wrap): pre-combine diagonal, combine with Old, drop, compact
// (NCH independent ballots) and write; the slots (and flags) are cleared.
template <int MODE, int NCH>
__device__ __forceinline__ void ring_emit_block(const RowOpParams& p, const WarpSmem& w, int lane, int64_t i,
                                                int F, int baseF, const int32_t* o_col, const double* o_val,
                                                int nOld, int& old_cur, double* __restrict__ crow_v,
                                                int32_t* __restrict__ crow_c, int& kept, double& ds, double& dc,
                                                double& nrm) {
    const int S = p.S;
    const int Fe = F + 32 * NCH;
    if ((int64_t)F <= i && i < (int64_t)Fe) {
        int pi = (int)(i - baseF);
        if (pi >= S) pi -= S;
        ds = lds64(w.acc + 8u * (uint32_t)pi);
    }
    if (MODE != 0) {
        while (old_cur < nOld) {
            const int q = old_cur + lane;
            const bool v = q < nOld;
            const int jo = v ? o_col[q] : INT_MAX;
            const bool inr = jo < Fe;
            if (inr) {
                const double x = o_val[q];
                int po = jo - baseF;
                if (po >= S) po -= S;
                const uint32_t sa = w.acc + 8u * (uint32_t)po;
                const double sv = lds64(sa);
                if (MODE == 2) {
                    const double df = __dsub_rn(sv, x);
                    nrm = __fma_rn(df, df, nrm);
                }
                const double tt = (p.old_mode == 1) ? __dmul_rn(p.beta, x) : 0.0;
                sts64(sa, __fma_rn(p.alpha, sv, tt));
                sts8(w.flg + (uint32_t)po, 1u);
            }
            const int n = __popc(__ballot_sync(FULL, inr));
            old_cur += n;
            if (n < 32) break;
        }
        __syncwarp();
    }
    double x[NCH];
    unsigned m[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        int pc = F + 32 * c - baseF;
        if (pc >= S) pc -= S;
        const uint32_t pa = w.acc + 8u * (uint32_t)(pc + lane);
        const double v = lds64(pa);
        sts64(pa, 0.0);
        bool flagged = false;
        if (MODE != 0) {
            const uint32_t fa = w.flg + (uint32_t)(pc + lane);
            flagged = lds8(fa) != 0;
            sts8(fa, 0u);
        }
        x[c] = v;
        if (!flagged) {
            if (p.alpha != 1.0) x[c] = __dmul_rn(p.alpha, v);
            if (MODE == 2) nrm = __fma_rn(v, v, nrm);
        }
        m[c] = __ballot_sync(FULL, fabs(x[c]) > p.tau);
    }
    const unsigned lt = (1u << lane) - 1u;
    int before = kept;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const bool keep = (m[c] >> lane) & 1u;
        const int pos = before + __popc(m[c] & lt);
        st_entry(keep && pos < p.C.w, crow_v + pos, crow_c + pos, x[c], F + 32 * c + lane);
        if ((int64_t)F + 32 * c + lane == i) dc = keep ? x[c] : 0.0;
        before += __popc(m[c]);
    }
    kept = before;
}

// Emit [F, Fto) (multiples of 32), four chunks at a time where possible; advances F, baseF.
template <int MODE>
__device__ __forceinline__ void ring_emit_range(const RowOpParams& p, const WarpSmem& w, int lane, int64_t i,
                                                int& F, int& baseF, int Fto, const int32_t* o_col,
                                                const double* o_val, int nOld, int& old_cur,
                                                double* __restrict__ crow_v, int32_t* __restrict__ crow_c,
                                                int& kept, double& ds, double& dc, double& nrm) {
    while (p.S >= 256 && F + 128 <= Fto) {  // a 128-column block wraps at most once
        ring_emit_block<MODE, 4>(p, w, lane, i, F, baseF, o_col, o_val, nOld, old_cur, crow_v, crow_c, kept, ds,
                                 dc, nrm);
        F += 128;
        while (F - baseF >= p.S) baseF += p.S;
    }
    while (F < Fto) {
        ring_emit_block<MODE, 1>(p, w, lane, i, F, baseF, o_col, o_val, nOld, old_cur, crow_v, crow_c, kept, ds,
                                 dc, nrm);
        F += 32;
        if (F - baseF >= p.S) baseF += p.S;
    }
    __syncwarp();
}

// Emission state of a ring row (kept in registers; copied by value through the rare
// out-of-line fallback so the unrolled step loop stays small).
struct EmitState {
    int F, baseF, old_cur, kept;
    double ds, dc, nrm;
};

template <int MODE>
__device__ __noinline__ EmitState ring_emit_fallback(const RowOpParams& p, WarpSmem w, int lane, int64_t i,
                                                      EmitState st, int target, const int32_t* o_col,
                                                      const double* o_val, int nOld, double* crow_v,
                                                      int32_t* crow_c) {
    ring_emit_range<MODE>(p, w, lane, i, st.F, st.baseF, target, o_col, o_val, nOld, st.old_cur, crow_v, crow_c,
                          st.kept, st.ds, st.dc, st.nrm);
    return st;
}

template <int G, int D, int MODE>
__device__ __forceinline__ void row_ring(const RowOpParams& p, const WarpSmem& w, int lane, int64_t i,
                                         const int32_t* a_col, const double* a_val, int nA,
                                         const int32_t* o_col, const double* o_val, int nOld,
                                         double* __restrict__ crow_v, int32_t* __restrict__ crow_c,
                                         int& kept, double& ds, double& dc, double& nrm) {
    constexpr int NS = D + 1;  // register ring slots
    const int S = p.S;
    const int hB = p.hB;
    const int ncols = (int)p.ncols;
    (void)ncols;
    // column extent of the row: products in [k_first - hB, k_last + hB], plus Old entries
    int lo_col = INT_MAX, hi_col = -1;
    if (nA > 0) {
        lo_col = max(0, a_col[0] - hB);
        hi_col = min(ncols - 1, a_col[nA - 1] + hB);
    }
    if (MODE != 0 && nOld > 0) {
        lo_col = min(lo_col, o_col[0]);
        hi_col = max(hi_col, o_col[nOld - 1]);
    }
    if (hi_col < lo_col) return;
    int F = lo_col & ~31;
    const int Fend = (hi_col + 32) & ~31;
    int baseF = F - F % S;  // multiple of S with baseF <= F < baseF + S
    int baseS = baseF;
    int old_cur = 0;
    const uint32_t trash = w.acc + 8u * (uint32_t)S;
    const int32_t* __restrict__ bcol = p.B.col;
    const double* __restrict__ bval = p.B.val;

    int2 rc[NS][G];
    double2 rv[NS][G];
    double ra[NS];
    int rnb[NS], rk[NS];
#ifdef ELL_TIMING
    long long t_row0 = clock64(), t_em = 0;
#endif
    for (int p0 = 0; p0 < nA; p0 += kStage) {
        const int cnt = min(kStage, nA - p0);
        stage_piece(p, w, lane, a_col, a_val, p0, cnt, nullptr);
        auto load = [&](int slot, int t) {
            const long long bo = stg_boff(w, t);
            const int nb = stg_anb(w, t);
            ra[slot] = stg_aa(w, t);
            rnb[slot] = nb;
            rk[slot] = stg_ak(w, t);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int q = 64 * g + 2 * lane;
                if (q < nb) {
                    rc[slot][g] = __ldg(reinterpret_cast<const int2*>(bcol + bo + q));
                    rv[slot][g] = __ldg(reinterpret_cast<const double2*>(bval + bo + q));
                }
            }
        };
#pragma unroll
        for (int d = 0; d < D; ++d)
            if (d < cnt) load(d, d);
        for (int t0 = 0; t0 < cnt; t0 += NS) {
            {
                // 1. once per block of NS steps: emit every final column (< floor32(k_t0 - hB));
                //    the ring's slack normally covers the block's k advance
                const int target = (rk[0] - hB) & ~31;
                if (target > F) {
#ifdef ELL_TIMING
                    long long te0 = clock64();
#endif
                    ring_emit_range<MODE>(p, w, lane, i, F, baseF, target, o_col, o_val, nOld, old_cur, crow_v,
                                          crow_c, kept, ds, dc, nrm);
#ifdef ELL_TIMING
                    t_em += clock64() - te0;
#endif
                }
            }
#pragma unroll
            for (int d = 0; d < NS; ++d) {
                const int t = t0 + d;
                if (t < cnt) {
                    const int kt = rk[d];
                    // 1b. rare: step k would reach a slot still holding an unemitted column
                    if (kt + hB >= F + S) {
                        EmitState st{F, baseF, old_cur, kept, ds, dc, nrm};
                        st = ring_emit_fallback<MODE>(p, w, lane, i, st, (kt - hB) & ~31, o_col, o_val, nOld,
                                                      crow_v, crow_c);
                        F = st.F; baseF = st.baseF; old_cur = st.old_cur; kept = st.kept;
                        ds = st.ds; dc = st.dc; nrm = st.nrm;
                    }
                    // 2. ring slot mapping for this step: columns [lo, k + hB], lo >= baseS
                    const int lo = max(0, kt - hB);
                    while (lo - baseS >= S) baseS += S;
                    const uint32_t abase = w.acc - 8u * (uint32_t)baseS;
                    const int jw = baseS + S;
                    const int nb = rnb[d];
                    const double a = ra[d];
                    uint32_t ad[G][2];
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const int q = 64 * g + 2 * lane;
                        const int j0 = rc[d][g].x, j1 = rc[d][g].y;
                        uint32_t a0 = abase + 8u * (uint32_t)j0 - (j0 >= jw ? 8u * (uint32_t)S : 0u);
                        uint32_t a1 = abase + 8u * (uint32_t)j1 - (j1 >= jw ? 8u * (uint32_t)S : 0u);
                        ad[g][0] = q < nb ? a0 : trash;
                        ad[g][1] = q + 1 < nb ? a1 : trash;
                    }
                    // 3. shared loads of the step
                    double old[G][2];
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        old[g][0] = lds64(ad[g][0]);
                        old[g][1] = lds64(ad[g][1]);
                    }
                    // 4. gathers for step t + D into the slot freed by step t - 1
                    if (t + D < cnt) load((d + D) % NS, t + D);
                    // 5. fma + shared stores
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        sts64(ad[g][0], __fma_rn(a, rv[d][g].x, old[g][0]));
                        sts64(ad[g][1], __fma_rn(a, rv[d][g].y, old[g][1]));
                    }
                    __syncwarp();
                }
            }
        }
    }
    // final chunks
#ifdef ELL_TIMING
    long long te1 = clock64();
#endif
    ring_emit_range<MODE>(p, w, lane, i, F, baseF, Fend, o_col, o_val, nOld, old_cur, crow_v, crow_c, kept, ds,
                          dc, nrm);
#ifdef ELL_TIMING
    long long te2 = clock64();
    t_em += te2 - te1;
    if (lane == 0 && p.timing) {
        unsigned long long* T = p.timing + 8 * (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
        atomicAdd(T + 0, 0ull);
        atomicAdd(T + 1, (unsigned long long)(te2 - t_row0 - t_em));
        atomicAdd(T + 2, (unsigned long long)t_em);
        atomicAdd(T + 3, 1ull);
        atomicAdd(T + 4, (unsigned long long)nA);
    }
#endif
    dc = warp_sum(dc);  // only the diagonal's lane holds a nonzero value (x + 0 = x exactly)
    ds = ds;            // ds is warp-uniform (broadcast shared load)
}

// -------------------------------------------------------------------------------- kernel

// Per-warp shared layout setup (window/ring + stage + flags).
template <int MODE>
__device__ __forceinline__ WarpSmem warp_smem(unsigned char* smem_raw, int wid, int S) {
    unsigned char* base = smem_raw + (size_t)wid * warp_smem_bytes(S, MODE != 0);
    WarpSmem w;
    w.acc = (uint32_t)__cvta_generic_to_shared(base);
    w.stg = w.acc + (uint32_t)((S + 2) * 8);
    w.flg = w.acc + (uint32_t)((S + 2) * 8 + kStage * 28);
    return w;
}

struct RowIO {
    const double* a_val;
    const int32_t* a_col;
    int32_t nA;
    const double* o_val;
    const int32_t* o_col;
    int32_t nOld;
    double* crow_v;
    int32_t* crow_c;
};

template <int MODE>
__device__ __forceinline__ RowIO row_io(const RowOpParams& p, int64_t i) {
    RowIO r;
    r.a_val = p.A.val + (size_t)i * p.A.w;
    r.a_col = p.A.col + (size_t)i * p.A.w;
    r.nA = (p.alpha != 0.0) ? p.A.nnz[i] : 0;
    r.o_val = nullptr;
    r.o_col = nullptr;
    r.nOld = 0;
    if (MODE != 0) {
        r.o_val = p.Old.val + (size_t)i * p.Old.w;
        r.o_col = p.Old.col + (size_t)i * p.Old.w;
        r.nOld = p.Old.nnz[i];
    }
    r.crow_v = p.C.val + (size_t)i * p.C.w;
    r.crow_c = p.C.col + (size_t)i * p.C.w;
    return r;
}

// stored diagonal of A (x2 traces), warp-uniform result
__device__ __forceinline__ double stored_diag_a(const RowIO& r, int lane, int64_t i) {
    double dA = 0.0;
    bool has = false;
    for (int q = lane; q < r.nA; q += 32)
        if (r.a_col[q] == (int)i) { dA = r.a_val[q]; has = true; }
    const unsigned m = __ballot_sync(FULL, has);
    return m ? __shfl_sync(FULL, dA, __ffs(m) - 1) : 0.0;
}

template <int MODE>
__device__ __forceinline__ void row_epilogue(const RowOpParams& p, int lane, int64_t i, int32_t kept, double dA,
                                             double ds, double dc, double nrm, int32_t& my_max_kept,
                                             int32_t& my_ovf) {
    if (lane == 0) p.C.nnz[i] = kept < p.C.w ? kept : p.C.w;
    my_max_kept = max(my_max_kept, kept);
    if (kept > p.C.w) ++my_ovf;
    if (p.diag_c && lane == 0) p.diag_c[i] = dc;
    if (p.diag_s && lane == 0) p.diag_s[i] = ds;
    if (p.diag_a && lane == 0) p.diag_a[i] = dA;
    if (MODE == 2 && p.normsq) {
        nrm = warp_sum(nrm);
        if (lane == 0) p.normsq[i] = nrm;
    }
}

__device__ __forceinline__ void flush_status(const RowOpParams& p, int lane, int32_t my_max_kept, int32_t my_ovf) {
    if (lane == 0) {
        if (my_ovf) atomicAdd(p.status + 0, my_ovf);
        if (my_max_kept) atomicMax(p.status + 1, my_max_kept);
    }
}

// Fast kernel: ring window, every row single-pass (host-verified: ring >= 2 hB + 33,
// B rows <= 64 G entries).
template <int G, int D, int MODE>
__global__ void __launch_bounds__(128, 1) row_fast_kernel(const RowOpParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const WarpSmem w = warp_smem<MODE>(smem_raw, wid, p.S);
    clear_window<MODE>(w, lane, p.S);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    int32_t my_max_kept = 0, my_ovf = 0;
    for (int64_t i = p.row_begin + gw; i < p.row_end; i += nwarps) {
        RowIO r = row_io<MODE>(p, i);
        const double dA = p.diag_a ? stored_diag_a(r, lane, i) : 0.0;
        if (p.stash_a || p.stash_old) {
            // C aliases an input and rows are emitted progressively: copy the input rows aside first
            double* sv = p.st_val + gw * p.st_stride;
            int32_t* sc = p.st_col + gw * p.st_stride;
            if (p.stash_a) {
                for (int q = lane; q < r.nA; q += 32) { sv[q] = r.a_val[q]; sc[q] = r.a_col[q]; }
                r.a_val = sv; r.a_col = sc;
                sv += p.A.w; sc += p.A.w;
            }
            if (MODE != 0 && p.stash_old) {
                for (int q = lane; q < r.nOld; q += 32) { sv[q] = r.o_val[q]; sc[q] = r.o_col[q]; }
                r.o_val = sv; r.o_col = sc;
            }
            __syncwarp();
        }
        int32_t kept = 0;
        double ds = 0.0, dc = 0.0, nrm = 0.0;
        row_ring<G, D, MODE>(p, w, lane, i, r.a_col, r.a_val, r.nA, r.o_col, r.o_val, r.nOld, r.crow_v, r.crow_c,
                             kept, ds, dc, nrm);
        row_epilogue<MODE>(p, lane, i, kept, dA, ds, dc, nrm, my_max_kept, my_ovf);
    }
    flush_status(p, lane, my_max_kept, my_ovf);
}

// General kernel: span pre-pass + ceil(span / S) passes of an S-double window with per-k
// cursors (rows wider than any ring that fits shared memory, B rows > 256 entries).
template <int MODE>
__global__ void __launch_bounds__(128, 1) row_general_kernel(const RowOpParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int S = p.S;
    const WarpSmem w = warp_smem<MODE>(smem_raw, wid, S);
    clear_window<MODE>(w, lane, S);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    int32_t my_max_kept = 0, my_ovf = 0;
    for (int64_t i = p.row_begin + gw; i < p.row_end; i += nwarps) {
        RowIO r = row_io<MODE>(p, i);
        const double* a_val = r.a_val;
        const int32_t* a_col = r.a_col;
        const double* o_val = r.o_val;
        const int32_t* o_col = r.o_col;
        const int32_t nA = r.nA, nOld = r.nOld;
        double* crow_v = r.crow_v;
        int32_t* crow_c = r.crow_c;
        const double dA = p.diag_a ? stored_diag_a(r, lane, i) : 0.0;
        int32_t kept = 0;
        double ds = 0.0, dc = 0.0, nrm = 0.0;
        {
            // ---- general path: span pre-pass + ceil(span / S) passes with cursors
            int lo = INT_MAX, hi = -1;
            for (int q = lane; q < nA; q += 32) {
                const int k = a_col[q];
                const int nb = __ldg(p.B.nnz + k);
                if (nb > 0) {
                    const int32_t* bc = p.B.col + (size_t)k * p.B.w;
                    lo = min(lo, __ldg(bc));
                    hi = max(hi, __ldg(bc + nb - 1));
                }
            }
            if (MODE != 0 && nOld > 0 && lane == 0) {
                lo = min(lo, o_col[0]);
                hi = max(hi, o_col[nOld - 1]);
            }
            lo = warp_min(lo) & ~1;  // even window start (16-byte slot pairs)
            hi = warp_max(hi);
            if (hi >= lo) {
                const int span = hi - lo + 1;
                const int npass = (span + S - 1) / S;
                const bool multi = npass > 1;
                int32_t* cur = p.cursors ? p.cursors + gw * p.cur_stride : nullptr;
                if (multi && (p.stash_a || p.stash_old)) {
                    double* sv = p.st_val + gw * p.st_stride;
                    int32_t* sc = p.st_col + gw * p.st_stride;
                    if (p.stash_a) {
                        for (int q = lane; q < nA; q += 32) { sv[q] = a_val[q]; sc[q] = a_col[q]; }
                        a_val = sv; a_col = sc;
                        sv += p.A.w; sc += p.A.w;
                    }
                    if (MODE != 0 && p.stash_old) {
                        for (int q = lane; q < nOld; q += 32) { sv[q] = o_val[q]; sc[q] = o_col[q]; }
                        o_val = sv; o_col = sc;
                    }
                    __syncwarp();
                }
                if (multi)
                    for (int q = lane; q < nA; q += 32) cur[q] = 0;
                __syncwarp();
                int old_cur = 0;
                for (int pass = 0; pass < npass; ++pass) {
                    const int c0 = lo + pass * S;
                    const int width = min(S, hi + 2 - c0) & ~1;  // even, covers [c0, hi]
                    for (int p0 = 0; p0 < nA; p0 += kStage) {
                        const int cnt = min(kStage, nA - p0);
                        stage_piece(p, w, lane, a_col, a_val, p0, cnt, multi ? cur : nullptr);
                        accumulate_multi(p, w, lane, cnt, c0, width);
                        if (multi) {
                            for (int q = lane; q < cnt; q += 32) cur[p0 + q] = stg_ast(w, q);
                            __syncwarp();
                        }
                    }
                    __syncwarp();
                    if ((int64_t)c0 <= i && i < (int64_t)c0 + width) ds = lds64(w.acc + (uint32_t)(i - c0) * 8u);
                    if (MODE != 0) combine_old<MODE>(p, w, lane, o_col, o_val, nOld, old_cur, c0, width, true, nrm);
                    if (p.diag_c && (int64_t)c0 <= i && i < (int64_t)c0 + width)
                        dc = window_diag<MODE>(p, w, (int)(i - c0), width);
                    emit_window<MODE>(p, w, lane, crow_v, crow_c, c0, width, kept, nrm);
                }
            }
        }

        row_epilogue<MODE>(p, lane, i, kept, dA, ds, dc, nrm, my_max_kept, my_ovf);
    }
    flush_status(p, lane, my_max_kept, my_ovf);
}

// Half-bandwidth probe: out[m] = max over rows of max(i - col[i][0], col[i][nnz-1] - i).
__global__ void bandwidth_kernel(KMat a, KMat b, KMat c, int64_t r0, int64_t r1, int64_t n, int32_t* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int bw[3] = {0, 0, 0};
    const KMat* ms[3] = {&a, &b, &c};
    if (i < n) {
#pragma unroll
        for (int m = 0; m < 3; ++m) {
            // A and Old only matter on the computed rows; B on every row
            if (m != 1 && (i < r0 || i >= r1)) continue;
            const KMat& x = *ms[m];
            if (x.nnz == nullptr) continue;
            const int nz = x.nnz[i];
            if (nz > 0) {
                const int f = x.col[(size_t)i * x.w], l = x.col[(size_t)i * x.w + nz - 1];
                bw[m] = max(max((int)(i - f), (int)(l - i)), 0);
            }
        }
    }
    int nzb = (i < n) ? b.nnz[i] : 0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        int v = m < 3 ? bw[m] : nzb;
#pragma unroll
        for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
        if ((threadIdx.x & 31) == 0 && v > 0) atomicMax(out + m, v);
    }
}

cudaError_t launch_bandwidth(KMat a, KMat b, KMat c, int nmat, int64_t r0, int64_t r1, int64_t n,
                             int32_t* out, cudaStream_t s) {
    (void)nmat;
    bandwidth_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, b, c, r0, r1, n, out);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------- dispatch

// Fast-kernel variants by G = ceil(max nnz_B / 64) (64-entry groups per step; prefetch
// depth D, the register ring holds D + 1 slots): G1: D 8, G2: D 6, G3: D 4, G4: D 3.
// cfg.R carries G; cfg.R == 0 selects the general kernel.
template <typename K>
static cudaError_t prep_kernel(K kern, const LaunchCfg& cfg, int* bps) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.smem);
    if (e) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, kern, cfg.warps_per_cta * 32, cfg.smem);
}

template <int MODE>
static cudaError_t prep_mode(const LaunchCfg& cfg, int* bps) {
    switch (cfg.R) {
        case 0: return prep_kernel(row_general_kernel<MODE>, cfg, bps);
        case 1: return prep_kernel(row_fast_kernel<1, 8, MODE>, cfg, bps);
        case 2: return prep_kernel(row_fast_kernel<2, 6, MODE>, cfg, bps);
        case 3: return prep_kernel(row_fast_kernel<3, 4, MODE>, cfg, bps);
        default: return prep_kernel(row_fast_kernel<4, 3, MODE>, cfg, bps);
    }
}

template <int MODE>
static void launch_mode(const RowOpParams& p, const LaunchCfg& cfg, cudaStream_t s) {
    dim3 block(cfg.warps_per_cta * 32), grid(cfg.grid);
    switch (cfg.R) {
        case 0: row_general_kernel<MODE><<<grid, block, cfg.smem, s>>>(p); break;
        case 1: row_fast_kernel<1, 8, MODE><<<grid, block, cfg.smem, s>>>(p); break;
        case 2: row_fast_kernel<2, 6, MODE><<<grid, block, cfg.smem, s>>>(p); break;
        case 3: row_fast_kernel<3, 4, MODE><<<grid, block, cfg.smem, s>>>(p); break;
        default: row_fast_kernel<4, 3, MODE><<<grid, block, cfg.smem, s>>>(p); break;
    }
}

static int mode_of(const RowOpParams& p) { return p.old_mode == 0 ? 0 : (p.normsq ? 2 : 1); }

size_t row_op_warp_smem(int S, bool has_old) { return warp_smem_bytes(S, has_old); }

cudaError_t plan_row_op(const RowOpParams& p, int S, int groups, int warps_opt, int num_sms, LaunchCfg* cfg) {
    S = (S + 31) & ~31;
    const size_t per_warp = warp_smem_bytes(S, p.old_mode != 0);
    const size_t cap = 227 * 1024;
    if (per_warp > cap) return cudaErrorInvalidConfiguration;
    cfg->S = S;
    cfg->R = !p.fast ? 0 : (groups < 1 ? 1 : (groups > 4 ? 4 : groups));
    const int mode = mode_of(p);
    // warps per CTA: maximise resident warps (rows in flight) per SM under the shared-memory
    // and register limits; ties go to the larger CTA
    int best_w = 0, best_wpc = 1, best_bps = 0;
    const int lo_w = warps_opt > 0 ? warps_opt : 1, hi_w = warps_opt > 0 ? warps_opt : 4;
    for (int wpc = hi_w; wpc >= lo_w; --wpc) {
        if ((size_t)wpc * per_warp > cap) continue;
        cfg->warps_per_cta = wpc;
        cfg->smem = (size_t)wpc * per_warp;
        int bps = 0;
        cudaError_t e = mode == 0 ? prep_mode<0>(*cfg, &bps) : mode == 1 ? prep_mode<1>(*cfg, &bps)
                                                                          : prep_mode<2>(*cfg, &bps);
        if (e) return e;
        if (bps * wpc > best_w) { best_w = bps * wpc; best_wpc = wpc; best_bps = bps; }
    }
    if (best_w < 1) return cudaErrorInvalidConfiguration;
    const int wpc = best_wpc, bps = best_bps;
    cfg->warps_per_cta = wpc;
    cfg->smem = (size_t)wpc * per_warp;
    {
        int dummy = 0;
        cudaError_t e = mode == 0 ? prep_mode<0>(*cfg, &dummy) : mode == 1 ? prep_mode<1>(*cfg, &dummy)
                                                                            : prep_mode<2>(*cfg, &dummy);
        if (e) return e;
    }
    const int64_t rows = p.row_end - p.row_begin;
    const int64_t need = (rows + wpc - 1) / wpc;
    const int64_t full = (int64_t)bps * num_sms;
    cfg->grid = (int)(need < full ? (need > 0 ? need : 1) : full);
    return cudaSuccess;
}

cudaError_t launch_row_op(const RowOpParams& p, const LaunchCfg& cfg, cudaStream_t s) {
    const int mode = mode_of(p);
    if (mode == 0) launch_mode<0>(p, cfg, s);
    else if (mode == 1) launch_mode<1>(p, cfg, s);
    else launch_mode<2>(p, cfg, s);
    return cudaGetLastError();
}

}  // namespace ell
