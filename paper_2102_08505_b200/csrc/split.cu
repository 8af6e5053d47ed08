// split.cu — the split-row ring kernel of libellpack (sm_100a, FP64 CUDA cores): W warps per
// output row (BJ north_star (1): "a warp or small CTA owns each output row").
//
// Same method as the ring path of spgemm.cu (readings R3, R5, R12):
// row i's products lie in columns [k - hB, k + hB] for the k of A_i in ascending order; column j
// accumulates in ring slot j mod S as the fma chain s <- fma(a_ik, b_kj, s) in ascending k; every
// column below the sweep's floor is final and is combined with Old, dropped (|c| > tau kept),
// compacted and written ("progressive emission"). What differs is who does the work:
//
//  * Column ownership. The row's CTA has W warps; 32-column chunk c = j >> 5 belongs to warp
//    c mod W. Every warp walks ALL k of A_i in ascending order but applies only the entries of
//    B row k in its own chunks, so each output entry is still one fma chain in ascending k, in one
//    warp (bitwise the oracle's), and no two warps ever touch the same ring slot (S is a multiple
//    of 32 W). The per-step work of a row is split W ways while the ring (the row's shared-memory
//    footprint) stays one ring: W times the warps per SM at the same shared memory, which is what
//    the accumulator needs (tools/microbench.cu: random FP64 smem read-modify-write 311 Gupd/s at
//    6 warps/SM vs 570 at 12 and 690 at 24, profiles/r02_microbench.json).
//  * Emission in 128-column blocks (S a multiple of 128, blocks 128-aligned: a block never wraps).
//    Warp w emits its NCH = 4 / W chunks of the block; the kept counts of the block's 4 chunks are
//    exchanged through shared memory (one named barrier per block), so every warp knows where its
//    runs go in the output row and the row stays one contiguous ascending run.
//  * B is read from a per-owner bank-balanced copy with 16-bit ring slots: B row k, owner w is a
//    record of 64 G entries (uint16 byte offset 8 (j mod S) | f64 value), 10 bytes per product
//    gathered instead of 12.
//
// Template parameters: W (warps per row: 1, 2), G (64-entry groups per sub-record step), HB
// (steps per register half), MODE (0: no Old; 1: Old operand; 2: Old + ||S - Old||^2).
#include "internal.cuh"
#include "devutil.cuh"

#include <climits>
#include <type_traits>

namespace ell {

#ifndef ELL_SPLIT_STAGE
#define ELL_SPLIT_STAGE 128  // A-row steps staged per warp: 128 measured 1-2 % faster than 64 after the lean emission
#endif
#ifndef ELL_SPLIT_META
#define ELL_SPLIT_META 0  // W = 1: the next half's step metadata read into registers one half ahead
#endif
#ifndef ELL_SPLIT_LEAN_EMIT
#define ELL_SPLIT_LEAN_EMIT 1  // W = 1: emission without per-block diagonal work (round 2)
#endif
#ifndef ELL_SPLIT_EMITN
#define ELL_SPLIT_EMITN 2  // W = 1, no Old, G >= 2: blocks emitted together when that many are pending
#endif
#ifndef ELL_SPLIT_CLEAR_STS
#define ELL_SPLIT_CLEAR_STS 0  // W = 1 lean emission: read + store zero instead of atom.exch
#endif
#ifndef ELL_SPLIT_HB_G3
#define ELL_SPLIT_HB_G3 2  // W = 1, G = 3: steps per register half
#endif
#ifndef ELL_SPLIT_HB_G2
#define ELL_SPLIT_HB_G2 3
#endif
#ifndef ELL_SPLIT_HB_G1
#define ELL_SPLIT_HB_G1 2  // measured: 1.65 vs 1.93 ms at cfg5 M = 64 (12 vs 8 rows/SM)
#endif
// W = 1: minimum resident CTAs (rows) per SM the register allocation must allow, by groups per step
// (narrow bands have small rings: registers, not shared memory, cap the rows per SM)
#ifndef ELL_SPLIT_MINB_G1
#define ELL_SPLIT_MINB_G1 16  // 128 registers, no spill: 16 rows/SM at M = 64 (S = 1408)
#endif
#ifndef ELL_SPLIT_MINB_G2
#define ELL_SPLIT_MINB_G2 6
#endif
#ifndef ELL_BAL_ATOMIC_RANK
#define ELL_BAL_ATOMIC_RANK 1  // balance pass: class ranks by shared atomics, float j mod S
#endif
#ifndef ELL_SPLIT_STAGE_G3
#define ELL_SPLIT_STAGE_G3 160  // G = 3 (cfg5 M = 256): one piece per row (<= 157 steps), 6 rows/SM kept
#endif
// A-row steps staged per warp (16 B each), by 64-entry groups per step
__host__ __device__ constexpr int split_stage(int G) { return G >= 3 ? ELL_SPLIT_STAGE_G3 : ELL_SPLIT_STAGE; }
constexpr int kSplitTrash = 16;  // trash slots S .. S + 15 (one per bank pair) for padding lanes

__host__ __device__ inline size_t split_smem_bytes(int S, int W, bool has_old, int G) {
    // acc[S + 16] f64 | stage[W][split_stage(G)] 16 B | xcnt[2][4] i32 | rowq[2] i64 | nrm[W] f64 | flags[S] u8
    return (size_t)(S + kSplitTrash) * 8 + (size_t)W * split_stage(G) * 16 + 32 + 16 + (size_t)W * 8 +
           (has_old ? (size_t)S : 0);
}

// ------------------------------------------------------------------ per-owner balanced B

// Record of B row k, owner w (chunk parity for W = 2): bt + (k W + w) * 640 G bytes:
//   uint16 slot8[64 G]: byte offset 8 (j mod S) of the entry's ring slot (padding: 8 (S + r), a
//   trash slot whose bank pair r no real entry of the same half-instruction uses), then
//   f64 val[64 G] at byte 128 G. bt_nbin[k W + w] = NB = 4 ceil(n_w / 64) used bins.
// Within a sub-record the entries are ranked by residue j mod 16 (bank pair) and dealt
// round-robin over the NB half-instruction bins (as balance_kernel in spgemm.cu): bin b is half
// (b >> 1) & 1 of group b >> 2, parity b & 1; position m in the bin -> slot
// 64 (b >> 2) + 2 (16 ((b >> 1) & 1) + m) + (b & 1). One lane's two slots of a group are adjacent:
// one 4-byte index load and one 16-byte value load per lane per group.
// NC 32-entry chunks per B row: 2G for W = 1 (nb <= 64 G), 8 for W = 2
template <int W, int NC>
__global__ void __launch_bounds__(128) balance_split_kernel(KMat b, int64_t k0, int64_t k1, int G, int S,
                                                            unsigned char* __restrict__ bt,
                                                            int32_t* __restrict__ bt_nbin) {
    static_assert((W == 1 || W == 2) && NC >= 1 && NC <= 8, "W, NC");
    __shared__ int hist_s[4][32];                             // per warp: entries per (owner, residue)
    __shared__ unsigned bmask_s[4][W][16];                    // per warp, owner, bin: bank pairs used
    __shared__ __align__(16) unsigned char rec_s[4][W][2560];  // per warp, owner: u16[256] | f64[256]
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    int* hist = hist_s[wi];
    const size_t rs = (size_t)640 * G;
#if ELL_BAL_ATOMIC_RANK
    const float invSf = 1.0f / (float)S;
#else
    const unsigned lt = (1u << lane) - 1u;
    const double invS = 1.0 / (double)S;
#endif
    for (int64_t k = k0 + (int64_t)blockIdx.x * 4 + wi; k < k1; k += (int64_t)gridDim.x * 4) {
        const int nb = b.nnz[k];  // <= 256 on the ring path
        const int32_t* __restrict__ bc = b.col + (size_t)k * b.w;
        const double* __restrict__ bv = b.val + (size_t)k * b.w;
        hist[lane] = 0;
        if (lane < W * 16) bmask_s[wi][lane >> 4][lane & 15] = 0u;
        __syncwarp();
        int jr[NC], rk[NC];
        double vr[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const int q = 32 * c + lane;
            jr[c] = q < nb ? __ldg(bc + q) : -1;
            vr[c] = q < nb ? __ldg(bv + q) : 0.0;
        }
#if ELL_BAL_ATOMIC_RANK
        // rank within the (owner, residue) class straight from a shared atomic: no warp collective
        // inside the (warp-uniform but unprovable) chunk guard. Any rank order within a class is a
        // valid dealing: each output column's fma chain is fixed by the k order of the steps alone.
#pragma unroll
        for (int c = 0; c < NC; ++c)
            rk[c] = jr[c] >= 0 ? atomicAdd(&hist[(((jr[c] >> 5) & (W - 1)) << 4) | (jr[c] & 15)], 1) : 0;
#else
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            rk[c] = 0;
            if (32 * c < nb) {  // warp-uniform
                const int key = jr[c] >= 0 ? ((((jr[c] >> 5) & (W - 1)) << 4) | (jr[c] & 15)) : 64 + lane;
                const unsigned m = __match_any_sync(FULL, key);
                const int leader = __ffs(m) - 1;
                int base = 0;
                if (lane == leader && jr[c] >= 0) base = atomicAdd(&hist[key], __popc(m));
                base = __shfl_sync(FULL, base, leader);
                rk[c] = base + __popc(m & lt);
            }
        }
#endif
        __syncwarp();
        // exclusive prefix over the residues of each owner (16-lane segments); owner totals
        const int h = hist[lane];
        int pre = h;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const int y = __shfl_up_sync(FULL, pre, o);
            if ((lane & 15) >= o) pre += y;
        }
        const int n0 = __shfl_sync(FULL, pre, 15);
        const int n1 = W > 1 ? __shfl_sync(FULL, pre, 31) : 0;
        pre -= h;
        if (lane < W) bt_nbin[k * W + lane] = 4 * (((lane ? n1 : n0) + 63) >> 6);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            if (ELL_BAL_ATOMIC_RANK || 32 * c < nb) {
                const int j = jr[c];
                const int key = j >= 0 ? ((((j >> 5) & (W - 1)) << 4) | (j & 15)) : 0;
                const int e = __shfl_sync(FULL, pre, key) + rk[c];
                if (j >= 0) {
                    const int own = key >> 4;
                    const int NB = 4 * (((own ? n1 : n0) + 63) >> 6);
                    // e / NB for e < 256, NB <= 16 by a float reciprocal: (e + 1/2) / NB is at least
                    // 1 / 32 from an integer, far above float rounding
                    const int pos = __float2int_rz(((float)e + 0.5f) * __frcp_rn((float)NB));
                    const int bin = e - pos * NB;
                    const int sl = 64 * (bin >> 2) + 2 * (16 * ((bin >> 1) & 1) + pos) + (bin & 1);
#if ELL_BAL_ATOMIC_RANK
                    // j < 2^24 is exact in float; a quotient off by one is corrected below
                    int qs = __float2int_rz(__int2float_rn(j) * invSf);
#else
                    int qs = __double2int_rz((double)j * invS);
#endif
                    int js = j - qs * S;
                    js += js < 0 ? S : 0;
                    js -= js >= S ? S : 0;
                    reinterpret_cast<uint16_t*>(rec_s[wi][own])[sl] = (uint16_t)(8 * js);
                    reinterpret_cast<double*>(rec_s[wi][own] + 512)[sl] = vr[c];
                    atomicOr(&bmask_s[wi][own][bin], 1u << (js & 15));
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int own = 0; own < W; ++own) {
            const int n = own ? n1 : n0;
            const int NB = 4 * ((n + 63) >> 6);
            const int nq = n / NB, nr = n - nq * NB;  // bin bb holds nq + (bb < nr) real entries
            uint16_t* so = reinterpret_cast<uint16_t*>(rec_s[wi][own]);
            double* sv = reinterpret_cast<double*>(rec_s[wi][own] + 512);
            for (int t = lane; t < NB * 16; t += 32) {
                const int bb = t >> 4, m = t & 15;
                const int fill = nq + (bb < nr ? 1 : 0);
                if (m >= fill) {
                    const int sl = 64 * (bb >> 2) + 2 * (16 * ((bb >> 1) & 1) + m) + (bb & 1);
                    // the (m - fill)-th bank pair no real entry of the bin uses
                    const unsigned f = ~bmask_s[wi][own][bb] & 0xffffu;
#if ELL_BAL_ATOMIC_RANK
                    // the (m - fill)-th set bit of f by a 4-step popcount search (f has >= 16 - fill bits)
                    int nth = m - fill, r = 0;
                    unsigned x = f;
                    int pc = __popc(x & 0xffu);
                    if (nth >= pc) { nth -= pc; x >>= 8; r += 8; }
                    pc = __popc(x & 0xfu);
                    if (nth >= pc) { nth -= pc; x >>= 4; r += 4; }
                    pc = __popc(x & 0x3u);
                    if (nth >= pc) { nth -= pc; x >>= 2; r += 2; }
                    r += (nth >= (int)(x & 1u)) ? 1 : 0;
#else
                    const int r = (int)__fns(f, 0, m - fill + 1);
#endif
                    so[sl] = (uint16_t)(8 * (S + ((r - S) & 15)));
                    sv[sl] = 0.0;
                }
            }
            __syncwarp();
            // used groups (NB / 4) leave in coalesced 16-byte stores
            unsigned char* dst = bt + ((size_t)k * W + own) * rs;
            const int groups = NB >> 2;
            for (int t = lane; t < groups * 8; t += 32)  // 128 B of indices per group
                reinterpret_cast<int4*>(dst)[t] = reinterpret_cast<const int4*>(so)[t];
            for (int t = lane; t < groups * 32; t += 32)  // 512 B of values per group
                reinterpret_cast<int4*>(dst + 128 * G)[t] = reinterpret_cast<const int4*>(sv)[t];
        }
        __syncwarp();
    }
}

cudaError_t launch_balance_split(KMat b, int64_t k0, int64_t k1, int W, int G, int S, unsigned char* bt,
                                 int32_t* bt_nbin, int num_sms, cudaStream_t s) {
    if (k1 <= k0) return cudaSuccess;
    const int64_t blocks_needed = (k1 - k0 + 3) / 4;
    const int64_t cap = (int64_t)num_sms * 12;
    const unsigned grid = (unsigned)(blocks_needed < cap ? blocks_needed : cap);
    if (W == 2) balance_split_kernel<2, 8><<<grid, 128, 0, s>>>(b, k0, k1, G, S, bt, bt_nbin);
    else if (G == 1) balance_split_kernel<1, 2><<<grid, 128, 0, s>>>(b, k0, k1, G, S, bt, bt_nbin);
    else if (G == 2) balance_split_kernel<1, 4><<<grid, 128, 0, s>>>(b, k0, k1, G, S, bt, bt_nbin);
    else if (G == 3) balance_split_kernel<1, 6><<<grid, 128, 0, s>>>(b, k0, k1, G, S, bt, bt_nbin);
    else balance_split_kernel<1, 8><<<grid, 128, 0, s>>>(b, k0, k1, G, S, bt, bt_nbin);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------ the row kernel

template <int OFF>
__device__ __forceinline__ void ldg_keep_u32_if(bool pr, const void* p, uint64_t pol, uint32_t& v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t"
                 "@q ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%2+%4], %3;\n\t}"
                 : "+r"(v) : "r"((int)pr), "l"(p), "l"(pol), "n"(OFF));
}

__device__ __forceinline__ void bar_cta(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <int W>
struct SplitSmem {
    uint32_t acc, stg, xcnt, rowq, nrmx, flg;
};

// Kernel state of the row in flight (every warp holds the same values except the per-warp
// diagonal / norm partials).
struct SplitRow {
    int64_t i;
    int F;       // first unemitted column (multiple of 128)
    int sF;      // ring slot of F (F mod S)
    int kept;    // entries kept so far (all warps agree)
    int old_cur; // Old-row cursor (entries with column < F merged or skipped)
    int xbuf;    // exchange buffer parity: alternates every block, across rows too (consecutive
                 // blocks of consecutive rows have no other barrier between them)
    double ds, dc, nrm;
};

// Merge this warp's Old entries with columns < Fe into the ring (see ring_merge_old, spgemm.cu).
template <int W, int MODE>
__device__ __forceinline__ void split_merge_old(const RowOpParams& p, const SplitSmem<W>& sm, int lane, int wid,
                                                int Fe, int F, int sF, const int32_t* o_col, const double* o_val,
                                                int nOld, int& old_cur, double& nrm) {
    while (old_cur < nOld) {
        const int q = old_cur + lane;
        const bool v = q < nOld;
        const int jo = v ? o_col[q] : INT_MAX;
        const bool inr = jo < Fe;
        if (inr && ((jo >> 5) & (W - 1)) == wid) {
            const double x = o_val[q];
            const uint32_t off = (uint32_t)(sF + (jo - F));  // jo in [F, Fe): the block never wraps
            const uint32_t sa = sm.acc + 8u * off;
            const double sv = lds64(sa);
            if (MODE == 2) {
                const double df = __dsub_rn(sv, x);
                nrm = __fma_rn(df, df, nrm);
            }
            const double tt = (p.old_mode == 1) ? __dmul_rn(p.beta, x) : 0.0;
            sts64(sa, __fma_rn(p.alpha, sv, tt));
            sts8(sm.flg + off, 1u);
        }
        const int n = __popc(__ballot_sync(FULL, inr));
        old_cur += n;
        if (n < 32) break;
    }
    __syncwarp();
}

// Emit blocks [R.F, Fto) (multiples of 128): per block, this warp's NCH chunks are read and
// cleared, combined, dropped and ballot-compacted; the block's four chunk counts are exchanged
// (W > 1) and each warp writes its runs at their place in the row.
template <int W, int MODE, bool A1, int NBK>
__device__ __forceinline__ void split_emit(const RowOpParams& p, const SplitSmem<W>& sm, int lane, int wid,
                                           SplitRow& R, int Fto, const int32_t* o_col, const double* o_val,
                                           int nOld, double* __restrict__ crow_v, int32_t* __restrict__ crow_c) {
    constexpr int NCH = 4 / W;
    const int S = p.S;
    const double tau = p.tau;
    const unsigned lt = (1u << lane) - 1u;
    const int cw = p.C.w;
    const uint64_t bv = opaque_u64((uint64_t)crow_v), bc = opaque_u64((uint64_t)crow_c);
    if constexpr (W == 1 && ELL_SPLIT_LEAN_EMIT) {
        // One warp owns the whole block: the diagonal bookkeeping only in the block that holds
        // column i (warp-uniform branch), the keep decision straight from the compare, one
        // bounds compare per chunk (entries past the width are counted, not written).
        const bool want_dc = MODE != 0 || p.diag_c != nullptr;
        while (R.F < Fto) {
            const int F = R.F, sF = R.sF;
            if (MODE == 0 && NBK > 1 && Fto - F >= 128 * NBK && (uint64_t)(R.i - (int64_t)F) >= 128u * NBK) {
                // NBK blocks without the diagonal (the row's tail after its last k, runs of blocks):
                // all 4 NBK read-and-clears in flight before the first compare, one latency chain
                // instead of NBK (each block's stores would otherwise hold the next block's reads)
                uint32_t bb[NBK];
                int sFb = sF;
#pragma unroll
                for (int b = 0; b < NBK; ++b) {
                    bb[b] = sm.acc + 8u * (uint32_t)(sFb + lane);
                    sFb = sFb + 128 == S ? 0 : sFb + 128;
                }
                double x[4 * NBK];
                unsigned m[4 * NBK];
#pragma unroll
                for (int t = 0; t < 4 * NBK; ++t) x[t] = lds64_clear(bb[t >> 2] + 256u * (uint32_t)(t & 3));
#pragma unroll
                for (int t = 0; t < 4 * NBK; ++t) {
                    if (!A1) x[t] = __dmul_rn(p.alpha, x[t]);
                    m[t] = __ballot_sync(FULL, fabs(x[t]) > tau);
                }
                uint32_t before = (uint32_t)R.kept;
#pragma unroll
                for (int t = 0; t < 4 * NBK; ++t) {
                    const uint32_t pos = before + (uint32_t)__popc(m[t] & lt);
                    st_entry(((m[t] >> lane) & 1u) && pos < (uint32_t)cw, reinterpret_cast<double*>(bv + 8ull * pos),
                             reinterpret_cast<int32_t*>(bc + 4ull * pos), x[t], F + 32 * t + lane);
                    before += (uint32_t)__popc(m[t]);
                }
                R.kept = (int)before;
                R.F = F + 128 * NBK;
                R.sF = sFb;
                continue;
            }
            const uint32_t di = (uint32_t)(R.i - (int64_t)F);
            const bool dblk = di < 128u;
            if (dblk && lane == (int)(di & 31u)) R.ds = lds64(sm.acc + 8u * (uint32_t)(sF + (int)di));
            if (MODE != 0)
                split_merge_old<W, MODE>(p, sm, lane, wid, F + 128, F, sF, o_col, o_val, nOld, R.old_cur, R.nrm);
            double x[4];
            bool kp[4];
            unsigned m[4];
            const uint32_t a0 = sm.acc + 8u * (uint32_t)(sF + lane);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint32_t off = (uint32_t)(sF + 32 * t + lane);
                double v;
                if (ELL_SPLIT_CLEAR_STS) {
                    v = lds64(a0 + 256u * t);
                    sts64(a0 + 256u * t, 0.0);
                } else {
                    v = lds64_clear(a0 + 256u * t);
                }
                bool flagged = false;
                if (MODE != 0) {
                    flagged = lds8(sm.flg + off) != 0;
                    sts8(sm.flg + off, 0u);
                }
                x[t] = v;
                if (!flagged) {
                    if (!A1) x[t] = __dmul_rn(p.alpha, v);
                    if (MODE == 2) R.nrm = __fma_rn(v, v, R.nrm);
                }
                kp[t] = fabs(x[t]) > tau;
                m[t] = __ballot_sync(FULL, kp[t]);
            }
            uint32_t before = (uint32_t)R.kept;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint32_t pos = before + (uint32_t)__popc(m[t] & lt);
                st_entry(kp[t] && pos < (uint32_t)cw, reinterpret_cast<double*>(bv + 8ull * pos),
                         reinterpret_cast<int32_t*>(bc + 4ull * pos), x[t], F + 32 * t + lane);
                before += (uint32_t)__popc(m[t]);
            }
            if (dblk && want_dc) {
                const uint32_t tq = di >> 5;  // selects, not an indexed (local-memory) access
                const double xs = tq == 0 ? x[0] : tq == 1 ? x[1] : tq == 2 ? x[2] : x[3];
                const bool ks = tq == 0 ? kp[0] : tq == 1 ? kp[1] : tq == 2 ? kp[2] : kp[3];
                if (lane == (int)(di & 31u)) R.dc = ks ? xs : 0.0;
            }
            R.kept = (int)before;
            R.F = F + 128;
            R.sF = sF + 128 == S ? 0 : sF + 128;
        }
    } else {
    while (R.F < Fto) {
        const int F = R.F, sF = R.sF;
        // the pre-combine diagonal s_ii (tr X^2 pre-drop, R5): read before the Old merge
        if ((int64_t)F <= R.i && R.i < (int64_t)F + 128 && (((int)R.i >> 5) & (W - 1)) == wid &&
            lane == ((int)R.i & 31))
            R.ds = lds64(sm.acc + 8u * (uint32_t)(sF + (int)(R.i - F)));
        if (MODE != 0)
            split_merge_old<W, MODE>(p, sm, lane, wid, F + 128, F, sF, o_col, o_val, nOld, R.old_cur, R.nrm);
        double x[NCH];
        unsigned m[NCH];
#pragma unroll
        for (int t = 0; t < NCH; ++t) {
            const int q = wid + W * t;
            const uint32_t off = (uint32_t)(sF + 32 * q + lane);
            const double v = lds64_clear(sm.acc + 8u * off);
            bool flagged = false;
            if (MODE != 0) {
                flagged = lds8(sm.flg + off) != 0;
                sts8(sm.flg + off, 0u);
            }
            x[t] = v;
            if (!flagged) {
                if (!A1) x[t] = __dmul_rn(p.alpha, v);
                if (MODE == 2) R.nrm = __fma_rn(v, v, R.nrm);
            }
            m[t] = __ballot_sync(FULL, fabs(x[t]) > tau);
        }
        int cnt[4];
        if (W == 1) {
#pragma unroll
            for (int t = 0; t < 4; ++t) cnt[t] = __popc(m[t]);
        } else {
            const uint32_t xb = sm.xcnt + 16u * (uint32_t)R.xbuf;
            if (lane == 0) {
#pragma unroll
                for (int t = 0; t < NCH; ++t) sts32i(xb + 4u * (uint32_t)(wid + W * t), __popc(m[t]));
            }
            bar_cta(32 * W);
#pragma unroll
            for (int q = 0; q < 4; ++q) cnt[q] = lds32i(xb + 4u * q);
            R.xbuf ^= 1;
        }
        const bool room = R.kept + 128 <= cw;
#pragma unroll
        for (int t = 0; t < NCH; ++t) {
            const int q = wid + W * t;
            int before = R.kept;
#pragma unroll
            for (int u = 0; u < 4; ++u) before += u < q ? cnt[u] : 0;
            const bool keep = (m[t] >> lane) & 1u;
            const uint32_t pos = (uint32_t)before + (uint32_t)__popc(m[t] & lt);
            const int col = F + 32 * q + lane;
            st_entry(keep && (room || pos < (uint32_t)cw), reinterpret_cast<double*>(bv + 8ull * pos),
                     reinterpret_cast<int32_t*>(bc + 4ull * pos), x[t], col);
            if (MODE != 0 && (int64_t)col == R.i) R.dc = keep ? x[t] : 0.0;
            if (MODE == 0 && p.diag_c && (int64_t)col == R.i) R.dc = keep ? x[t] : 0.0;
        }
        R.kept += cnt[0] + cnt[1] + cnt[2] + cnt[3];
        R.F = F + 128;
        R.sF = sF + 128 == S ? 0 : sF + 128;
    }
    }
}

template <int W, int MODE, int NBK>
__device__ __forceinline__ void split_emit_to(const RowOpParams& p, const SplitSmem<W>& sm, int lane, int wid,
                                              SplitRow& R, int Fto, const int32_t* o_col, const double* o_val,
                                              int nOld, double* __restrict__ crow_v, int32_t* __restrict__ crow_c) {
    if (p.alpha == 1.0) split_emit<W, MODE, true, NBK>(p, sm, lane, wid, R, Fto, o_col, o_val, nOld, crow_v, crow_c);
    else split_emit<W, MODE, false, NBK>(p, sm, lane, wid, R, Fto, o_col, o_val, nOld, crow_v, crow_c);
}

// One output row, warp `wid` of W: the ring sweep of row_ring (spgemm.cu) over this warp's
// sub-records, register bursts of HB steps in a two-half register ring (a half touches its own
// burst, emits if the sweep would wrap onto unemitted columns, issues the next half's burst,
// then runs its steps branch-free).
// c0 / c1: the first / last column of A_i when the caller already has them (c1 < 0: not known).
// nxt_col / nxt_n: the next row of the caller's chunk (nxt_n <= 0: none): its first and last columns
// are loaded into nxt_c0 / nxt_c1 before this row's tail emission, which hides their latency.
// dA: the stored a_ii, read from the staged steps (p.diag_a set).
template <int W, int G, int HB, int MODE>
__device__ __forceinline__ void row_split(const RowOpParams& p, const SplitSmem<W>& sm, int lane, int wid,
                                          SplitRow& R, const int32_t* a_col, const double* a_val, int nA,
                                          const int32_t* o_col, const double* o_val, int nOld,
                                          double* __restrict__ crow_v, int32_t* __restrict__ crow_c, int c0, int c1,
                                          const int32_t* nxt_col, int nxt_n, int& nxt_c0, int& nxt_c1, double& dA) {
    constexpr int kPiece = split_stage(G) - 2 * HB + 1;  // real steps per piece
    // blocks emitted together in runs (no Old): G = 1 keeps one (the extra registers would cost it
    // rows per SM: 16 -> 12 measured)
    constexpr int kEmitBlocks = G >= 2 ? ELL_SPLIT_EMITN : 1;
    constexpr int RS = 640 * G;                        // sub-record bytes
    const int S = p.S;
    const int hB = p.hB;
    const int ncols = (int)p.ncols;
    int lo_col = INT_MAX, hi_col = -1;
    if (nA > 0) {
        if (c1 < 0) {
            c0 = __ldg(a_col);
            c1 = __ldg(a_col + nA - 1);
        }
        lo_col = max(0, c0 - hB);
        hi_col = min(ncols - 1, c1 + hB);
    }
    if (MODE != 0 && nOld > 0) {
        lo_col = min(lo_col, o_col[0]);
        hi_col = max(hi_col, o_col[nOld - 1]);
    }
    double da = 0.0;  // this lane's a_ii candidate (one lane at most holds it)
    bool has_da = false;
    if (hi_col < lo_col) {
        if (nxt_n > 0) {
            nxt_c0 = __ldg(nxt_col);
            nxt_c1 = __ldg(nxt_col + nxt_n - 1);
        }
        dA = 0.0;
        return;
    }
    R.F = lo_col & ~127;
    R.sF = R.F % S;
    const int Fend = (hi_col + 128) & ~127;
    const uint32_t acc = sm.acc;
    const uint32_t stg = sm.stg;
    const unsigned char* __restrict__ btl = p.bt + (size_t)wid * RS;  // this warp's sub-record of row 0
    const uint64_t pol = l2_evict_last_policy();

    uint32_t ro[2][HB][G];
    double2 rv[2][HB][G];
    // step metadata (a_ik, k, NB of this warp's sub-record): W = 1 keeps the next half's in
    // registers, read one half ahead (ELL_SPLIT_META); W = 2 re-reads it from the stage where used
    constexpr bool kMeta = ELL_SPLIT_META && W == 1;
    double am[2][HB];
    int km[2][HB], nbm[2][HB];
    auto get = [&](int t, double& a, int& k, int& nb) {
        unsigned long long x, y;
        asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(stg + 16u * t) : "memory");
        a = __longlong_as_double((long long)x);
        k = (int)(uint32_t)y;
        nb = (int)(y >> 32);
    };
    auto meta = [&](auto Xc, int h) {
        constexpr int X = decltype(Xc)::value;
#pragma unroll
        for (int e = 0; e < HB; ++e) get(h * HB + e, am[X][e], km[X][e], nbm[X][e]);
    };
    auto burst = [&](auto Xc, int h) {
        constexpr int X = decltype(Xc)::value;
#pragma unroll
        for (int e = 0; e < HB; ++e) {
            double a_u;
            int k_u, nb;
            if (kMeta) { k_u = km[X][e]; nb = nbm[X][e]; }
            else get(h * HB + e, a_u, k_u, nb);
            const unsigned char* __restrict__ rp = btl + (size_t)(uint32_t)k_u * (W * RS);
            const unsigned char* __restrict__ sp = rp + 4 * lane;
            const unsigned char* __restrict__ vp = rp + 16 * lane;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                if (g == 0) { ldg_keep_u32_if<0>(nb > 0, sp, pol, ro[X][e][0]); ldg_keep_d2_if<128 * G>(nb > 0, vp, pol, rv[X][e][0]); }
                if (g == 1) { ldg_keep_u32_if<128>(nb > 4, sp, pol, ro[X][e][1]); ldg_keep_d2_if<128 * G + 512>(nb > 4, vp, pol, rv[X][e][1]); }
                if (g == 2) { ldg_keep_u32_if<256>(nb > 8, sp, pol, ro[X][e][2]); ldg_keep_d2_if<128 * G + 1024>(nb > 8, vp, pol, rv[X][e][2]); }
                if (g == 3) { ldg_keep_u32_if<384>(nb > 12, sp, pol, ro[X][e][3]); ldg_keep_d2_if<128 * G + 1536>(nb > 12, vp, pol, rv[X][e][3]); }
            }
        }
    };
    auto step = [&](int X, int e, double a, int nb) {
        double old[G][2];
        bool gl[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            gl[g] = nb > 4 * g;
            old[g][0] = lds64_if(gl[g], acc + (ro[X][e][g] & 0xffffu));
            old[g][1] = lds64_if(gl[g], acc + (ro[X][e][g] >> 16));
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            sts64_if(gl[g], acc + (ro[X][e][g] & 0xffffu), __fma_rn(a, rv[X][e][g].x, old[g][0]));
            sts64_if(gl[g], acc + (ro[X][e][g] >> 16), __fma_rn(a, rv[X][e][g].y, old[g][1]));
        }
        __syncwarp();
    };
    auto half = [&](auto Xc, int h) {
        constexpr int X = decltype(Xc)::value;
        double a_[HB];
        int k_[HB], nb_[HB];
        if (kMeta) {
#pragma unroll
            for (int e = 0; e < HB; ++e) { a_[e] = am[X][e]; k_[e] = km[X][e]; nb_[e] = nbm[X][e]; }
            meta(std::integral_constant<int, X ^ 1>{}, h + 1);
        } else {
#pragma unroll
            for (int e = 0; e < HB; ++e) get(h * HB + e, a_[e], k_[e], nb_[e]);
        }
        if (nb_[0] > 0) sts32i(acc + 8u * (uint32_t)S, (int)ro[X][0][0]);  // touch: waits for this burst
        const int kf = k_[0], kl = k_[HB - 1];
        if (kf + hB >= R.F + S) split_emit_to<W, MODE, kEmitBlocks>(p, sm, lane, wid, R, (kf - hB) & ~127, o_col, o_val, nOld,
                                                       crow_v, crow_c);
        __syncwarp();
        burst(std::integral_constant<int, X ^ 1>{}, h + 1);
        if (kl + hB < R.F + S) {
#pragma unroll
            for (int e = 0; e < HB; ++e) step(X, e, a_[e], nb_[e]);
        } else {
#pragma unroll
            for (int e = 0; e < HB; ++e) {
                const int kt = k_[e];
                if (kt + hB >= R.F + S)
                    split_emit_to<W, MODE, kEmitBlocks>(p, sm, lane, wid, R, (kt - hB) & ~127, o_col, o_val, nOld, crow_v, crow_c);
                step(X, e, a_[e], nb_[e]);
            }
        }
    };
    for (int p0 = 0; p0 < nA; p0 += kPiece) {
        const int cnt = min(kPiece, nA - p0);
        const int nh = (cnt + HB - 1) / HB;
        // stage the piece (a_ik, k, NB(k)), null steps after it: every global load of the piece is
        // issued before the first shared store (an asm store with a memory clobber would otherwise
        // hold each lane's next loads behind it: ~5 dependent round trips per row)
        constexpr int NI = (split_stage(G) + 31) / 32;
        const int lim = (nh + 1) * HB;
        const int kfill = __ldg(a_col + p0 + cnt - 1);
        int kq[NI], nbq[NI];
        double aq[NI];
#pragma unroll
        for (int u = 0; u < NI; ++u) {
            const int q = lane + 32 * u;
            kq[u] = q < cnt ? __ldg(a_col + p0 + q) : kfill;
            aq[u] = q < cnt ? __ldg(a_val + p0 + q) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < NI; ++u) nbq[u] = lane + 32 * u < cnt ? __ldg(p.bt_nbin + (size_t)kq[u] * W + wid) : 0;
        if (p.diag_a) {
#pragma unroll
            for (int u = 0; u < NI; ++u)
                if (lane + 32 * u < cnt && kq[u] == (int)R.i) { da = aq[u]; has_da = true; }
        }
#pragma unroll
        for (int u = 0; u < NI; ++u) {
            const int q = lane + 32 * u;
            if (q < lim) {
                const unsigned long long knb =
                    (unsigned long long)(uint32_t)kq[u] | ((unsigned long long)(uint32_t)nbq[u] << 32);
                asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(stg + 16u * q), "l"(__double_as_longlong(aq[u])),
                             "l"(knb) : "memory");
            }
        }
        __syncwarp();
        if (kMeta) meta(std::integral_constant<int, 0>{}, 0);
        burst(std::integral_constant<int, 0>{}, 0);
        for (int h = 0; h < nh; h += 2) {
            half(std::integral_constant<int, 0>{}, h);
            if (h + 1 < nh) half(std::integral_constant<int, 1>{}, h + 1);
        }
    }
    if (nxt_n > 0) {  // in flight during the tail emission
        nxt_c0 = __ldg(nxt_col);
        nxt_c1 = __ldg(nxt_col + nxt_n - 1);
    }
    split_emit_to<W, MODE, kEmitBlocks>(p, sm, lane, wid, R, Fend, o_col, o_val, nOld, crow_v, crow_c);
    const unsigned mm = __ballot_sync(FULL, has_da);
    dA = mm ? __shfl_sync(FULL, da, __ffs(mm) - 1) : 0.0;
}

template <int W, int G, int HB, int MODE>
__global__ void __launch_bounds__(32 * W, W == 1 && G == 1 ? ELL_SPLIT_MINB_G1 : (W == 1 && G == 2 ? ELL_SPLIT_MINB_G2 : 6))
    row_split_kernel(const RowOpParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int S = p.S;
    SplitSmem<W> sm;
    sm.acc = (uint32_t)__cvta_generic_to_shared(smem_raw);
    sm.stg = sm.acc + (uint32_t)((S + kSplitTrash) * 8) + (uint32_t)(wid * split_stage(G) * 16);
    sm.xcnt = sm.acc + (uint32_t)((S + kSplitTrash) * 8 + W * split_stage(G) * 16);
    sm.rowq = sm.xcnt + 32u;
    sm.nrmx = sm.rowq + 16u;
    sm.flg = sm.nrmx + 8u * W;
    for (int jj = 2 * (int)threadIdx.x; jj < S + kSplitTrash; jj += 64 * W) sts128(sm.acc + 8u * jj, 0.0, 0.0);
    if (MODE != 0)
        for (int jj = 4 * (int)threadIdx.x; jj < S; jj += 128 * W) sts32i(sm.flg + jj, 0);
    __syncthreads();
    int32_t my_max_kept = 0, my_ovf = 0;
    int xbuf = 0;
    const int chunk = p.row_chunk;
    for (int it = 0;; ++it) {
        const uint32_t rq = sm.rowq + 8u * (uint32_t)(it & 1);  // double-buffered row ticket
        if (threadIdx.x == 0) {
            const unsigned long long t = atomicAdd(p.row_ticket, 1ull);
            asm volatile("st.shared.s64 [%0], %1;" ::"r"(rq), "l"((long long)(p.row_begin + chunk * (int64_t)t))
                         : "memory");
        }
        __syncthreads();
        long long i0;
        asm volatile("ld.shared.s64 %0, [%1];" : "=l"(i0) : "r"(rq) : "memory");
        if (i0 >= p.row_end) break;
        // rows of the chunk: the next row's count is loaded one row ahead, its first and last
        // columns during this row's tail emission (row_split)
        const int64_t iend = min((int64_t)i0 + chunk, p.row_end);
        int nA_n = p.alpha != 0.0 ? __ldg(p.A.nnz + i0) : 0;
        int c0_n = 0, c1_n = -1;
        for (int64_t i = i0; i < iend; ++i) {
            const double* a_val = p.A.val + (size_t)i * p.A.w;
            const int32_t* a_col = p.A.col + (size_t)i * p.A.w;
            const int nA = nA_n;
            const int c0 = c0_n, c1 = c1_n;
            nA_n = (p.alpha != 0.0 && i + 1 < iend) ? __ldg(p.A.nnz + i + 1) : 0;
            c1_n = -1;
            const double* o_val = nullptr;
            const int32_t* o_col = nullptr;
            int nOld = 0;
            if (MODE != 0) {
                o_val = p.Old.val + (size_t)i * p.Old.w;
                o_col = p.Old.col + (size_t)i * p.Old.w;
                nOld = p.Old.nnz[i];
            }
            double* crow_v = p.C.val + (size_t)i * p.C.w;
            int32_t* crow_c = p.C.col + (size_t)i * p.C.w;
            SplitRow R;
            R.i = i;
            R.kept = 0;
            R.old_cur = 0;
            R.xbuf = xbuf;
            R.ds = R.dc = R.nrm = 0.0;
            double dA = 0.0;
            row_split<W, G, HB, MODE>(p, sm, lane, wid, R, a_col, a_val, nA, o_col, o_val, nOld, crow_v, crow_c, c0, c1,
                                      p.A.col + (size_t)(i + 1) * p.A.w, nA_n, c0_n, c1_n, dA);
            xbuf = R.xbuf;
            // epilogue: the diagonal values live in the owning warp's lane (x + 0 = x exactly)
            const double ds = warp_sum(R.ds), dc = warp_sum(R.dc);
            const bool owner = (((int)i >> 5) & (W - 1)) == wid;
            if (owner && lane == 0) {
                if (p.diag_c) p.diag_c[i] = dc;
                if (p.diag_s) p.diag_s[i] = ds;
            }
            if (MODE == 2 && p.normsq) {
                const double nr = warp_sum(R.nrm);
                if (W == 1) {
                    if (lane == 0) p.normsq[i] = nr;
                } else {
                    if (lane == 0) sts64(sm.nrmx + 8u * wid, nr);
                    bar_cta(32 * W);
                    if (wid == 0 && lane == 0) {
                        double t = 0.0;
#pragma unroll
                        for (int q = 0; q < W; ++q) t = __dadd_rn(t, lds64(sm.nrmx + 8u * q));
                        p.normsq[i] = t;
                    }
                    bar_cta(32 * W);
                }
            }
            if (wid == 0) {
                if (lane == 0) {
                    p.C.nnz[i] = R.kept < p.C.w ? R.kept : p.C.w;
                    if (p.diag_a) p.diag_a[i] = dA;
                }
                my_max_kept = max(my_max_kept, R.kept);
                if (R.kept > p.C.w) ++my_ovf;
            }
        }
    }
    if (wid == 0 && lane == 0) {
        if (my_ovf) atomicAdd(p.status + 0, my_ovf);
        if (my_max_kept) atomicMax(p.status + 1, my_max_kept);
    }
}

// ------------------------------------------------------- warp-specialized ring kernel (WS)
//
// One CTA per output row in flight, two warps: the ACCUMULATOR warp walks A_i and applies every
// B row to the ring (one warp per row: the full 123-entry records keep the bank balance of the
// one-warp kernel), the EMITTER warp turns finished 128-column blocks into output (combine with
// Old, drop, compact, write) and clears them. Emission -- half of the one-warp kernel's
// instructions -- then overlaps accumulation instead of interrupting it.
//
// The ring's NB = S / 128 regions (block b of the row lives in region b mod NB) are handed over
// with mbarriers: the accumulator arrives on full[r] when block b is final (every later k has
// k - hB >= 128 (b + 1)), the emitter arrives on empty[r] after emitting it. Before touching
// block b the accumulator waits until the block that last used region r was emitted. Blocks are
// acquired, released and emitted in ascending order (across rows too), so with the live window
// of a step (33 blocks for hB = 2048) below NB every wait is on a block already released: no
// deadlock. Row headers (row, first block, end block) travel through a 4-entry queue with its own
// full/empty mbarriers; a header with row -1 ends the emitter.
#ifndef ELL_WS_HB_G3
#define ELL_WS_HB_G3 1
#endif
constexpr int kWsStage = 64;
constexpr int kWsHQ = 4;

__host__ __device__ inline size_t ws_smem_bytes(int S, bool has_old) {
    // acc[S + 16] f64 | stage[kWsStage] 16 B | full[NB], empty[NB] u64 | hq[4] 16 B | hfull[4], hempty[4] u64
    // | flags[S] u8
    const int NB = S / 128;
    return (size_t)(S + kSplitTrash) * 8 + (size_t)kWsStage * 16 + (size_t)NB * 16 + kWsHQ * 16 + kWsHQ * 16 +
           (has_old ? (size_t)S : 0);
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(a), "r"(parity) : "memory");
}

struct WsSmem {
    uint32_t acc, stg, full, empty, hq, hfull, hempty, flg;
    int NB;
};

// Emitter: one block [F, F + 128) of row i (ring slots sF ..), Old merged first.
template <int MODE, bool A1>
__device__ __forceinline__ void ws_emit_block(const RowOpParams& p, const WsSmem& sm, int lane, int64_t i, int F,
                                              int sF, const int32_t* o_col, const double* o_val, int nOld,
                                              int& old_cur, double* __restrict__ crow_v, int32_t* __restrict__ crow_c,
                                              int& kept, double& ds, double& dc, double& nrm) {
    const double tau = p.tau;
    const unsigned lt = (1u << lane) - 1u;
    const int cw = p.C.w;
    if ((int64_t)F <= i && i < (int64_t)F + 128 && lane == ((int)i & 31))
        ds = lds64(sm.acc + 8u * (uint32_t)(sF + (int)(i - F)));
    if (MODE != 0) {
        SplitSmem<1> s1;
        s1.acc = sm.acc;
        s1.flg = sm.flg;
        split_merge_old<1, MODE>(p, s1, lane, 0, F + 128, F, sF, o_col, o_val, nOld, old_cur, nrm);
    }
    double x[4];
    unsigned m[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t off = (uint32_t)(sF + 32 * q + lane);
        const double v = lds64_clear(sm.acc + 8u * off);
        bool flagged = false;
        if (MODE != 0) {
            flagged = lds8(sm.flg + off) != 0;
            sts8(sm.flg + off, 0u);
        }
        x[q] = v;
        if (!flagged) {
            if (!A1) x[q] = __dmul_rn(p.alpha, v);
            if (MODE == 2) nrm = __fma_rn(v, v, nrm);
        }
        m[q] = __ballot_sync(FULL, fabs(x[q]) > tau);
    }
    const bool room = kept + 128 <= cw;
    const uint64_t bv = opaque_u64((uint64_t)crow_v), bc = opaque_u64((uint64_t)crow_c);
    int before = kept;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const bool keep = (m[q] >> lane) & 1u;
        const uint32_t pos = (uint32_t)before + (uint32_t)__popc(m[q] & lt);
        const int col = F + 32 * q + lane;
        st_entry(keep && (room || pos < (uint32_t)cw), reinterpret_cast<double*>(bv + 8ull * pos),
                 reinterpret_cast<int32_t*>(bc + 4ull * pos), x[q], col);
        if ((int64_t)col == i) dc = keep ? x[q] : 0.0;
        before += __popc(m[q]);
    }
    kept = before;
}

template <int MODE>
__device__ __forceinline__ void ws_emitter(const RowOpParams& p, const WsSmem& sm, int lane) {
    const int S = p.S;
    uint64_t e_par = 0;  // per region: parity of the next full-phase to wait for
    int32_t my_max_kept = 0, my_ovf = 0;
    for (int q = 0;; ++q) {
        const int h = q % kWsHQ;
        mbar_wait(sm.hfull + 8u * h, (uint32_t)((q / kWsHQ) & 1));
        long long i;
        int F0, Fend;
        asm volatile("ld.shared.s64 %0, [%1];" : "=l"(i) : "r"(sm.hq + 16u * h) : "memory");
        F0 = lds32i(sm.hq + 16u * h + 8u);
        Fend = lds32i(sm.hq + 16u * h + 12u);
        __syncwarp();
        if (lane == 0) mbar_arrive(sm.hempty + 8u * h);
        if (i < 0) break;
        const double* o_val = nullptr;
        const int32_t* o_col = nullptr;
        int nOld = 0;
        if (MODE != 0) {
            o_val = p.Old.val + (size_t)i * p.Old.w;
            o_col = p.Old.col + (size_t)i * p.Old.w;
            nOld = p.Old.nnz[i];
        }
        double* crow_v = p.C.val + (size_t)i * p.C.w;
        int32_t* crow_c = p.C.col + (size_t)i * p.C.w;
        int kept = 0, old_cur = 0;
        double ds = 0.0, dc = 0.0, nrm = 0.0;
        for (int F = F0; F < Fend; F += 128) {
            const int b = F >> 7;
            const int r = b % sm.NB;
            mbar_wait(sm.full + 8u * r, (uint32_t)((e_par >> r) & 1u));
            e_par ^= 1ull << r;
            const int sF = r * 128;  // F mod S (S = 128 NB)
            if (p.alpha == 1.0)
                ws_emit_block<MODE, true>(p, sm, lane, i, F, sF, o_col, o_val, nOld, old_cur, crow_v, crow_c, kept,
                                          ds, dc, nrm);
            else
                ws_emit_block<MODE, false>(p, sm, lane, i, F, sF, o_col, o_val, nOld, old_cur, crow_v, crow_c, kept,
                                           ds, dc, nrm);
            __syncwarp();
            if (lane == 0) mbar_arrive(sm.empty + 8u * r);
        }
        (void)S;
        ds = warp_sum(ds);
        dc = warp_sum(dc);
        if (MODE == 2 && p.normsq) nrm = warp_sum(nrm);
        if (lane == 0) {
            p.C.nnz[i] = kept < p.C.w ? kept : p.C.w;
            if (p.diag_c) p.diag_c[i] = dc;
            if (p.diag_s) p.diag_s[i] = ds;
            if (MODE == 2 && p.normsq) p.normsq[i] = nrm;
        }
        if (p.diag_a) {
            const double* a_val = p.A.val + (size_t)i * p.A.w;
            const int32_t* a_col = p.A.col + (size_t)i * p.A.w;
            const int nA = (p.alpha != 0.0) ? p.A.nnz[i] : 0;
            double dA = 0.0;
            bool has = false;
            for (int t = lane; t < nA; t += 32)
                if (a_col[t] == (int)i) { dA = a_val[t]; has = true; }
            const unsigned mm = __ballot_sync(FULL, has);
            dA = mm ? __shfl_sync(FULL, dA, __ffs(mm) - 1) : 0.0;
            if (lane == 0) p.diag_a[i] = dA;
        }
        my_max_kept = max(my_max_kept, kept);
        if (kept > p.C.w) ++my_ovf;
    }
    if (lane == 0) {
        if (my_ovf) atomicAdd(p.status + 0, my_ovf);
        if (my_max_kept) atomicMax(p.status + 1, my_max_kept);
    }
}

// Accumulator: the ring sweep of row_split (W = 1) without emission; blocks are acquired before
// the steps that may touch them and released once final.
template <int G, int HB>
struct WsAcc {
    const RowOpParams& p;
    const WsSmem& sm;
    int lane;
    uint64_t used = 0, par = 0;  // per region: used before, parity of the next empty-phase to wait for
    int acq = -1;                // highest acquired block
    int rel = 0;                 // next block to release
    int endb = 0;                // one past the row's last block
    __device__ WsAcc(const RowOpParams& p_, const WsSmem& sm_, int lane_) : p(p_), sm(sm_), lane(lane_) {}
    __device__ __forceinline__ void acquire_to(int b) {
        if (b >= endb) b = endb - 1;
        while (acq < b) {
            ++acq;
            const int r = acq % sm.NB;
            if ((used >> r) & 1ull) {
                mbar_wait(sm.empty + 8u * r, (uint32_t)((par >> r) & 1ull));
                par ^= 1ull << r;
            } else {
                used |= 1ull << r;
            }
        }
    }
    __device__ __forceinline__ void release_below(int b) {  // every block < b is final
        if (b > endb) b = endb;
        if (rel >= b) return;
        acquire_to(b - 1);  // (blocks no product touched are still handed over: zeroed, owned)
        __syncwarp();
        if (lane == 0)
            for (int q = rel; q < b; ++q) mbar_arrive(sm.full + 8u * (uint32_t)(q % sm.NB));
        rel = b;
    }
};

template <int G, int HB>
__device__ __forceinline__ void ws_accumulate_row(const RowOpParams& p, WsAcc<G, HB>& A, int lane,
                                                  const int32_t* a_col, const double* a_val, int nA, int F0) {
    constexpr int kPiece = kWsStage - 2 * HB + 1;
    constexpr int RS = 640 * G;
    const int hB = p.hB;
    const WsSmem& sm = A.sm;
    const uint32_t acc = sm.acc, stg = sm.stg;
    const unsigned char* __restrict__ btl = p.bt;
    const uint64_t pol = l2_evict_last_policy();
    const int NB = sm.NB;
    uint32_t ro[2][HB][G];
    double2 rv[2][HB][G];
    auto get = [&](int t, double& a, int& k, int& nb) {
        unsigned long long x, y;
        asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(stg + 16u * t) : "memory");
        a = __longlong_as_double((long long)x);
        k = (int)(uint32_t)y;
        nb = (int)(y >> 32);
    };
    auto burst = [&](auto Xc, int h) {
        constexpr int X = decltype(Xc)::value;
#pragma unroll
        for (int e = 0; e < HB; ++e) {
            double a_u;
            int k_u, nb;
            get(h * HB + e, a_u, k_u, nb);
            const unsigned char* __restrict__ rp = btl + (size_t)(uint32_t)k_u * RS;
            const unsigned char* __restrict__ sp = rp + 4 * lane;
            const unsigned char* __restrict__ vp = rp + 16 * lane;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                if (g == 0) { ldg_keep_u32_if<0>(nb > 0, sp, pol, ro[X][e][0]); ldg_keep_d2_if<128 * G>(nb > 0, vp, pol, rv[X][e][0]); }
                if (g == 1) { ldg_keep_u32_if<128>(nb > 4, sp, pol, ro[X][e][1]); ldg_keep_d2_if<128 * G + 512>(nb > 4, vp, pol, rv[X][e][1]); }
                if (g == 2) { ldg_keep_u32_if<256>(nb > 8, sp, pol, ro[X][e][2]); ldg_keep_d2_if<128 * G + 1024>(nb > 8, vp, pol, rv[X][e][2]); }
                if (g == 3) { ldg_keep_u32_if<384>(nb > 12, sp, pol, ro[X][e][3]); ldg_keep_d2_if<128 * G + 1536>(nb > 12, vp, pol, rv[X][e][3]); }
            }
        }
    };
    auto step = [&](int X, int e, double a, int nb) {
        double old[G][2];
        bool gl[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            gl[g] = nb > 4 * g;
            old[g][0] = lds64_if(gl[g], acc + (ro[X][e][g] & 0xffffu));
            old[g][1] = lds64_if(gl[g], acc + (ro[X][e][g] >> 16));
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            sts64_if(gl[g], acc + (ro[X][e][g] & 0xffffu), __fma_rn(a, rv[X][e][g].x, old[g][0]));
            sts64_if(gl[g], acc + (ro[X][e][g] >> 16), __fma_rn(a, rv[X][e][g].y, old[g][1]));
        }
        __syncwarp();
    };
    // floor((k - hB) / 128) for k - hB possibly negative: blocks below it are final before step k
    auto fin = [&](int k) { return (k - hB) >= 0 ? ((k - hB) >> 7) : -1; };
    auto half = [&](auto Xc, int h) {
        constexpr int X = decltype(Xc)::value;
        double a_[HB];
        int k_[HB], nb_[HB];
#pragma unroll
        for (int e = 0; e < HB; ++e) get(h * HB + e, a_[e], k_[e], nb_[e]);
        if (nb_[0] > 0) sts32i(acc + 8u * (uint32_t)p.S, (int)ro[X][0][0]);  // touch: waits for this burst
        const int kf = k_[0], kl = k_[HB - 1];
        A.release_below(fin(kf));
        const int top = (kl + hB) >> 7;
        __syncwarp();
        burst(std::integral_constant<int, X ^ 1>{}, h + 1);
        if (top < A.rel + NB) {
            A.acquire_to(top);
#pragma unroll
            for (int e = 0; e < HB; ++e) step(X, e, a_[e], nb_[e]);
        } else {
#pragma unroll
            for (int e = 0; e < HB; ++e) {
                A.release_below(fin(k_[e]));
                A.acquire_to((k_[e] + hB) >> 7);
                step(X, e, a_[e], nb_[e]);
            }
        }
    };
    for (int p0 = 0; p0 < nA; p0 += kPiece) {
        const int cnt = min(kPiece, nA - p0);
        const int nh = (cnt + HB - 1) / HB;
        for (int q = lane; q < (nh + 1) * HB; q += 32) {
            int k, nb;
            double a;
            if (q < cnt) {
                k = a_col[p0 + q];
                nb = __ldg(p.bt_nbin + k);
                a = a_val[p0 + q];
            } else {
                k = a_col[p0 + cnt - 1];
                nb = 0;
                a = 0.0;
            }
            const unsigned long long knb = (unsigned long long)(uint32_t)k | ((unsigned long long)(uint32_t)nb << 32);
            asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(stg + 16u * q), "l"(__double_as_longlong(a)),
                         "l"(knb) : "memory");
        }
        __syncwarp();
        burst(std::integral_constant<int, 0>{}, 0);
        for (int h = 0; h < nh; h += 2) {
            half(std::integral_constant<int, 0>{}, h);
            if (h + 1 < nh) half(std::integral_constant<int, 1>{}, h + 1);
        }
    }
    (void)F0;
}

// next ticket of row_chunk rows (lane 0 takes it, the warp gets it)
__device__ __forceinline__ int64_t ws_next_row(const RowOpParams& p, int lane) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(p.row_ticket, 1ull);
    return (int64_t)__shfl_sync(FULL, t, 0);
}

template <int G, int HB, int MODE>
__global__ void __launch_bounds__(64, 6) row_ws_kernel(const RowOpParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int S = p.S;
    WsSmem sm;
    sm.NB = S / 128;
    sm.acc = (uint32_t)__cvta_generic_to_shared(smem_raw);
    sm.stg = sm.acc + (uint32_t)((S + kSplitTrash) * 8);
    sm.full = sm.stg + (uint32_t)(kWsStage * 16);
    sm.empty = sm.full + 8u * (uint32_t)sm.NB;
    sm.hq = sm.empty + 8u * (uint32_t)sm.NB;
    sm.hfull = sm.hq + 16u * kWsHQ;
    sm.hempty = sm.hfull + 8u * kWsHQ;
    sm.flg = sm.hempty + 8u * kWsHQ;
    for (int jj = 2 * (int)threadIdx.x; jj < S + kSplitTrash; jj += 128) sts128(sm.acc + 8u * jj, 0.0, 0.0);
    if (MODE != 0)
        for (int jj = 4 * (int)threadIdx.x; jj < S; jj += 256) sts32i(sm.flg + jj, 0);
    if (threadIdx.x == 0) {
        for (int r = 0; r < sm.NB; ++r) {
            mbar_init(sm.full + 8u * r, 1);
            mbar_init(sm.empty + 8u * r, 1);
        }
        for (int h = 0; h < kWsHQ; ++h) {
            mbar_init(sm.hfull + 8u * h, 1);
            mbar_init(sm.hempty + 8u * h, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (wid == 1) {
        ws_emitter<MODE>(p, sm, lane);
        return;
    }
    // accumulator warp
    WsAcc<G, HB> A(p, sm, lane);
    const int hB = p.hB;
    const int ncols = (int)p.ncols;
    const int chunk = p.row_chunk;
    int q = 0;  // headers sent
    auto send = [&](long long i, int F0, int Fend) {
        const int h = q % kWsHQ;
        if (q >= kWsHQ) mbar_wait(sm.hempty + 8u * h, (uint32_t)(((q / kWsHQ) - 1) & 1));
        if (lane == 0) {
            asm volatile("st.shared.s64 [%0], %1;" ::"r"(sm.hq + 16u * h), "l"(i) : "memory");
            sts32i(sm.hq + 16u * h + 8u, F0);
            sts32i(sm.hq + 16u * h + 12u, Fend);
            mbar_arrive(sm.hfull + 8u * h);
        }
        __syncwarp();
        ++q;
    };
    for (int64_t i0 = p.row_begin + chunk * ws_next_row(p, lane); i0 < p.row_end;
         i0 = p.row_begin + chunk * ws_next_row(p, lane)) {
        for (int64_t i = i0; i < i0 + chunk && i < p.row_end; ++i) {
            const double* a_val = p.A.val + (size_t)i * p.A.w;
            const int32_t* a_col = p.A.col + (size_t)i * p.A.w;
            const int nA = (p.alpha != 0.0) ? p.A.nnz[i] : 0;
            int lo_col = INT_MAX, hi_col = -1;
            if (nA > 0) {
                lo_col = max(0, a_col[0] - hB);
                hi_col = min(ncols - 1, a_col[nA - 1] + hB);
            }
            if (MODE != 0) {
                const int nOld = p.Old.nnz[i];
                if (nOld > 0) {
                    const int32_t* o_col = p.Old.col + (size_t)i * p.Old.w;
                    lo_col = min(lo_col, o_col[0]);
                    hi_col = max(hi_col, o_col[nOld - 1]);
                }
            }
            if (hi_col < lo_col) {
                send(i, 0, 0);
                continue;
            }
            const int F0 = lo_col & ~127, Fend = (hi_col + 128) & ~127;
            send(i, F0, Fend);
            A.acq = (F0 >> 7) - 1;
            A.rel = F0 >> 7;
            A.endb = Fend >> 7;
            ws_accumulate_row<G, HB>(p, A, lane, a_col, a_val, nA, F0);
            A.release_below(A.endb);
        }
    }
    send(-1, 0, 0);
}

template <int MODE, typename Fn>
static void ws_dispatch(int G, Fn f) {
    switch (G) {
        case 1: f(row_ws_kernel<1, 3, MODE>); break;
        case 2: f(row_ws_kernel<2, 2, MODE>); break;
        case 3: f(row_ws_kernel<3, ELL_WS_HB_G3, MODE>); break;
        default: f(row_ws_kernel<4, 1, MODE>); break;
    }
}

// -------------------------------------------------------------------------- dispatch

template <typename K>
static cudaError_t split_prep(K kern, int threads, size_t smem, int* bps) {
    return occupancy_cached((const void*)kern, threads, smem, bps);
}

template <int W, int MODE, typename Fn>
static void split_dispatch(int G, Fn f) {
    // steps per register half: deep bursts for one warp per row (255 registers); W = 2 runs 6
    // two-warp CTAs per SM, 168 registers per thread
    switch (G) {
        case 1: f(row_split_kernel<W, 1, W == 1 ? ELL_SPLIT_HB_G1 : 3, MODE>); break;
        case 2: f(row_split_kernel<W, 2, W == 1 ? ELL_SPLIT_HB_G2 : 2, MODE>); break;
        case 3: f(row_split_kernel<W, 3, W == 1 ? ELL_SPLIT_HB_G3 : 1, MODE>); break;
        default: f(row_split_kernel<W, 4, W == 1 ? 2 : 1, MODE>); break;
    }
}

template <int W, int MODE>
static cudaError_t split_prep_wm(int G, size_t smem, int* bps) {
    cudaError_t e = cudaSuccess;
    split_dispatch<W, MODE>(G, [&](auto k) { e = split_prep(k, 32 * W, smem, bps); });
    return e;
}

template <int W, int MODE>
static void split_launch_wm(int G, const RowOpParams& p, int grid, size_t smem, cudaStream_t s) {
    split_dispatch<W, MODE>(G, [&](auto k) { k<<<grid, 32 * W, smem, s>>>(p); });
}

static int split_mode_of(const RowOpParams& p) { return p.old_mode == 0 ? 0 : (p.normsq ? 2 : 1); }

size_t split_row_smem(int S, int W, bool has_old, int G) { return split_smem_bytes(S, W, has_old, G); }

cudaError_t plan_split(const RowOpParams& p, int S, int W, int G, int num_sms, LaunchCfg* cfg) {
    if (S % 128 || W < 1 || W > 2 || G < 1 || G > 4) return cudaErrorInvalidValue;
    const size_t smem = split_smem_bytes(S, W, p.old_mode != 0, G);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    int bps = 0;
    const int mode = split_mode_of(p);
    cudaError_t e;
    if (W == 2) e = mode == 0 ? split_prep_wm<2, 0>(G, smem, &bps) : mode == 1 ? split_prep_wm<2, 1>(G, smem, &bps)
                                                                          : split_prep_wm<2, 2>(G, smem, &bps);
    else e = mode == 0 ? split_prep_wm<1, 0>(G, smem, &bps) : mode == 1 ? split_prep_wm<1, 1>(G, smem, &bps)
                                                                      : split_prep_wm<1, 2>(G, smem, &bps);
    if (e) return e;
    if (bps < 1) return cudaErrorInvalidConfiguration;
    cfg->S = S;
    cfg->R = G;
    cfg->warps_per_cta = W;
    cfg->smem = smem;
    cfg->bps = bps;
    const int64_t rows = p.row_end - p.row_begin;
    const int64_t full = (int64_t)bps * num_sms;
    cfg->grid = (int)(rows < full ? (rows > 0 ? rows : 1) : full);
    return cudaSuccess;
}

cudaError_t launch_split(const RowOpParams& p, const LaunchCfg& cfg, cudaStream_t s) {
    const int mode = split_mode_of(p);
    const int G = cfg.R;
    if (cfg.warps_per_cta == 2) {
        if (mode == 0) split_launch_wm<2, 0>(G, p, cfg.grid, cfg.smem, s);
        else if (mode == 1) split_launch_wm<2, 1>(G, p, cfg.grid, cfg.smem, s);
        else split_launch_wm<2, 2>(G, p, cfg.grid, cfg.smem, s);
    } else {
        if (mode == 0) split_launch_wm<1, 0>(G, p, cfg.grid, cfg.smem, s);
        else if (mode == 1) split_launch_wm<1, 1>(G, p, cfg.grid, cfg.smem, s);
        else split_launch_wm<1, 2>(G, p, cfg.grid, cfg.smem, s);
    }
    return cudaGetLastError();
}

template <int MODE>
static cudaError_t ws_prep_m(int G, size_t smem, int* bps) {
    cudaError_t e = cudaSuccess;
    ws_dispatch<MODE>(G, [&](auto k) { e = split_prep(k, 64, smem, bps); });
    return e;
}

cudaError_t plan_ws(const RowOpParams& p, int S, int G, int num_sms, LaunchCfg* cfg) {
    if (S % 128 || S / 128 > 64 || G < 1 || G > 4) return cudaErrorInvalidValue;
    const size_t smem = ws_smem_bytes(S, p.old_mode != 0);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    int bps = 0;
    const int mode = split_mode_of(p);
    cudaError_t e = mode == 0 ? ws_prep_m<0>(G, smem, &bps) : mode == 1 ? ws_prep_m<1>(G, smem, &bps)
                                                                    : ws_prep_m<2>(G, smem, &bps);
    if (e) return e;
    if (bps < 1) return cudaErrorInvalidConfiguration;
    cfg->S = S;
    cfg->R = G;
    cfg->warps_per_cta = 2;
    cfg->smem = smem;
    cfg->bps = bps;
    const int64_t rows = p.row_end - p.row_begin;
    const int64_t full = (int64_t)bps * num_sms;
    cfg->grid = (int)(rows < full ? (rows > 0 ? rows : 1) : full);
    return cudaSuccess;
}

cudaError_t launch_ws(const RowOpParams& p, const LaunchCfg& cfg, cudaStream_t s) {
    const int mode = split_mode_of(p);
    auto go = [&](auto k) { k<<<cfg.grid, 64, cfg.smem, s>>>(p); };
    if (mode == 0) ws_dispatch<0>(cfg.R, go);
    else if (mode == 1) ws_dispatch<1>(cfg.R, go);
    else ws_dispatch<2>(cfg.R, go);
    return cudaGetLastError();
}

}  // namespace ell
