// spgemm.cu — the row kernels of libellpack (sm_100a, FP64 CUDA cores).
//
// One warp owns one output row at a time (BJ north_star (1): "a warp or small CTA owns each
// output row"); rows are handed out dynamically. Per row:
//   a1  window: the host probes the half-bandwidths of A, B (and Old) once per launch. If every
//       B row has <= 256 entries and a ring of S >= 2 h_B + 33 doubles keeps >= 4 rows per SM,
//       the ring path (row_fast_kernel) runs; otherwise the general path (row_general_kernel):
//       S-aligned windows of 1024 doubles, one pass per window the row touches, B rows split
//       at the window starts by precomputed breakpoints.
//   a2  gather + accumulate: for k ascending in A's row, every entry (j, b_kj) of B row k does
//       acc[j] = fma(a_ik, b_kj, acc[j]) in shared memory. The entries of one B row have
//       distinct columns, so they are applied in any order by the lanes; a __syncwarp between
//       consecutive k orders the read-modify-writes, so every output entry is the fma chain in
//       ascending k (reading R12 -> bitwise equal to the oracle). The ring path reads B from a
//       bank-balanced copy with the ring slots precomputed (balance_kernel) and gathers it in
//       half-ring register bursts (see row_ring).
//   a3  combine + drop + compact: Old entries (C_old / the SP2 iterate) are merged with
//       c = fma(alpha, s, beta*old); chunks of 32 columns keep |c| > tau, compact with
//       ballot/popc and write each chunk's kept run with one coalesced store per array,
//       counting overflow past C.w.
//   a4  per-row trace / norm inputs (stored a_ii, pre-drop s_ii, stored c_ii,
//       ||S - Old||^2), reduced later in canonical order (reduce.cu).
// With A = B = Old = X one launch is the fused SP2 step (BJ north_star (2)):
// SQUARE = (alpha 1, old_mode 2), EXPAND = (alpha -1, beta 2, old_mode 1) since
// fma(-1, s, 2x) = round(2x - s) exactly (2x is exact). For a bitwise-symmetric X the general
// kernel can compute only the columns j >= i of each row (p.upper, §8f-f4 ii); the
// sym_assemble_kernel below then writes each row as its mirrored lower part followed by U_i.
//
// Template parameters: G (64-entry groups per B row), HB (steps per register half), MODE
// (0: no Old operand; 1: Old operand; 2: Old operand + ||S - Old||^2 norm). Whether Old enters
// the value (beta*old, p.old_mode == 1) or only the union (p.old_mode == 2) is a runtime,
// warp-uniform choice.
#include "internal.cuh"
#include "devutil.cuh"
#include <climits>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

namespace ell {

#ifndef ELL_GEN_STAGE
#define ELL_GEN_STAGE 64
#endif
constexpr int kStage = ELL_GEN_STAGE;  // general path: A-row entries staged per piece
#ifndef ELL_SEG_PIPE
#define ELL_SEG_PIPE 1  // general path: software-pipelined rounds (accumulate_pipe)
#endif
#ifndef ELL_SEG_U
#define ELL_SEG_U 4  // general path: gathers per lane per round
#endif
#ifndef ELL_STAGE_F
#define ELL_STAGE_F 128  // fast path: stage entries (16 B each); 128 measured best vs 64, 96, 160, 192, 256
#endif
constexpr int kStageF = ELL_STAGE_F;
#ifndef ELL_ABLATE
#define ELL_ABLATE 0  // 1: compile the ELLPACK_OPT_ABLATE timing experiments into the ring kernel
#endif
// ablation bit b requested (always false in normal builds: no parameter read on the hot path)
#define ABL(p, b) (ELL_ABLATE && ((p).ablate & (b)))
#ifndef ELL_META_REGS
#define ELL_META_REGS 1  // fast path: keep step metadata in registers from the burst
#endif
#ifndef ELL_G3_HB
#define ELL_G3_HB 2  // fast path, 3 groups per step: steps per register half
#endif

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
__device__ __forceinline__ uint32_t stg_anb_a(const WarpSmem& w, int t) { return w.stg + 16u * kStage + 4u * t; }
__device__ __forceinline__ uint32_t stg_ast_a(const WarpSmem& w, int t) { return w.stg + 20u * kStage + 4u * t; }
__device__ __forceinline__ uint32_t stg_ak_a(const WarpSmem& w, int t) { return w.stg + 24u * kStage + 4u * t; }
__device__ __forceinline__ int stg_anb(const WarpSmem& w, int t) { return lds32i(stg_anb_a(w, t)); }
__device__ __forceinline__ int stg_ast(const WarpSmem& w, int t) { return lds32i(stg_ast_a(w, t)); }
__device__ __forceinline__ int stg_ak(const WarpSmem& w, int t) { return lds32i(stg_ak_a(w, t)); }

// acc has S + kTrash slots: acc[S .. S + 15] are trash slots (one per bank pair) that padding
// lanes of the fast path update; acc[S] is also the general path's trash slot.
constexpr int kTrash = 16;
__host__ __device__ inline size_t warp_smem_bytes(int S, bool has_old, bool fast) {
    return (size_t)(S + kTrash) * 8 + (fast ? (size_t)kStageF * 16 : (size_t)kStage * 28) + (has_old ? (size_t)S : 0);
}


// ------------------------------------------------------------- bank-balanced B (fast path)
//
// The accumulator of an output row is a ring of S doubles (S a multiple of 32): column j lives
// in slot j mod S for every row (the ring base is always a multiple of S), so the slot of a B
// entry does not depend on the output row and is precomputed here: the accumulate step is
// then LDS / DFMA / STS per entry, with no address arithmetic.
//
// Bank conflicts. Slot j mod S is bank pair j mod 16. Measured on B200 (tools/bank_bench.cu):
// a warp-wide 64-bit shared access is served as two 16-lane halves; each half costs as many
// wavefronts as its most-repeated bank pair (loads retire two wavefronts per clock, stores
// one). Column indices of a sorted B row are random modulo 16, so consecutive entries cost
// 3-6 wavefronts per instruction (r01 profile). The entries of ONE B row have distinct
// columns, so the order in which the lanes apply them within a step is free: the fma chain of
// every output entry stays ascending in k (R12). Each B row is stored permuted:
//   1. rank the row's entries by residue r = j mod 16 (stable counting sort): e in [0, n);
//   2. deal the ranks round-robin over NB = ceil(n / 16) half-instruction bins:
//      bin b = e mod NB, position m = e / NB (a residue with c_r <= NB entries lands in
//      c_r distinct bins);
//   3. bin b is half h = (b >> 1) & 1 of instruction (group g = b >> 2, parity b & 1):
//      slot 64 g + 2 (16 h + m) + (b & 1), so a lane's two slots of a group are adjacent
//      (one 8-byte index load, one 16-byte value load);
//   4. unused positions of a used group are padding: value 0 and a trash slot S + m (m the
//      position in the bin: distinct bank pairs among a bin's padding lanes), so padding lanes
//      run the same LDS / DFMA / STS.
// Record of row k (12 * 64 G bytes): int32 slot8[64 G] (= 8 * slot) then f64 val[64 G].
// bt_nbin[k] = NB: group g holds entries iff NB > 4 g.
__global__ void balance_kernel(KMat b, int64_t k0, int64_t k1, int wt, int S, unsigned char* __restrict__ bt,
                               int32_t* __restrict__ bt_nbin) {
    __shared__ int hist_s[8][16];        // per warp: entries per residue (256-thread blocks)
    __shared__ unsigned bmask_s[8][16];  // per warp and bin: residues of its real entries
    // per warp: the record is assembled here (scattered slots) and leaves in coalesced 16-byte
    // stores: int32 slots [256] then f64 values [256] (the used groups' prefixes are copied)
    __shared__ __align__(16) unsigned char rec_s[8][12 * 256];
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int* hist = hist_s[threadIdx.x >> 5];
    unsigned* bmask = bmask_s[threadIdx.x >> 5];
    int32_t* so = reinterpret_cast<int32_t*>(rec_s[threadIdx.x >> 5]);
    double* sv = reinterpret_cast<double*>(rec_s[threadIdx.x >> 5] + 4 * 256);
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double invS = 1.0 / (double)S;
    for (int64_t k = k0 + w0; k < k1; k += nw) {
        const int nb = b.nnz[k];  // <= 256 on the fast path (8 chunks)
        // bins: every bin of the 64-entry groups a step loads anyway (4 ceil(nb / 64), not
        // ceil(nb / 16)), so the entries of a residue class spread over more bins: fewer
        // same-bank pairs in a half-instruction at no extra instruction or load
        const int NB = 4 * ((nb + 63) >> 6);
        const int32_t* __restrict__ bc = b.col + (size_t)k * b.w;
        const double* __restrict__ bv = b.val + (size_t)k * b.w;
        int32_t* __restrict__ oo = reinterpret_cast<int32_t*>(bt + (size_t)k * 12 * wt);
        double* __restrict__ ov = reinterpret_cast<double*>(bt + (size_t)k * 12 * wt + 4 * (size_t)wt);
        if (lane == 0) bt_nbin[k] = NB;
        if (lane < 16) { hist[lane] = 0; bmask[lane] = 0u; }
        __syncwarp();
        // rank within residue (stable: chunk order, then lane order): one match per chunk
        int jr[8], rk[8];
        double vr[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int q = 32 * c + lane;
            jr[c] = q < nb ? __ldg(bc + q) : -1;
            vr[c] = q < nb ? __ldg(bv + q) : 0.0;
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            rk[c] = 0;
            if (32 * c < nb) {  // warp-uniform
                const int res = jr[c] >= 0 ? (jr[c] & 15) : 16 + lane;  // padding lanes: unique keys
                const unsigned m = __match_any_sync(FULL, res);
                const int leader = __ffs(m) - 1;
                int base = 0;
                if (lane == leader && jr[c] >= 0) base = atomicAdd(&hist[res], __popc(m));
                base = __shfl_sync(FULL, base, leader);
                rk[c] = base + __popc(m & lt);
            }
        }
        __syncwarp();
        // exclusive prefix over the residues (lanes 0..15)
        int h = lane < 16 ? hist[lane] : 0, pre = h;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const int y = __shfl_up_sync(FULL, pre, o);
            if (lane >= o) pre += y;
        }
        pre -= h;  // exclusive
        // e / NB by multiply-high (exact for e < 2^16; NB == 1 has no 32-bit magic)
        const unsigned magic = NB > 1 ? 0xffffffffu / (unsigned)NB + 1u : 0u;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (32 * c < nb) {
                const int j = jr[c];
                const int e = __shfl_sync(FULL, pre, j >= 0 ? (j & 15) : 0) + rk[c];
                if (j >= 0) {
                    const int pos = NB > 1 ? (int)__umulhi((unsigned)e, magic) : e;
                    const int bin = e - pos * NB;
                    const int sl = 64 * (bin >> 2) + 2 * (16 * ((bin >> 1) & 1) + pos) + (bin & 1);
                    int qs = __double2int_rz((double)j * invS);
                    int js = j - qs * S;
                    js += js < 0 ? S : 0;
                    js -= js >= S ? S : 0;
                    so[sl] = 8 * js;
                    sv[sl] = vr[c];
                    atomicOr(&bmask[bin], 1u << (js & 15));  // bank pair of the slot
                }
            }
        }
        __syncwarp();
        // padding: bin b holds fill_b = ceil((nb - b) / NB) entries at positions 0..fill_b-1;
        // positions fill_b..15 get trash slots S + r, r distinct and unused by the bin's entries
        const int nbins = 4 * ((NB + 3) >> 2);
        for (int t = lane; t < nbins * 16; t += 32) {
            const int bb = t >> 4, m = t & 15;
            const int fill = bb < NB ? (nb - bb + NB - 1) / NB : 0;
            if (m >= fill) {
                const int sl = 64 * (bb >> 2) + 2 * (16 * ((bb >> 1) & 1) + m) + (bb & 1);
                // the (m - fill)-th residue no real entry of the bin uses (16 - distinct residues
                // >= the bin's padding positions), so padding lanes add no same-bank pair
                unsigned f = ~bmask[bb] & 0xffffu;
                for (int q = m - fill; q > 0; --q) f &= f - 1u;
                so[sl] = 8 * (S + ((__ffs(f) - 1 - S) & 15));
                sv[sl] = 0.0;
            }
        }
        __syncwarp();
        const int used = 16 * nbins;  // slots of the used groups (64 per group)
        for (int t = lane; t < used / 4; t += 32)
            reinterpret_cast<int4*>(oo)[t] = reinterpret_cast<const int4*>(so)[t];
        for (int t = lane; t < used / 2; t += 32)
            reinterpret_cast<int4*>(ov)[t] = reinterpret_cast<const int4*>(sv)[t];
        __syncwarp();
    }
}

cudaError_t launch_balance(KMat b, int64_t k0, int64_t k1, int wt, int S, unsigned char* bt, int32_t* bt_nbin,
                           int num_sms, cudaStream_t s) {
    if (k1 <= k0) return cudaSuccess;
    const int64_t blocks_needed = (k1 - k0 + 7) / 8;
    const int64_t cap = (int64_t)num_sms * 8;
    balance_kernel<<<(unsigned)(blocks_needed < cap ? blocks_needed : cap), 256, 0, s>>>(b, k0, k1, wt, S, bt,
                                                                                         bt_nbin);
    return cudaGetLastError();
}

// Fast-path stage: 16 B per A entry {a_ik f64, k i32, NB(k) i32} (one 16-byte shared load per step)
__device__ __forceinline__ void stage_fast_get(const WarpSmem& w, int t, double& a, int& k, int& nb) {
    unsigned long long x, y;
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(w.stg + 16u * t) : "memory");
    a = __longlong_as_double((long long)x);
    k = (int)(uint32_t)y;
    nb = (int)(y >> 32);
}

// ------------------------------------------------------------------------- general path

// Window accumulate of the general path: for staged step t, B row k's entries whose columns
// fall in the window [c0, c0 + S) are exactly the slots [ast(t), anb(t)) (precomputed
// breakpoints, windows aligned to multiples of S), so there is no range test and no cursor.
// Each round issues U independent gathers per lane (U * 32 entries) before the updates.
template <int U>
__device__ __forceinline__ void accumulate_seg(const RowOpParams& p, const WarpSmem& w, int lane, int cnt, int c0) {
    const int32_t* __restrict__ bcol = p.B.col;
    const double* __restrict__ bval = p.B.val;
    const uint32_t abase = w.acc - 8u * (uint32_t)c0;
    for (int t = 0; t < cnt; ++t) {
        const long long bo = stg_boff(w, t);
        const int e = stg_anb(w, t);
        int q0 = stg_ast(w, t);
        const double a = stg_aa(w, t);
        if (e - q0 <= 32) {  // short segment (wide sparse rows): one entry per lane
            const int q = q0 + lane;
            const int j = q < e ? __ldg(bcol + bo + q) : -1;
            const double v = q < e ? __ldg(bval + bo + q) : 0.0;
            const double x = lds64_if(j >= 0, abase + 8u * (uint32_t)j);
            sts64_if(j >= 0, abase + 8u * (uint32_t)j, __fma_rn(a, v, x));
            __syncwarp();
            continue;
        }
        for (; q0 < e; q0 += 32 * U) {
            int j[U];
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = q0 + 32 * u + lane;
                j[u] = q < e ? __ldg(bcol + bo + q) : -1;
                v[u] = q < e ? __ldg(bval + bo + q) : 0.0;
            }
            double x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) x[u] = lds64_if(j[u] >= 0, abase + 8u * (uint32_t)j[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) sts64_if(j[u] >= 0, abase + 8u * (uint32_t)j[u], __fma_rn(a, v[u], x[u]));
        }
        __syncwarp();
    }
}

// Software-pipelined variant: the segments' rounds (U * 32 entries of one B row each) form one
// sequence; round r + 1's gathers are issued before round r's updates, into the other of two
// register sets. ptxas gives every gather the same scoreboard and a consumer waits for the
// youngest, so round r's registers are first touched (a store to the trash slot, issued while
// nothing younger is in flight), then round r + 1 is issued, then round r's updates run on
// ready registers. Rounds of consecutive segments stay in program order (the accumulator RAW).
template <int U>
__device__ __forceinline__ void accumulate_pipe(const RowOpParams& p, const WarpSmem& w, int lane, int cnt, int c0) {
    if (cnt <= 0) return;
    const int32_t* __restrict__ bcol = p.B.col;
    const double* __restrict__ bval = p.B.val;
    const uint32_t abase = w.acc - 8u * (uint32_t)c0;
    const uint32_t trash = w.acc + 8u * (uint32_t)p.S;
    int t = 0;
    long long bo = stg_boff(w, 0);
    int e = stg_anb(w, 0), q0 = stg_ast(w, 0);
    double a = stg_aa(w, 0);
    int j0[U], j1[U];
    double v0[U], v1[U];
    double a0 = a, a1 = 0.0;
    auto load = [&](int (&j)[U], double (&v)[U]) {
        // one 64-bit base per round; the U gathers use immediate offsets from it
        const int32_t* __restrict__ cp = bcol + bo + q0 + lane;
        const double* __restrict__ vp = bval + bo + q0 + lane;
        const int rem = e - q0 - lane;  // entries left for this lane's slot 0
#pragma unroll
        for (int u = 0; u < U; ++u) {
            j[u] = 32 * u < rem ? __ldg(cp + 32 * u) : -1;
            v[u] = 32 * u < rem ? __ldg(vp + 32 * u) : 0.0;
        }
    };
    auto advance = [&]() -> bool {  // cursor to the next round; false past the last segment
        q0 += 32 * U;
        if (q0 < e) return true;
        if (++t >= cnt) return false;
        bo = stg_boff(w, t);
        e = stg_anb(w, t);
        q0 = stg_ast(w, t);
        a = stg_aa(w, t);
        return true;
    };
    auto update = [&](const int (&j)[U], const double (&v)[U], double aa) {
        double x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = lds64_if(j[u] >= 0, abase + 8u * (uint32_t)j[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) sts64_if(j[u] >= 0, abase + 8u * (uint32_t)j[u], __fma_rn(aa, v[u], x[u]));
    };
    load(j0, v0);
    for (;;) {
        sts32i(trash, j0[0]);  // touch round r (set 0)
        bool more = advance();
        if (more) { load(j1, v1); a1 = a; }
        update(j0, v0, a0);
        if (!more) break;
        sts32i(trash, j1[0]);  // touch round r + 1 (set 1)
        more = advance();
        if (more) { load(j0, v0); a0 = a; }
        update(j1, v1, a1);
        if (!more) break;
    }
    __syncwarp();
}

// Breakpoints of B for windows aligned to multiples of S: bp[k * np + q] = number of entries of
// row k with column < q * S (q = 0 .. np - 1, np = ceil(N / S) + 1). Warp per row, lanes
// binary-search the window starts.
__global__ void breakpoints_kernel(KMat b, int64_t n, int S, int np, int32_t* __restrict__ bp) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = w0; k < n; k += nw) {
        const int nb = b.nnz[k];
        const int32_t* __restrict__ bc = b.col + (size_t)k * b.w;
        for (int q = lane; q < np; q += 32) {
            const long long x = (long long)q * S;
            int lo = 0, hi = nb;  // first index with col >= x
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if ((long long)__ldg(bc + mid) < x) lo = mid + 1; else hi = mid;
            }
            bp[k * np + q] = lo;
        }
    }
}

cudaError_t launch_breakpoints(KMat b, int64_t n, int S, int np, int32_t* bp, int num_sms, cudaStream_t s) {
    const int64_t blocks_needed = (n + 7) / 8;
    const int64_t cap = (int64_t)num_sms * 8;
    breakpoints_kernel<<<(unsigned)(blocks_needed < cap ? blocks_needed : cap), 256, 0, s>>>(b, n, S, np, bp);
    return cudaGetLastError();
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

// Combine the Old entries with columns < Fe (ascending, from old_cur) into the ring:
// s <- fma(alpha, s, beta*old) (old_mode 1) or fma(alpha, s, +0) (old_mode 2, with the
// ||S - Old||^2 term), and flag the slot so the emit does not scale it again.
template <int MODE>
__device__ __forceinline__ void ring_merge_old(const RowOpParams& p, const WarpSmem& w, int lane, int Fe,
                                               int baseF, const int32_t* o_col, const double* o_val, int nOld,
                                               int& old_cur, double& nrm) {
    const int S = p.S;
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

// Emit NCH consecutive 32-column chunks [F, F + 32 NCH) (column j lives in ring slot
// j - baseF, minus S past the wrap): pre-combine diagonal, combine with Old, drop, compact
// (NCH independent ballots) and write; the slots (and flags) are cleared. One slot per lane
// per chunk, so each chunk's kept entries are ONE contiguous run written by one store
// instruction per array (fully coalesced). A1: alpha == 1 (no scaling of product-only slots).
template <int MODE, int NCH, bool A1>
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
    if (MODE != 0) ring_merge_old<MODE>(p, w, lane, Fe, baseF, o_col, o_val, nOld, old_cur, nrm);
    double x[NCH];
    unsigned m[NCH];
    const double tau = p.tau;
    // slot of chunk c: pc0 + 32 c, minus S from the chunk where the ring wraps (S, pc0 multiples
    // of 32: a chunk never straddles the wrap)
    const int pc0 = F - baseF;
    const uint32_t sa0 = w.acc + 8u * (uint32_t)(pc0 + lane);
    const uint32_t wrapb = 8u * (uint32_t)S;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const uint32_t pa = sa0 + 256u * c - (pc0 + 32 * c >= S ? wrapb : 0u);
        const double v = lds64_clear(pa);  // read the slot and leave +0.0 behind (one instruction)
        bool flagged = false;
        if (MODE != 0) {
            const uint32_t fa = w.flg + (uint32_t)(pc0 + 32 * c - (pc0 + 32 * c >= S ? S : 0) + lane);
            flagged = lds8(fa) != 0;
            sts8(fa, 0u);
        }
        x[c] = v;
        if (!flagged) {
            if (!A1) x[c] = __dmul_rn(p.alpha, v);
            if (MODE == 2) nrm = __fma_rn(v, v, nrm);
        }
        m[c] = __ballot_sync(FULL, fabs(x[c]) > tau);
    }
    const unsigned lt = (1u << lane) - 1u;
    const int cw = p.C.w;
    const uint64_t bv = opaque_u64((uint64_t)crow_v), bc = opaque_u64((uint64_t)crow_c);
    // the width test is needed only when this block can reach the row's end (overflow rows)
    const bool room = kept + 32 * NCH <= cw && !ABL(p, 1);
    int before = kept;
    const int col0 = F + lane;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const bool keep = (m[c] >> lane) & 1u;
        const uint32_t pos = (uint32_t)before + (uint32_t)__popc(m[c] & lt);
        const int col = col0 + 32 * c;
        st_entry(keep && (room || (pos < (uint32_t)cw && !ABL(p, 1))), reinterpret_cast<double*>(bv + 8ull * pos),
                 reinterpret_cast<int32_t*>(bc + 4ull * pos), x[c], col);
        if (MODE != 0 && (int64_t)col == i) dc = keep ? x[c] : 0.0;
        before += __popc(m[c]);
    }
    kept = before;
}

#ifndef ELL_EMIT_NCH
#define ELL_EMIT_NCH 4  // ring emission: 32-column chunks per block (<= 4: a block wraps at most once)
#endif
// Emit [F, Fto) (multiples of 32), ELL_EMIT_NCH chunks at a time where possible; advances F, baseF.
template <int MODE, bool A1>
__device__ __forceinline__ void ring_emit_range_t(const RowOpParams& p, const WarpSmem& w, int lane, int64_t i,
                                                  int& F, int& baseF, int Fto, const int32_t* o_col,
                                                  const double* o_val, int nOld, int& old_cur,
                                                  double* __restrict__ crow_v, int32_t* __restrict__ crow_c,
                                                  int& kept, double& ds, double& dc, double& nrm) {
    while (p.S >= 256 && F + 32 * ELL_EMIT_NCH <= Fto) {  // a block of <= 128 columns wraps at most once
        ring_emit_block<MODE, ELL_EMIT_NCH, A1>(p, w, lane, i, F, baseF, o_col, o_val, nOld, old_cur, crow_v,
                                                crow_c, kept, ds, dc, nrm);
        F += 32 * ELL_EMIT_NCH;
        while (F - baseF >= p.S) baseF += p.S;
    }
    while (F < Fto) {
        ring_emit_block<MODE, 1, A1>(p, w, lane, i, F, baseF, o_col, o_val, nOld, old_cur, crow_v, crow_c, kept,
                                     ds, dc, nrm);
        F += 32;
        if (F - baseF >= p.S) baseF += p.S;
    }
    __syncwarp();
}

template <int MODE>
__device__ __forceinline__ void ring_emit_range(const RowOpParams& p, const WarpSmem& w, int lane, int64_t i,
                                                int& F, int& baseF, int Fto, const int32_t* o_col,
                                                const double* o_val, int nOld, int& old_cur,
                                                double* __restrict__ crow_v, int32_t* __restrict__ crow_c,
                                                int& kept, double& ds, double& dc, double& nrm) {
    if (ABL(p, 8)) {  // timing experiment: no emission work at all
        while (F < Fto) {
            F += 32;
            if (F - baseF >= p.S) baseF += p.S;
        }
        return;
    }
    if (p.alpha == 1.0)
        ring_emit_range_t<MODE, true>(p, w, lane, i, F, baseF, Fto, o_col, o_val, nOld, old_cur, crow_v, crow_c,
                                      kept, ds, dc, nrm);
    else
        ring_emit_range_t<MODE, false>(p, w, lane, i, F, baseF, Fto, o_col, o_val, nOld, old_cur, crow_v, crow_c,
                                       kept, ds, dc, nrm);
}

// One output row on the ring fast path. B is the bank-balanced copy (p.bt, 64 G slots per
// row, precomputed ring slots); A's row is staged in pieces of at most kPieceF entries,
// padded with null steps (nb = 0: no loads, no accumulator access) to whole halves of HB
// steps.
//
// Gathers go straight to registers in bursts of one half (HB steps) into a two-half register
// ring. ptxas gives every gather the same variable-latency scoreboard and a consumer waits
// for the whole scoreboard (i.e. for the youngest gather), and it drains the scoreboard at
// loop heads and control-flow joins. So a half runs: touch its own registers (waits for its
// burst, issued one half earlier, while nothing younger is outstanding) -> emit if needed
// (branchy; nothing young to drain) -> issue the next half's burst -> HB branch-free steps
// whose operands are all ready. A step is, per entry, LDS -> DFMA -> STS on the precomputed
// slot (padding lanes hit trash slots).
//
// Before a half, every column below floor32(k_first - hB) is final and is emitted when the
// half's first step would otherwise wrap onto it; if the whole half then fits the ring
// (k_last + hB < F + S) its steps need no checks, else (rare: k jumps > slack) the half runs
// step by step with per-step emission checks.

template <int G, int HB, int MODE>
__device__ __forceinline__ void row_ring(const RowOpParams& p, const WarpSmem& w, int lane, int64_t i,
                                         const int32_t* a_col, const double* a_val, int nA,
                                         const int32_t* o_col, const double* o_val, int nOld,
                                         double* __restrict__ crow_v, int32_t* __restrict__ crow_c,
                                         int& kept, double& ds, double& dc, double& nrm) {
    constexpr int kPieceF = kStageF - 2 * HB + 1;  // real steps per piece (room for padding + a null half)
    constexpr int RS = 12 * 64 * G;                // balanced row record bytes (p.bt_w == 64 G)
    const int S = p.S;
    const int hB = p.hB;
    const int ncols = (int)p.ncols;
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
    int old_cur = 0;
    const uint32_t acc = w.acc;
    const unsigned char* __restrict__ btl = p.bt + 8 * lane;  // this lane's slot pair of a record
    const uint64_t pol = l2_evict_last_policy();

    int2 ro[2][HB][G];
    double2 rv[2][HB][G];
#if ELL_META_REGS
    double am[2][HB];  // per-step metadata of each register half (read once, by the burst)
    int km[2][HB], nbm[2][HB];
#endif
#if ELL_META_REGS
    // the stage metadata (a, k, nb) of half h into register half X: read at the top of the
    // previous half so the shared-load latency overlaps its touch wait
    auto meta = [&](auto Xc, int h) {
        constexpr int X = decltype(Xc)::value;
#pragma unroll
        for (int e = 0; e < HB; ++e) stage_fast_get(w, h * HB + e, am[X][e], km[X][e], nbm[X][e]);
    };
#endif
    // burst: the gathers of half h into register half X
    auto burst = [&](auto Xc, int h) {
        constexpr int X = decltype(Xc)::value;
#pragma unroll
        for (int e = 0; e < HB; ++e) {
#if ELL_META_REGS
            const int nb = ABL(p, 4) ? 0 : nbm[X][e];
            const unsigned char* __restrict__ rp = btl + (size_t)(uint32_t)km[X][e] * RS;
#else
            double a_u;
            int k_u, nb_u;
            stage_fast_get(w, h * HB + e, a_u, k_u, nb_u);
            const int nb = ABL(p, 4) ? 0 : nb_u;
            const unsigned char* __restrict__ rp = btl + (size_t)(uint32_t)k_u * RS;
#endif
            const unsigned char* __restrict__ vp = rp + 8 * lane;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                // immediate offsets: indices at 256 g, values at 256 G + 512 g (+ 8 lane via vp)
                if (g == 0) { ldg_keep_i2_if<0>(nb > 0, rp, pol, ro[X][e][0]); ldg_keep_d2_if<256 * G>(nb > 0, vp, pol, rv[X][e][0]); }
                if (g == 1) { ldg_keep_i2_if<256>(nb > 4, rp, pol, ro[X][e][1]); ldg_keep_d2_if<256 * G + 512>(nb > 4, vp, pol, rv[X][e][1]); }
                if (g == 2) { ldg_keep_i2_if<512>(nb > 8, rp, pol, ro[X][e][2]); ldg_keep_d2_if<256 * G + 1024>(nb > 8, vp, pol, rv[X][e][2]); }
                if (g == 3) { ldg_keep_i2_if<768>(nb > 12, rp, pol, ro[X][e][3]); ldg_keep_d2_if<256 * G + 1536>(nb > 12, vp, pol, rv[X][e][3]); }
            }
        }
    };
    // accumulate one step from register half X, slot e
    auto step = [&](int X, int e, double a, int nb) {
        double old[G][2];
        bool gl[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            gl[g] = nb > 4 * g && !ABL(p, 2);  // warp-uniform: group holds entries
            old[g][0] = lds64_if(gl[g], acc + (uint32_t)ro[X][e][g].x);
            old[g][1] = lds64_if(gl[g], acc + (uint32_t)ro[X][e][g].y);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            sts64_if(gl[g], acc + (uint32_t)ro[X][e][g].x, __fma_rn(a, rv[X][e][g].x, old[g][0]));
            sts64_if(gl[g], acc + (uint32_t)ro[X][e][g].y, __fma_rn(a, rv[X][e][g].y, old[g][1]));
        }
        __syncwarp();
    };
    // one half of HB steps from register half X
    auto half = [&](auto Xc, int h) {
        constexpr int X = decltype(Xc)::value;
#if ELL_META_REGS
        const double* a_ = am[X];
        const int* k_ = km[X];
        const int* nb_ = nbm[X];
#else
        // step metadata re-read from the stage (fewer live registers across the half)
        double a_[HB];
        int k_[HB], nb_[HB];
#pragma unroll
        for (int e = 0; e < HB; ++e) stage_fast_get(w, h * HB + e, a_[e], k_[e], nb_[e]);
#endif
#if ELL_META_REGS
        meta(std::integral_constant<int, X ^ 1>{}, h + 1);
#endif
        // touch this half's burst: the store waits for it (and for nothing younger)
        if (nb_[0] > 0) sts32i(acc + 8u * (uint32_t)S, ro[X][0][0].x);
        const int kf = k_[0], kl = k_[HB - 1];
        if (kf + hB >= F + S)
            ring_emit_range<MODE>(p, w, lane, i, F, baseF, (kf - hB) & ~31, o_col, o_val, nOld, old_cur,
                                  crow_v, crow_c, kept, ds, dc, nrm);
        __syncwarp();
        burst(std::integral_constant<int, X ^ 1>{}, h + 1);  // the next half (a null half past the piece end: no loads)
        if (kl + hB < F + S) {
#pragma unroll
            for (int e = 0; e < HB; ++e) step(X, e, a_[e], nb_[e]);
        } else {
#pragma unroll
            for (int e = 0; e < HB; ++e) {
                const int kt = k_[e];
                if (kt + hB >= F + S)
                    ring_emit_range<MODE>(p, w, lane, i, F, baseF, (kt - hB) & ~31, o_col, o_val, nOld, old_cur,
                                          crow_v, crow_c, kept, ds, dc, nrm);
                step(X, e, a_[e], nb_[e]);
            }
        }
    };
    for (int p0 = 0; p0 < nA; p0 += kPieceF) {
        const int cnt = min(kPieceF, nA - p0);
        const int nh = (cnt + HB - 1) / HB;  // halves, the last padded with null steps
        // stage: real steps, then null steps (k = last real k, nb = 0, a = 0) through half nh
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
            asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(w.stg + 16u * q),
                         "l"(__double_as_longlong(a)), "l"(knb) : "memory");
        }
        __syncwarp();
#if ELL_META_REGS
        meta(std::integral_constant<int, 0>{}, 0);
#endif
        burst(std::integral_constant<int, 0>{}, 0);
        for (int h = 0; h < nh; h += 2) {
            half(std::integral_constant<int, 0>{}, h);
            if (h + 1 < nh) half(std::integral_constant<int, 1>{}, h + 1);
        }
    }
    // final chunks
    ring_emit_range<MODE>(p, w, lane, i, F, baseF, Fend, o_col, o_val, nOld, old_cur, crow_v, crow_c, kept, ds,
                          dc, nrm);
    dc = warp_sum(dc);  // only the diagonal's lane holds a nonzero value (x + 0 = x exactly)
}

// -------------------------------------------------------------------------------- kernel

// Per-warp shared layout setup (window/ring + stage + flags).
template <int MODE>
__device__ __forceinline__ WarpSmem warp_smem(unsigned char* smem_raw, int wid, int S, bool fast) {
    unsigned char* base = smem_raw + (size_t)wid * warp_smem_bytes(S, MODE != 0, fast);
    WarpSmem w;
    w.acc = (uint32_t)__cvta_generic_to_shared(base);
    w.stg = w.acc + (uint32_t)((S + kTrash) * 8);
    w.flg = w.acc + (uint32_t)((S + kTrash) * 8 + (fast ? kStageF * 16 : kStage * 28));
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


// Next ticket (relative to row_begin) for this warp: lane 0 takes it, all lanes get it.
__device__ __forceinline__ int64_t next_row(const RowOpParams& p, int lane) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(p.row_ticket, 1ull);
    return (int64_t)__shfl_sync(FULL, t, 0);
}

// Fast kernel: ring window, every row single-pass (host-verified: ring >= 2 hB + 33,
// B rows <= 64 G entries). One warp per CTA: the ring base is then a compile-time constant
// and folds into the shared-memory address of every accumulator access.
template <int G, int B, int MODE>
__global__ void __launch_bounds__(32, 8) row_fast_kernel(const RowOpParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x;
    const WarpSmem w = warp_smem<MODE>(smem_raw, 0, p.S, true);
    clear_window<MODE>(w, lane, p.S);
    const int64_t gw = blockIdx.x;
    int32_t my_max_kept = 0, my_ovf = 0;
    // Rows are handed out dynamically (one atomic per row): 6 resident warps share 4 schedulers
    // unevenly (2, 2, 1, 1), so a static stride would leave the lone warps idle at the tail.
    // Tickets hand out chunks of p.row_chunk consecutive rows (fewer atomics on the critical path,
    // neighbouring rows share B records in L2).
    // (p.row_chunk: 4, or 1 when a launch has < 64 rows per warp so the tail stays short)
    const int chunk = p.row_chunk;
    for (int64_t i0 = p.row_begin + chunk * next_row(p, lane); i0 < p.row_end;
         i0 = p.row_begin + chunk * next_row(p, lane))
    for (int64_t i = i0; i < i0 + chunk && i < p.row_end; ++i) {
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
        row_ring<G, B, MODE>(p, w, lane, i, r.a_col, r.a_val, r.nA, r.o_col, r.o_val, r.nOld, r.crow_v, r.crow_c,
                             kept, ds, dc, nrm);
        row_epilogue<MODE>(p, lane, i, kept, dA, ds, dc, nrm, my_max_kept, my_ovf);
    }
    flush_status(p, lane, my_max_kept, my_ovf);
}

// General kernel: span pre-pass + one pass per S-aligned window the row touches; B rows are
// split at window boundaries by precomputed breakpoints (rows wider than any ring that fits
// shared memory, B rows > 256 entries: the densifying SP2 iterates).
#ifndef ELL_GEN_MINB
#define ELL_GEN_MINB 1  // general kernel: min resident 128-thread CTAs per SM (register cap)
#endif
template <int MODE>
__device__ __forceinline__ void row_general_body(const RowOpParams& p, unsigned char* smem_raw) {
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int S = p.S;
    const WarpSmem w = warp_smem<MODE>(smem_raw, wid, S, false);
    clear_window<MODE>(w, lane, S);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
    int32_t my_max_kept = 0, my_ovf = 0;
    unsigned long long my_exec = 0;  // products this lane staged (p.exec_products)
    for (int64_t i = p.row_begin + next_row(p, lane); i < p.row_end; i = p.row_begin + next_row(p, lane)) {
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
            // ---- general path: span pre-pass, then one pass per window [q S, (q + 1) S) that
            //      the row's span touches (windows aligned so breakpoints are per B row)
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
            lo = warp_min(lo);
            if (p.upper) lo = max(lo, (int)i);  // symmetric step: columns j >= i only
            lo &= ~1;  // even window start (16-byte slot pairs)
            hi = warp_max(hi);
            if (hi >= lo) {
                const bool multi = hi / S > lo / S;  // more than one aligned window
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
                __syncwarp();
                int old_cur = 0;
                if (MODE != 0 && p.upper) {  // Old entries below the diagonal belong to L_i
                    int lo_o = 0, hi_o = nOld;
                    while (lo_o < hi_o) {
                        const int mid = (lo_o + hi_o) >> 1;
                        if (o_col[mid] < (int)i) lo_o = mid + 1; else hi_o = mid;
                    }
                    old_cur = lo_o;
                }
                const int np = p.bp_np;
                for (int pass = lo / S; pass <= hi / S; ++pass) {
                    const int c0 = pass * S;
                    const int width = min(S, (int)p.ncols - c0 + 1) & ~1;  // even, covers [c0, min(c0 + S, N))
                    for (int p0 = 0; p0 < nA; p0 += kStage) {
                        const int cnt = min(kStage, nA - p0);
                        // stage (compacted, k ascending): B-row offset, a_ik and the window's slot
                        // range [bp(k, pass), bp(k, pass + 1)) of the A entries whose B row has
                        // entries in this window -- wide sparse rows touch few k per window
                        int ns = 0;
                        for (int q0 = 0; q0 < cnt; q0 += 32) {
                            const int q = q0 + lane;
                            int k = 0, sb = 0, se = 0;
                            if (q < cnt) {
                                k = a_col[p0 + q];
                                if (p.bp) {
                                    const int32_t* bpk = p.bp + (size_t)k * np + pass;
                                    sb = __ldg(bpk);
                                    se = __ldg(bpk + 1);
                                } else {  // one window covers every column (S >= N): the whole B row
                                    se = __ldg(p.B.nnz + k);
                                }
                                if (p.upper && c0 <= (int)i && (int64_t)i < (int64_t)c0 + S) {
                                    // first entry of B row k with column >= i
                                    const int32_t* bck = p.B.col + (size_t)k * p.B.w;
                                    int lo_b = sb, hi_b = se;
                                    while (lo_b < hi_b) {
                                        const int mid = (lo_b + hi_b) >> 1;
                                        if (__ldg(bck + mid) < (int)i) lo_b = mid + 1; else hi_b = mid;
                                    }
                                    sb = lo_b;
                                }
                            }
                            const bool ne = se > sb;
                            if (ne) my_exec += (unsigned long long)(se - sb);
                            const unsigned m = __ballot_sync(FULL, ne);
                            if (ne) {
                                const int t = ns + __popc(m & ((1u << lane) - 1u));
                                const long long bo = (long long)k * p.B.w;
                                asm volatile("st.shared.s64 [%0], %1;" ::"r"(w.stg + 8u * t), "l"(bo) : "memory");
                                sts64(w.stg + 8u * (kStage + t), a_val[p0 + q]);
                                sts32i(stg_ast_a(w, t), sb);
                                sts32i(stg_anb_a(w, t), se);
                            }
                            ns += __popc(m);
                        }
                        __syncwarp();
#if ELL_SEG_PIPE
                        accumulate_pipe<ELL_SEG_U>(p, w, lane, ns, c0);
#else
                        accumulate_seg<ELL_SEG_U>(p, w, lane, ns, c0);
#endif
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
    if (p.exec_products) {
#pragma unroll
        for (int o = 16; o; o >>= 1) my_exec += __shfl_xor_sync(FULL, my_exec, o);
        if (lane == 0 && my_exec) atomicAdd(p.exec_products, my_exec);
    }
}


template <int MODE>
__global__ void __launch_bounds__(128, ELL_GEN_MINB) row_general_kernel(const RowOpParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    row_general_body<MODE>(p, smem_raw);
}

// The same kernel with (alpha, beta, old_mode) read from device memory (p.dyn): the SP2 step of
// the device-resident loop (§8f-f3), whose branch is decided on the device between launches of
// one captured CUDA graph.
template <int MODE>
__global__ void __launch_bounds__(128, ELL_GEN_MINB) row_general_dyn_kernel(const RowOpParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RowOpParams q = p;
    q.alpha = p.dyn[0];
    q.beta = p.dyn[1];
    q.old_mode = (int)p.dyn[2];
    row_general_body<MODE>(q, smem_raw);
}

// Half-bandwidth probe: out[m] = max over rows of max(i - col[i][0], col[i][nnz-1] - i) (a and c
// over rows [r0, r1), b over rows [b0, b1)); out[3] = max nnz of b over [b0, b1); out[4] = max over
// those B rows of the larger chunk-parity half (the split kernel's sub-rows, W = 2; counted only when
// count_sub, else out[4] = out[3]); the B rows the
// A rows [r0, r1) reference are [INT_MAX - out[5], out[6] - 1] (zero-initialised maxima of
// INT_MAX - first column and last column + 1).
__global__ void bandwidth_kernel(KMat a, KMat b, KMat c, int64_t r0, int64_t r1, int64_t b0, int64_t b1,
                                 int64_t n, int count_sub, int32_t* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int bw[3] = {0, 0, 0};
    int reach[2] = {0, 0};
    const KMat* ms[3] = {&a, &b, &c};
    if (i < n) {
#pragma unroll
        for (int m = 0; m < 3; ++m) {
            // A and Old only matter on the computed rows; B on its probed rows
            if (m != 1 && (i < r0 || i >= r1)) continue;
            if (m == 1 && (i < b0 || i >= b1)) continue;
            const KMat& x = *ms[m];
            if (x.nnz == nullptr) continue;
            const int nz = x.nnz[i];
            if (nz > 0) {
                const int f = x.col[(size_t)i * x.w], l = x.col[(size_t)i * x.w + nz - 1];
                bw[m] = max(max((int)(i - f), (int)(l - i)), 0);
                if (m == 0) { reach[0] = INT_MAX - f; reach[1] = l + 1; }
            }
        }
    }
    int nzb = (i >= b0 && i < b1) ? b.nnz[i] : 0;
    // the larger chunk-parity half of the B row (split kernel, W = 2: columns j with (j >> 5) & 1)
    int sub = nzb;
    if (count_sub && nzb > 64 && nzb <= 256) {
        const int32_t* bc = b.col + (size_t)i * b.w;
        int odd = 0;
        for (int q = 0; q < nzb; ++q) odd += (bc[q] >> 5) & 1;
        sub = max(odd, nzb - odd);
    }
#pragma unroll
    for (int m = 0; m < 7; ++m) {
        int v = m < 3 ? bw[m] : (m == 3 ? nzb : (m == 4 ? sub : reach[m - 5]));
#pragma unroll
        for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
        if ((threadIdx.x & 31) == 0 && v > 0) atomicMax(out + m, v);
    }
}

cudaError_t launch_bandwidth(KMat a, KMat b, KMat c, int64_t r0, int64_t r1, int64_t b0, int64_t b1, int64_t n,
                             int count_sub, int32_t* out, cudaStream_t s) {
    bandwidth_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, b, c, r0, r1, b0, b1, n, count_sub, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------ symmetric SP2 step (f4 ii)
// S = X^2 of a bitwise-symmetric X is bitwise symmetric (each s_ji is the same fma chain over the
// same products as s_ij, P4), and so is X_{n+1}. The row kernel then computes only U_i (columns
// j >= i, upper = 1) and row i of X_{n+1} is L_i || U_i with L_i = column i of the rows j < i.

// bad[0] = 1 unless every stored (i, j, v) has a stored (j, i) with identical bits. Warp per row,
// one entry per lane (the binary searches of a row run side by side).
__global__ void sym_check_kernel(KMat h, int64_t r0, int64_t r1, int32_t* bad) {
    const int lane = threadIdx.x & 31;
    const int64_t i = r0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (i >= r1) return;
    const int nz = h.nnz[i];
    bool ok = true;
    for (int q = lane; q < nz && ok; q += 32) {
        const int j = h.col[(size_t)i * h.w + q];
        const int32_t* cj = h.col + (size_t)j * h.w;
        int lo = 0, hi = h.nnz[j];
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cj[mid] < (int)i) lo = mid + 1; else hi = mid;
        }
        ok = lo < h.nnz[j] && cj[lo] == (int)i &&
             __double_as_longlong(h.val[(size_t)j * h.w + lo]) == __double_as_longlong(h.val[(size_t)i * h.w + q]);
    }
    if (!ok) atomicOr(bad, 1);
}

cudaError_t launch_sym_check(KMat h, int64_t r0, int64_t r1, int32_t* bad, cudaStream_t s) {
    if (r1 <= r0) return cudaSuccess;
    sym_check_kernel<<<(unsigned)(((r1 - r0) * 32 + 255) / 256), 256, 0, s>>>(h, r0, r1, bad);
    return cudaGetLastError();
}

// reach[0] = max over rows j of (last column of U_j) - j  (the L_i gather range)
__global__ void upper_reach_kernel(KMat u, int64_t r0, int64_t r1, int32_t* reach) {
    const int64_t j = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int v = 0;
    if (j < r1) {
        const int nz = u.nnz[j];
        if (nz > 0) v = max(0, (int)(u.col[(size_t)j * u.w + nz - 1] - j));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
    if ((threadIdx.x & 31) == 0 && v > 0) atomicMax(reach, v);
}

cudaError_t launch_upper_reach(KMat u, int64_t r0, int64_t r1, int32_t* reach, cudaStream_t s) {
    const int64_t rows = r1 - r0;
    if (rows <= 0) return cudaSuccess;
    upper_reach_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(u, r0, r1, reach);
    return cudaGetLastError();
}

// Warp per row i: L_i by testing the candidate rows j in [i - reach, i) 32 at a time (binary search
// of column i in U_j; a ballot keeps ascending j), then U_i; status and the full Frobenius term.
__global__ void __launch_bounds__(256) sym_assemble_kernel(KMat u, KMat x, KOut y, int64_t r0, int64_t r1,
                                                           const int32_t* reach_p, const double* diag_s,
                                                           double* normsq, int32_t* status) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int reach = *reach_p;
    int32_t my_max = 0, my_ovf = 0;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = r0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < r1; i += nw) {
        double* yv = y.val + (size_t)i * y.w;
        int32_t* yc = y.col + (size_t)i * y.w;
        int kept = 0;
        const int64_t j0 = i - reach > 0 ? i - reach : 0;
        for (int64_t jb = j0; jb < i; jb += 32) {
            const int64_t j = jb + lane;
            bool found = false;
            double v = 0.0;
            if (j < i) {
                const int nz = u.nnz[j];
                const int32_t* cj = u.col + (size_t)j * u.w;
                if (nz > 0 && cj[nz - 1] >= (int)i) {
                    int lo = 0, hi = nz;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (cj[mid] < (int)i) lo = mid + 1; else hi = mid;
                    }
                    if (cj[lo] == (int)i) { found = true; v = u.val[(size_t)j * u.w + lo]; }
                }
            }
            const unsigned m = __ballot_sync(FULL, found);
            const int pos = kept + __popc(m & lt);
            if (found && pos < y.w) { yv[pos] = v; yc[pos] = (int32_t)j; }
            kept += __popc(m);
        }
        const int nu = u.nnz[i];
        for (int q = lane; q < nu; q += 32) {
            const int pos = kept + q;
            if (pos < y.w) {
                yv[pos] = u.val[(size_t)i * u.w + q];
                yc[pos] = u.col[(size_t)i * u.w + q];
            }
        }
        kept += nu;
        if (lane == 0) {
            y.nnz[i] = kept < y.w ? kept : y.w;
            if (normsq) {
                // upper norm counted (s - x)^2 once for j > i and once for j = i: full = 2 up - diag
                const int nx = x.nnz[i];
                const int32_t* cx = x.col + (size_t)i * x.w;
                int lo = 0, hi = nx;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (cx[mid] < (int)i) lo = mid + 1; else hi = mid;
                }
                const double xd = (lo < nx && cx[lo] == (int)i) ? x.val[(size_t)i * x.w + lo] : 0.0;
                const double d = __dsub_rn(diag_s[i], xd);
                normsq[i] = __fma_rn(2.0, normsq[i], -__dmul_rn(d, d));
            }
        }
        my_max = max(my_max, kept);
        if (kept > y.w) ++my_ovf;
    }
    if (lane == 0) {
        if (my_ovf) atomicAdd(status, my_ovf);
        if (my_max) atomicMax(status + 1, my_max);
    }
}

cudaError_t launch_sym_assemble(KMat u, KMat x, KOut y, int64_t r0, int64_t r1, const int32_t* reach,
                                const double* diag_s, double* normsq, int32_t* status, int num_sms,
                                cudaStream_t s) {
    const int64_t rows = r1 - r0;
    if (rows <= 0) return cudaSuccess;
    const int64_t blocks = (rows + 7) / 8;
    const int64_t cap = (int64_t)num_sms * 8;
    sym_assemble_kernel<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, s>>>(u, x, y, r0, r1, reach, diag_s,
                                                                                normsq, status);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------- dispatch

// Fast-kernel variants by G = ceil(max nnz_B / 64) (64-entry groups per step; prefetch
// half-ring B, the register ring holds 2 B slots): G1: B 4, G2: B 3, G3: B 3, G4: B 2.
// cfg.R carries G; cfg.R == 0 selects the general kernel.
template <typename K>
static cudaError_t prep_kernel(K kern, const LaunchCfg& cfg, int* bps) {
    return occupancy_cached((const void*)kern, cfg.warps_per_cta * 32, cfg.smem, bps);
}

template <int MODE>
static cudaError_t prep_mode(const LaunchCfg& cfg, int* bps) {
    switch (cfg.R) {
        case 0: {
            cudaError_t e = prep_kernel(row_general_dyn_kernel<MODE>, cfg, bps);
            return e ? e : prep_kernel(row_general_kernel<MODE>, cfg, bps);
        }
        case 1: return prep_kernel(row_fast_kernel<1, 4, MODE>, cfg, bps);
        case 2: return prep_kernel(row_fast_kernel<2, 3, MODE>, cfg, bps);
        case 3: return prep_kernel(row_fast_kernel<3, ELL_G3_HB, MODE>, cfg, bps);
        default: return prep_kernel(row_fast_kernel<4, 2, MODE>, cfg, bps);
    }
}

template <int MODE>
static void launch_mode(const RowOpParams& p, const LaunchCfg& cfg, cudaStream_t s) {
    dim3 block(cfg.warps_per_cta * 32), grid(cfg.grid);
    switch (cfg.R) {
        case 0:
            if (p.dyn) row_general_dyn_kernel<MODE><<<grid, block, cfg.smem, s>>>(p);
            else row_general_kernel<MODE><<<grid, block, cfg.smem, s>>>(p);
            break;
        case 1: row_fast_kernel<1, 4, MODE><<<grid, block, cfg.smem, s>>>(p); break;
        case 2: row_fast_kernel<2, 3, MODE><<<grid, block, cfg.smem, s>>>(p); break;
        case 3: row_fast_kernel<3, ELL_G3_HB, MODE><<<grid, block, cfg.smem, s>>>(p); break;
        default: row_fast_kernel<4, 2, MODE><<<grid, block, cfg.smem, s>>>(p); break;
    }
}

static int mode_of(const RowOpParams& p) { return p.old_mode == 0 ? 0 : (p.normsq ? 2 : 1); }

size_t row_op_warp_smem(int S, bool has_old, bool fast) { return warp_smem_bytes(S, has_old, fast); }

cudaError_t plan_row_op(const RowOpParams& p, int S, int groups, int warps_opt, int num_sms, LaunchCfg* cfg) {
    S = (S + 31) & ~31;
    const size_t per_warp = warp_smem_bytes(S, p.old_mode != 0, p.fast != 0);
    const size_t cap = 227 * 1024;
    if (per_warp > cap) return cudaErrorInvalidConfiguration;
    cfg->S = S;
    cfg->R = !p.fast ? 0 : (groups < 1 ? 1 : (groups > 4 ? 4 : groups));
    const int mode = mode_of(p);
    // warps per CTA: maximise resident warps (rows in flight) per SM under the shared-memory
    // and register limits; ties go to the larger CTA
    int best_w = 0, best_wpc = 1, best_bps = 0;
    int lo_w = warps_opt > 0 ? warps_opt : 1, hi_w = warps_opt > 0 ? warps_opt : 4;
    if (p.fast) lo_w = hi_w = 1;  // the fast kernel is one warp per CTA
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
    cfg->bps = bps;
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

cudaError_t occupancy_cached(const void* kern, int threads, size_t smem, int* bps) {
    struct Ent {
        const void* k;
        int dev, threads;
        size_t smem;
        int bps;
    };
    static std::mutex mu;
    static std::vector<Ent> tab;                        // (kernel, device, threads, smem) -> CTAs/SM
    static std::vector<std::pair<const void*, int>> lim;  // (kernel, device) -> smem limit set (bytes)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e) return e;
    std::lock_guard<std::mutex> g(mu);
    for (const Ent& t : tab)
        if (t.k == kern && t.dev == dev && t.threads == threads && t.smem == smem) {
            *bps = t.bps;
            return cudaSuccess;
        }
    int have = -1;
    for (auto& l : lim)
        if (l.first == kern && (l.second >> 20) == dev) have = l.second & 0xfffff;
    if (have < (int)smem) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e) return e;
        lim.push_back({kern, (dev << 20) | (int)smem});
    }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, kern, threads, smem);
    if (e) return e;
    tab.push_back({kern, dev, threads, smem, *bps});
    return cudaSuccess;
}

}  // namespace ell
