// dense.cu — dense-regime X^2 / SP2 step of libellpack (sm_100a, FP64 CUDA cores).
//
// Three kernels (dense.cuh states the exactness argument):
//  * densify_kernel: a warp per ELLPACK row scatters its entries into a zeroed np x np array and
//    marks the 128 x 16 / 16 x 128 blocks they fall in (the GEMM skips k blocks that are empty on
//    either side: banded iterates keep most of them empty until late in the run);
//  * dense_gemm_kernel: 128 x 128 tile per CTA, 256 threads with 8 x 8 outputs each, a 4-stage
//    cp.async pipeline of 16-row k blocks, k strictly ascending through the stages and inside each
//    -- every output is the fma chain s <- fma(a_ik, b_kj, s) in ascending k, which is the sparse
//    kernels' chain plus exact-zero terms. No tensor cores: tcgen05 has no FP64 kind, and DMMA's
//    internal summation order is not the chain's;
//  * dense_emit_kernel: a warp per output row walks the dense row (and the dense copy of Old) in
//    128-column steps, combines / drops / compacts as split_emit (split.cu) does, and writes the
//    ELLPACK row, its diagonals, its norm partial and the overflow status.
#include "dense.cuh"
#include "devutil.cuh"

#include <climits>
#include <mutex>

namespace ell {

// ------------------------------------------------------------------------------ densify

__global__ void __launch_bounds__(256) densify_kernel(KMat a, int64_t i0, int64_t i1, int np, int transpose,
                                                      double* __restrict__ D, unsigned char* __restrict__ fa,
                                                      unsigned char* __restrict__ fb) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int KB = np / kDenseK, T = np / kDenseTile;
    for (int64_t i = i0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < i1; i += nw) {
        const int nnz = a.nnz[i];
        const int32_t* c = a.col + (size_t)i * a.w;
        const double* v = a.val + (size_t)i * a.w;
        for (int q = lane; q < nnz; q += 32) {
            const int j = c[q];
            const double x = v[q];
            if (transpose) D[(size_t)j * np + i] = x;
            else D[(size_t)i * np + j] = x;
            if (fa) fa[(size_t)(i / kDenseTile) * KB + j / kDenseK] = 1;
            if (fb) fb[(size_t)(i / kDenseK) * T + j / kDenseTile] = 1;
        }
    }
}

cudaError_t launch_densify(KMat a, int64_t i0, int64_t i1, int np, bool transpose, double* D, unsigned char* fa,
                           unsigned char* fb, cudaStream_t s) {
    if (i1 <= i0) return cudaSuccess;
    const int64_t blocks = (i1 - i0 + 7) / 8;
    densify_kernel<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s>>>(a, i0, i1, np, transpose ? 1 : 0,
                                                                                   D, fa, fb);
    return cudaGetLastError();
}

// Byte flags -> bitsets, one bitset of k blocks per 128-row block (Fa, from fa [T][KB]) and per
// 128-column tile (Fb, from fb [KB][T]): the GEMM reads one 64-bit word per 64 k blocks instead of a
// byte per k block (with a strided column of fb) -- at N = 65536 every tile's scan is 64 words.
__global__ void __launch_bounds__(256) pack_flags_kernel(const unsigned char* __restrict__ fa,
                                                         const unsigned char* __restrict__ fb, int T, int KB,
                                                         int kbw, unsigned long long* __restrict__ Fa,
                                                         unsigned long long* __restrict__ Fb) {
    const int64_t total = (int64_t)T * kbw;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(t / kbw), w = (int)(t % kbw);
        unsigned long long a = 0ull, b = 0ull;
        for (int q = 0; q < 64; ++q) {
            const int kb = 64 * w + q;
            if (kb >= KB) break;
            if (fa[(size_t)r * KB + kb]) a |= 1ull << q;
            if (fb[(size_t)kb * T + r]) b |= 1ull << q;
        }
        Fa[t] = a;
        Fb[t] = b;
    }
}

cudaError_t launch_pack_flags(const unsigned char* fa, const unsigned char* fb, int np, unsigned long long* Fa,
                              unsigned long long* Fb, int num_sms, cudaStream_t s) {
    const int T = np / kDenseTile, KB = np / kDenseK, kbw = dense_kbw(np);
    const int64_t total = (int64_t)T * kbw;
    const int64_t blocks = (total + 255) / 256;
    pack_flags_kernel<<<(unsigned)(blocks < num_sms * 4 ? blocks : num_sms * 4), 256, 0, s>>>(fa, fb, T, KB, kbw, Fa, Fb);
    return cudaGetLastError();
}

// --------------------------------------------------------------------------------- GEMM

#ifndef ELL_DENSE_STAGES
#define ELL_DENSE_STAGES 4  // cp.async pipeline depth (k blocks in flight)
#endif
#ifndef ELL_DENSE_TY
#define ELL_DENSE_TY 16  // large tiles: 16 TY threads, 128 / TY rows x 8 columns each
#endif
constexpr int kDenseStages = ELL_DENSE_STAGES;

template <int BM>
__host__ __device__ constexpr int stage_bytes() { return (kDenseK * BM + kDenseK * kDenseTile) * 8; }  // At block + B block

size_t dense_gemm_smem(int np) { return (size_t)kDenseStages * stage_bytes<128>() + sizeof(int) * (size_t)(np / kDenseK); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

#ifndef ELL_DENSE_TMA
#define ELL_DENSE_TMA 1  // stages arrive by bulk copies on an mbarrier (1) or by per-thread cp.async (0)
#endif
__device__ __forceinline__ void dmbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void dmbar_expect(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void dmbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tDWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra DWAIT_%=;\n\t}" ::"r"(a), "r"(parity) : "memory");
}
// one contiguous global -> shared bulk copy (the TMA engine), completing `bytes` on the mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

__device__ __forceinline__ void stg128(double* p, double x, double y) {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(x), "d"(y) : "memory");
}

// A BM x 128 tile of S per CTA, 16 TY threads: thread (ty, tx) = (tid / 16, tid % 16) owns rows
// 2 TY g + 2 ty + r (g < RM / 2, r < 2) and columns 32 h + 2 tx + c (h < 4, c < 2). Its A and B
// fragments are 16-byte shared loads that a warp (two ty, sixteen tx) serves in 1 (A: two
// broadcast addresses) and 2 (B: 256 contiguous bytes) wavefronts.
//   BM = 128, TY = 16: 8 x 8 per thread, the large-N kernel (SYM: tiles bi <= bj, each also stored
//                      transposed);
//   BM = 16,  TY = 8:  2 x 8 per thread, 128 threads: small N, where 128-row tiles leave most SMs idle.
template <int BM, int TY, bool SYM>
__global__ void __launch_bounds__(16 * TY, BM == 128 ? (TY == 8 ? 2 : 1) : 4)
    dense_gemm_kernel(const double* __restrict__ At, const double* __restrict__ B, int np,
                      const unsigned long long* __restrict__ Fa, const unsigned long long* __restrict__ Fb,
                      double* __restrict__ S, unsigned char* __restrict__ tw, unsigned long long* exec, int bi0) {
    static_assert(!SYM || BM == kDenseTile, "symmetric tiles are square");
    constexpr int NT = 16 * TY, NW = NT / 32, RM = BM / TY, SB = stage_bytes<BM>();
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int wcnt[NW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = tid & 15, ty = tid >> 4;
    const int T = np / kDenseTile, KB = np / kDenseK;
    int bi, bj;  // bi: BM-row block, bj: 128-column block
    if (SYM) {
        int t = blockIdx.x;
        bi = 0;
        while (t >= T - bi) { t -= T - bi; ++bi; }
        bj = bi + t;
    } else {
        bi = bi0 + (int)(blockIdx.x / T);  // a rank's rows start at row block bi0
        bj = blockIdx.x % T;
    }
    const int bf = bi * BM / kDenseTile;  // the 128-row flag block of this tile's rows
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    int* list = reinterpret_cast<int*>(smem + kDenseStages * SB);
#if ELL_DENSE_TMA
    __shared__ __align__(8) unsigned long long fullbar[kDenseStages];
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(fullbar);
    if (tid == 0) {
#pragma unroll
        for (int st = 0; st < kDenseStages; ++st) dmbar_init(bar0 + 8u * st, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // (the first __syncthreads of the k-block scan below publishes the initialised barriers)
#endif
    // the k blocks with an entry on both sides, ascending: one 64-bit word of each bitset per thread
    const int kbw = dense_kbw(np);
    int nact = 0;
    for (int w0 = 0; w0 < kbw; w0 += NT) {
        const int w = w0 + tid;
        const unsigned long long m = w < kbw ? Fa[(size_t)bf * kbw + w] & Fb[(size_t)bj * kbw + w] : 0ull;
        const int cnt = __popcll(m);
        int incl = cnt;  // inclusive warp scan of the counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wcnt[warp] = incl;
        __syncthreads();
        int off = nact, tot = 0;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            off += q < warp ? wcnt[q] : 0;
            tot += wcnt[q];
        }
        off += incl - cnt;
        for (unsigned long long r = m; r; r &= r - 1) list[off++] = 64 * w + __ffsll((long long)r) - 1;
        __syncthreads();
        nact += tot;
    }
    (void)KB;
    const double* a0 = At + (size_t)bi * BM;
    const double* b0 = B + (size_t)bj * kDenseTile;
#if ELL_DENSE_TMA
    // warp 0: lane 0 arms the stage's barrier with its byte count, then 32 bulk copies (one k row of
    // A^T or of B each) complete on it -- the stage's arrival is tracked by the barrier, not by the
    // threads' scoreboards, so shared loads of the current stage never wait on the copies in flight
    auto load_stage = [&](int st, int kb) {
        const uint32_t sa = sbase + (uint32_t)(st * SB), sb = sa + (uint32_t)(kDenseK * BM * 8);
        const uint32_t bar = bar0 + 8u * (uint32_t)st;
        const size_t r0 = (size_t)kb * kDenseK;
        if (lane == 0) dmbar_expect(bar, (uint32_t)SB);
        __syncwarp();
        const int r = lane & 15;
        if (lane < 16) bulk_g2s(sa + (uint32_t)(r * BM * 8), a0 + (r0 + r) * np, (uint32_t)(BM * 8), bar);
        else bulk_g2s(sb + (uint32_t)(r * 1024), b0 + (r0 + r) * np, 1024u, bar);
    };
#else
    auto load_stage = [&](int st, int kb) {
        const uint32_t sa = sbase + (uint32_t)(st * SB), sb = sa + (uint32_t)(kDenseK * BM * 8);
        const size_t r0 = (size_t)kb * kDenseK;
        constexpr int CA = kDenseK * BM / 2, CB = kDenseK * kDenseTile / 2;  // 16-byte chunks
#pragma unroll
        for (int u = 0; u < (CA + NT - 1) / NT; ++u) {
            const int c = tid + NT * u;
            if (CA % NT == 0 || c < CA) {
                const int r = c / (BM / 2), q = c % (BM / 2);
                cp_async16(sa + (uint32_t)(r * BM * 8 + q * 16), a0 + (r0 + r) * np + 2 * q);
            }
        }
#pragma unroll
        for (int u = 0; u < CB / NT; ++u) {
            const int c = tid + NT * u;
            const int r = c >> 6, q = c & 63;
            cp_async16(sb + (uint32_t)(r * 1024 + q * 16), b0 + (r0 + r) * np + 2 * q);
        }
    };
#endif
    double acc[RM][8];
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;
#if ELL_DENSE_TMA
    if (warp == 0) {
#pragma unroll
        for (int st = 0; st < kDenseStages - 1; ++st)
            if (st < nact) load_stage(st, list[st]);
    }
    for (int t = 0; t < nact; ++t) {
        __syncthreads();  // every thread is done with stage t - 1: its slot takes stage t + S - 1
        {
            const int tn = t + kDenseStages - 1;
            if (warp == 0 && tn < nact) load_stage(tn % kDenseStages, list[tn]);
        }
        dmbar_wait(bar0 + 8u * (uint32_t)(t % kDenseStages), (uint32_t)((t / kDenseStages) & 1));
#else
#pragma unroll
    for (int st = 0; st < kDenseStages - 1; ++st) {
        if (st < nact) load_stage(st, list[st]);
        cp_async_commit();
    }
    for (int t = 0; t < nact; ++t) {
        cp_async_wait<kDenseStages - 2>();
        __syncthreads();  // stage t landed for every thread; stage t - 1 is free
        {
            const int tn = t + kDenseStages - 1;
            if (tn < nact) load_stage(tn % kDenseStages, list[tn]);
            cp_async_commit();
        }
#endif
        const uint32_t sa = sbase + (uint32_t)((t % kDenseStages) * SB), sb = sa + (uint32_t)(kDenseK * BM * 8);
#pragma unroll
        for (int k = 0; k < kDenseK; ++k) {
            double a[RM], b[8];
#pragma unroll
            for (int g = 0; g < RM / 2; ++g)
                lds128(sa + (uint32_t)((k * BM + 2 * TY * g + 2 * ty) * 8), a[2 * g], a[2 * g + 1]);
#pragma unroll
            for (int h = 0; h < 4; ++h) lds128(sb + (uint32_t)(k * 1024 + (32 * h + 2 * tx) * 8), b[2 * h], b[2 * h + 1]);
#pragma unroll
            for (int r = 0; r < RM; ++r)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[r][c] = __fma_rn(a[r], b[c], acc[r][c]);
        }
    }
#if !ELL_DENSE_TMA
    cp_async_wait<0>();
#endif
    // tile (bi, bj), and for SYM off the diagonal its transpose at (bj, bi). A tile with no occupied k
    // block is exactly zero: it is not stored, its tw flag tells the epilogue to read zeros instead
    if (tid == 0) {
        tw[(size_t)bi * T + bj] = nact > 0;
        if (SYM && bi != bj) tw[(size_t)bj * T + bi] = nact > 0;
    }
    if (nact == 0) return;
#pragma unroll
    for (int g = 0; g < RM / 2; ++g)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            double* row = S + (size_t)(bi * BM + 2 * TY * g + 2 * ty + r) * np + bj * kDenseTile;
#pragma unroll
            for (int h = 0; h < 4; ++h) stg128(row + 32 * h + 2 * tx, acc[2 * g + r][2 * h], acc[2 * g + r][2 * h + 1]);
        }
    if (SYM && bi != bj) {
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                double* row = S + (size_t)(bj * kDenseTile + 32 * h + 2 * tx + c) * np + bi * BM;
#pragma unroll
                for (int g = 0; g < RM / 2; ++g)
                    stg128(row + 2 * TY * g + 2 * ty, acc[2 * g][2 * h + c], acc[2 * g + 1][2 * h + c]);
            }
    }
    if (exec && tid == 0 && nact)
        atomicAdd(exec, (unsigned long long)nact * kDenseK * BM * kDenseTile);
}

template <int BM, int TY, bool SYM>
cudaError_t launch_gemm_t(unsigned grid, const double* At, const double* B, int np, const unsigned long long* fa,
                          const unsigned long long* fb, double* S, unsigned char* tw, unsigned long long* exec,
                          int bi0, cudaStream_t s) {
    static int attr[64];  // dynamic shared memory opted in so far (per instantiation and device)
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    const size_t smem = (size_t)kDenseStages * stage_bytes<BM>() + sizeof(int) * (size_t)(np / kDenseK);
    if (smem > 48 * 1024 && attr[dev] < (int)smem) {
        cudaError_t e = cudaFuncSetAttribute(dense_gemm_kernel<BM, TY, SYM>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e) return e;
        attr[dev] = (int)smem;
    }
    dense_gemm_kernel<BM, TY, SYM><<<grid, 16 * TY, smem, s>>>(At, B, np, fa, fb, S, tw, exec, bi0);
    return cudaGetLastError();
}

int dense_tile_rows(int np, int64_t rows, bool sym, int num_sms) {
    const int64_t T = np / kDenseTile, R = rows / kDenseTile;
    const int64_t tiles = sym ? T * (T + 1) / 2 : R * T;
    // 128-row tiles while they fill most of the SMs; below that 16-row tiles (8x the CTAs)
    return tiles >= (num_sms * 4) / 5 ? 128 : 16;
}

// ----------------------------------------------------------------- FP64 MMA variant (DMMA)
//
// The same tiles, k blocks and pipeline, with the 8 x 8 x 4 FP64 MMA (mma.sync.m8n8k4.f64) doing the
// multiply-adds: one warp instruction = 256 of them, where the FMA kernel issues 8 (FP64 pipe 74 % busy,
// bound by issue). Its use rests on reading R23: on sm_100a the MMA computes each output as the
// ascending fma chain d = fma(a3, b3, fma(a2, b2, fma(a1, b1, fma(a0, b0, c)))) -- checked bit for
// bit on 4.5e8 outputs including planted cancellations (tools/dmma_order.cu, profiles/r02_dmma_order.log)
// and again on every device before first use (dense_mma_selfcheck); chained over the k blocks in
// ascending order it is the sparse kernels' chain exactly.
//
// 8 warps as 2 x 4, each a 64 x 32 sub-tile = 8 x 4 MMA tiles (64 accumulators per lane). Stage rows
// are padded to 132 doubles: the fragments (A: lane l reads row k0 + l % 4, column m0 + l / 4) then
// hit 16 distinct bank pairs per half-warp.
constexpr int kMmaPad = 132;  // padded stage row (doubles)
#ifndef ELL_MMA_KPS
#define ELL_MMA_KPS 3  // k blocks per pipeline stage (one barrier per stage; 3 x 2 stages measured best)
#endif
#ifndef ELL_MMA_STAGES
#define ELL_MMA_STAGES 2
#endif
constexpr int kMmaKps = ELL_MMA_KPS, kMmaStages = ELL_MMA_STAGES;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int BM, bool SYM>
__global__ void __launch_bounds__(BM == 128 ? 256 : 128, BM == 128 ? 1 : 4)
    dense_mma_kernel(const double* __restrict__ At, const double* __restrict__ B, int np,
                     const unsigned long long* __restrict__ Fa, const unsigned long long* __restrict__ Fb,
                     double* __restrict__ S, unsigned char* __restrict__ tw, unsigned long long* exec, int bi0) {
    static_assert(!SYM || BM == kDenseTile, "symmetric tiles are square");
    // BM = 128: 8 warps as 2 x 4 of 64 x 32; BM = 16: 4 warps of 16 x 32 (small N: 8x the CTAs)
    constexpr int NW = BM == 128 ? 8 : 4, WM = BM == 128 ? 2 : 1, MB = BM / WM / 8;
    constexpr int PA = BM + 4;  // padded A^T stage row: the fragments hit 16 bank pairs per half-warp
    constexpr int SA = kMmaKps * kDenseK * PA, SB = kMmaKps * kDenseK * kMmaPad;  // doubles per stage part
    constexpr int STG = (SA + SB) * 8;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int wcnt[NW];
    __shared__ __align__(8) unsigned long long fullbar[kMmaStages];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int T = np / kDenseTile;
    int bi, bj;
    if (SYM) {
        int t = blockIdx.x;
        bi = 0;
        while (t >= T - bi) { t -= T - bi; ++bi; }
        bj = bi + t;
    } else {
        bi = bi0 + (int)(blockIdx.x / T);
        bj = blockIdx.x % T;
    }
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    int* list = reinterpret_cast<int*>(smem + kMmaStages * STG);
    const int bf = bi * BM / kDenseTile;  // the 128-row flag block of this tile's rows
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(fullbar);
    if (tid == 0) {
#pragma unroll
        for (int st = 0; st < kMmaStages; ++st) dmbar_init(bar0 + 8u * st, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int kbw = dense_kbw(np);
    int nact = 0;
    for (int w0 = 0; w0 < kbw; w0 += 32 * NW) {
        const int w = w0 + tid;
        const unsigned long long m = w < kbw ? Fa[(size_t)bf * kbw + w] & Fb[(size_t)bj * kbw + w] : 0ull;
        const int cnt = __popcll(m);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wcnt[warp] = incl;
        __syncthreads();
        int off = nact, tot = 0;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            off += q < warp ? wcnt[q] : 0;
            tot += wcnt[q];
        }
        off += incl - cnt;
        for (unsigned long long r = m; r; r &= r - 1) list[off++] = 64 * w + __ffsll((long long)r) - 1;
        __syncthreads();
        nact += tot;
    }
    const double* a0 = At + (size_t)bi * BM;
    const double* b0 = B + (size_t)bj * kDenseTile;
    const int nst = (nact + kMmaKps - 1) / kMmaKps;  // stages: kMmaKps listed k blocks each
    auto load_stage = [&](int slot, int st) {  // warp 0: one bulk copy per k row of A^T and of B
        const uint32_t sa = sbase + (uint32_t)(slot * STG), sb = sa + (uint32_t)(SA * 8);
        const uint32_t bar = bar0 + 8u * (uint32_t)slot;
        const int ne = min(kMmaKps, nact - st * kMmaKps);
        if (lane == 0) dmbar_expect(bar, (uint32_t)ne * kDenseK * (BM + kDenseTile) * 8u);
        __syncwarp();
        const int r = lane & 15;
        for (int j = 0; j < ne; ++j) {
            const size_t r0 = (size_t)list[st * kMmaKps + j] * kDenseK;
            if (lane < 16) bulk_g2s(sa + (uint32_t)((j * kDenseK + r) * PA * 8), a0 + (r0 + r) * np, (uint32_t)(BM * 8), bar);
            else bulk_g2s(sb + (uint32_t)((j * kDenseK + r) * kMmaPad * 8), b0 + (r0 + r) * np, 1024u, bar);
        }
    };
    const int wm = warp >> 2, wn = warp & 3;  // (8 MB)-row x 32-column sub-tile
    const int fr = lane & 3, fc = lane >> 2;  // fragment: k offset, row / column offset
    double acc[MB][4][2];
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) acc[mb][nb][0] = acc[mb][nb][1] = 0.0;
    if (warp == 0) {
#pragma unroll
        for (int st = 0; st < kMmaStages - 1; ++st)
            if (st < nst) load_stage(st, st);
    }
    for (int t = 0; t < nst; ++t) {
        __syncthreads();  // every warp is done with stage t - 1: its slot takes stage t + S - 1
        {
            const int tn = t + kMmaStages - 1;
            if (warp == 0 && tn < nst) load_stage(tn % kMmaStages, tn);
        }
        dmbar_wait(bar0 + 8u * (uint32_t)(t % kMmaStages), (uint32_t)((t / kMmaStages) & 1));
        const double* sa = reinterpret_cast<const double*>(smem + (t % kMmaStages) * STG);
        const double* sb = sa + SA;
        const int krows = min(kMmaKps, nact - t * kMmaKps) * kDenseK;
#pragma unroll 4
        for (int k4 = 0; k4 < krows; k4 += 4) {  // k ascending: 4 per MMA, the MMAs in order
            double a[MB], b[4];
            const double* ak = sa + (k4 + fr) * PA + wm * (8 * MB) + fc;
            const double* bk = sb + (k4 + fr) * kMmaPad + wn * 32 + fc;
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) a[mb] = ak[8 * mb];
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) b[nb] = bk[8 * nb];
#pragma unroll
            for (int mb = 0; mb < MB; ++mb)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb][0], acc[mb][nb][1], a[mb], b[nb]);
        }
    }
    if (tid == 0) {
        tw[(size_t)bi * T + bj] = nact > 0;
        if (SYM && bi != bj) tw[(size_t)bj * T + bi] = nact > 0;
    }
    if (nact == 0) return;
    // accumulator (mb, nb, h): row wm 8 MB + 8 mb + lane / 4, column wn 32 + 8 nb + 2 (lane % 4) + h
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) {
        double* row = S + (size_t)(bi * BM + wm * (8 * MB) + 8 * mb + fc) * np + bj * kDenseTile + wn * 32 + 2 * fr;
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) stg128(row + 8 * nb, acc[mb][nb][0], acc[mb][nb][1]);
    }
    if (SYM && bi != bj) {
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double* col = S + (size_t)(bj * kDenseTile + wn * 32 + 8 * nb + 2 * fr + h) * np + bi * BM +
                              wm * (8 * MB) + fc;
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) col[8 * mb] = acc[mb][nb][h];
            }
    }
    if (exec && tid == 0)
        atomicAdd(exec, (unsigned long long)nact * kDenseK * BM * kDenseTile);
}

// R23 on this device: MMA outputs vs the ascending fma chain on random, mixed-magnitude and planted-
// cancellation inputs (the cases where other orders differ); bad[0] counts mismatches.
__global__ void dense_mma_selfcheck_kernel(unsigned long long* bad) {
    const int lane = threadIdx.x & 31;
    uint64_t sd = 0x5eed0000ull + 7919ull * (blockIdx.x * 32 + lane);
    auto rnd = [&](int mode) {
        sd += 0x9e3779b97f4a7c15ull;
        uint64_t z = sd;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        const double u = (double)(z >> 11) * 0x1p-53 * 2.0 - 1.0;
        return mode ? ldexp(u, (int)((z >> 3) % 60) - 30) : u;
    };
    __shared__ double A[8][4], Bm[4][8], C[8][8];
    unsigned long long nb = 0;
    for (int t = 0; t < 64; ++t) {
        const int mode = t % 3;
        A[lane >> 2][lane & 3] = rnd(mode);
        Bm[lane >> 3][lane & 7] = rnd(mode);
        for (int q = lane; q < 64; q += 32) C[q >> 3][q & 7] = rnd(mode);
        __syncwarp();
        if (mode == 2) {  // c = -(the products' sum), perturbed: the chain's rounding decides everything
            for (int q = lane; q < 64; q += 32) {
                const int i = q >> 3, j = q & 7;
                double sum = 0.0;
                for (int k = 0; k < 4; ++k) sum = __fma_rn(A[i][k], Bm[k][j], sum);
                C[i][j] = -sum * (1.0 + ldexp((double)(q % 7 - 3), -50));
            }
            __syncwarp();
        }
        double d0 = C[lane >> 2][2 * (lane & 3)], d1 = C[lane >> 2][2 * (lane & 3) + 1];
        dmma(d0, d1, A[lane >> 2][lane & 3], Bm[lane & 3][lane >> 2]);
        for (int h = 0; h < 2; ++h) {
            const int i = lane >> 2, j = 2 * (lane & 3) + h;
            double ch = C[i][j];
            for (int k = 0; k < 4; ++k) ch = __fma_rn(A[i][k], Bm[k][j], ch);
            if (__double_as_longlong(h ? d1 : d0) != __double_as_longlong(ch)) ++nb;
        }
        __syncwarp();
    }
    if (nb) atomicAdd(bad, nb);
}

// 1: the MMA variant may run on this device (R23 holds here), 0: it may not. Checked once per device.
int dense_mma_ok(cudaStream_t s) {
    static std::mutex mu;  // contexts of different host threads may ask at once
    static int checked[64];
    static int verdict[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
    std::lock_guard<std::mutex> lock(mu);
    if (checked[dev]) return verdict[dev];
    unsigned long long* bad = nullptr;
    unsigned long long h = 1;
    if (cudaMallocAsync((void**)&bad, 8, s) == cudaSuccess && cudaMemsetAsync(bad, 0, 8, s) == cudaSuccess) {
        dense_mma_selfcheck_kernel<<<148, 32, 0, s>>>(bad);
        if (cudaMemcpyAsync(&h, bad, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
            h = 1;
        cudaFreeAsync(bad, s);
    }
    cudaGetLastError();
    checked[dev] = 1;
    verdict[dev] = h == 0;
    return verdict[dev];
}

template <int BM, bool SYM>
cudaError_t launch_mma_t(unsigned grid, const double* At, const double* B, int np, const unsigned long long* fa,
                         const unsigned long long* fb, double* S, unsigned char* tw, unsigned long long* exec, int bi0,
                         cudaStream_t s) {
    static int attr[64];  // per device
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    const size_t stage = (size_t)kMmaKps * kDenseK * ((BM + 4) + kMmaPad) * 8;
    const size_t smem = (size_t)kMmaStages * stage + sizeof(int) * (size_t)(np / kDenseK);
    if (smem > 48 * 1024 && attr[dev] < (int)smem) {
        cudaError_t e = cudaFuncSetAttribute(dense_mma_kernel<BM, SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e) return e;
        attr[dev] = (int)smem;
    }
    dense_mma_kernel<BM, SYM><<<grid, BM == 128 ? 256 : 128, smem, s>>>(At, B, np, fa, fb, S, tw, exec, bi0);
    return cudaGetLastError();
}

cudaError_t launch_dense_gemm(const double* At, const double* B, int np, bool sym, const unsigned long long* fa,
                              const unsigned long long* fb, double* S, unsigned char* tw, unsigned long long* exec,
                              int64_t row0, int64_t row1, int bm, bool mma, cudaStream_t s) {
    if (np <= 0 || np % kDenseTile || row0 % kDenseTile || (row1 - row0) % kDenseTile || row1 <= row0)
        return cudaErrorInvalidValue;
    const int T = np / kDenseTile;
    const int R = (int)((row1 - row0) / kDenseTile);
    if (sym && (row0 != 0 || row1 != np)) return cudaErrorInvalidValue;  // symmetric tiles: all rows
    if (bm == 128 && mma) {
        if (sym) return launch_mma_t<128, true>((unsigned)(T * (T + 1) / 2), At, B, np, fa, fb, S, tw, exec, 0, s);
        return launch_mma_t<128, false>((unsigned)(R * T), At, B, np, fa, fb, S, tw, exec, (int)(row0 / 128), s);
    }
    // (16-row tiles stay on FP64 FMAs: the MMA variant measured slower there -- 0.36 vs 0.25 ms at
    // N = 1024 -- with two fragments of A per four of B and 117 KB of stages per CTA)
    if (bm == 128) {
        if (sym) return launch_gemm_t<128, ELL_DENSE_TY, true>((unsigned)(T * (T + 1) / 2), At, B, np, fa, fb, S, tw,
                                                               exec, 0, s);
        return launch_gemm_t<128, ELL_DENSE_TY, false>((unsigned)(R * T), At, B, np, fa, fb, S, tw, exec,
                                                       (int)(row0 / 128), s);
    }
    return launch_gemm_t<16, 8, false>((unsigned)(8 * R * T), At, B, np, fa, fb, S, tw, exec, (int)(row0 / 16), s);
}

// Zero the 128 x 16 blocks of D that fa flags (D holds nonzeros only there): the dense array returns
// to all-zero at the cost of the previous iterate's band instead of N^2. A warp per block.
__global__ void __launch_bounds__(256) dense_clear_kernel(double* __restrict__ D, int np,
                                                          const unsigned char* __restrict__ fa) {
    const int lane = threadIdx.x & 31;
    const int KB = np / kDenseK;
    const int64_t nblk = (int64_t)(np / kDenseTile) * KB;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nblk; b += nw) {
        if (!fa[b]) continue;
        const int64_t bi = b / KB, kb = b % KB;
        double* base = D + (size_t)bi * kDenseTile * np + (size_t)kb * kDenseK;
        // 128 rows x 16 doubles: 1024 16-byte stores, 32 per lane (8 lanes per row)
#pragma unroll 4
        for (int q = lane; q < 1024; q += 32) stg128(base + (size_t)(q >> 3) * np + 2 * (q & 7), 0.0, 0.0);
    }
}

cudaError_t launch_dense_clear(double* D, int np, const unsigned char* fa, int num_sms, cudaStream_t s) {
    dense_clear_kernel<<<(unsigned)(num_sms * 8), 256, 0, s>>>(D, np, fa);
    return cudaGetLastError();
}

// ------------------------------------------------------------------- dense work of X X

// F[t][w] bit b = some entry of x in rows [128 t, 128 t + 128) and columns [16 (64 w + b), + 16):
// the left operand's 128 x 16 occupancy as bitsets (for a symmetric x also the right operand's,
// transposed). A warp per row; each lane ORs the bits of a contiguous piece of the (ascending) row
// in a register and flushes one atomicOr per 64-bit word it touches.
__global__ void __launch_bounds__(256) occupancy_kernel(KMat x, int64_t n, int kbw, unsigned long long* __restrict__ F) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
        const int nnz = x.nnz[i];
        const int32_t* c = x.col + (size_t)i * x.w;
        unsigned long long* row = F + (size_t)(i / kDenseTile) * kbw;
        const int per = (nnz + 31) / 32;
        const int q0 = lane * per, q1 = min(nnz, q0 + per);
        int word = -1;
        unsigned long long bits = 0ull;
        for (int q = q0; q < q1; ++q) {
            const int kb = c[q] / kDenseK;
            if ((kb >> 6) != word) {
                if (bits) atomicOr(row + word, bits);
                word = kb >> 6;
                bits = 0ull;
            }
            bits |= 1ull << (kb & 63);
        }
        if (bits) atomicOr(row + word, bits);
    }
}

cudaError_t launch_occupancy(KMat x, int64_t n, int np, unsigned long long* F, int num_sms, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int64_t blocks = (n + 7) / 8;
    occupancy_kernel<<<(unsigned)(blocks < (int64_t)num_sms * 16 ? blocks : (int64_t)num_sms * 16), 256, 0, s>>>(
        x, n, np / kDenseK / 64 + ((np / kDenseK) % 64 ? 1 : 0), F);
    return cudaGetLastError();
}

// out += the occupied k blocks of every symmetric tile bi <= bj: popc(F[bi] & F[bj]) (x symmetric:
// row block bj's occupancy is column tile bj's) -- the symmetric GEMM's work, exactly, in k blocks.
__global__ void __launch_bounds__(256) dense_work_kernel(const unsigned long long* __restrict__ F, int T, int kbw,
                                                         unsigned long long* out) {
    const int lane = threadIdx.x & 31;
    const int64_t tiles = (int64_t)T * T;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    unsigned long long mine = 0ull;
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < tiles; t += nw) {
        const int bi = (int)(t / T), bj = (int)(t % T);
        if (bj < bi) continue;
        const unsigned long long* a = F + (size_t)bi * kbw;
        const unsigned long long* b = F + (size_t)bj * kbw;
        for (int w = lane; w < kbw; w += 32) mine += (unsigned long long)__popcll(a[w] & b[w]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(FULL, mine, o);
    if (lane == 0 && mine) atomicAdd(out, mine);
}

cudaError_t launch_dense_work(const unsigned long long* F, int np, unsigned long long* out, int num_sms,
                              cudaStream_t s) {
    const int T = np / kDenseTile;
    const int kbw = np / kDenseK / 64 + ((np / kDenseK) % 64 ? 1 : 0);
    dense_work_kernel<<<(unsigned)(num_sms * 4), 256, 0, s>>>(F, T, kbw, out);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------- emission

// MODE as the row kernels: 0 no Old operand; 1 Old operand; 2 Old operand and the norm
// ||S - Old||^2. p.old_mode (runtime): 1 Old enters the value (beta old), 2 only the union and the
// norm (SP2 SQUARE). The Old row is read from its dense copy dOld: a column absent from Old reads
// x = +0, and with x = +0 the row kernels' formula for a column OUTSIDE Old (c = alpha s, norm term
// s^2) and the one for a column INSIDE Old (c = fma(alpha, s, beta x or +0), norm term (s - x)^2)
// agree on everything kept or summed (they can differ only in the sign of a zero c, which is
// dropped) -- so no merge of the Old row is needed. A warp per row, 128 columns (four 32-column
// chunks, column j on lane j mod 32) per iteration with the loads of all four issued first.
template <int MODE>
__global__ void __launch_bounds__(256) dense_emit_kernel(const double* __restrict__ S, int np, const RowOpParams p,
                                                         const double* __restrict__ dA,
                                                         const double* __restrict__ dOld,
                                                         const unsigned char* __restrict__ tw, int tw_rows,
                                                         const unsigned long long* __restrict__ fold) {
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int n = (int)p.ncols;
    const int cw = p.C.w;
    const double tau = p.tau;
    // (alpha, beta, old_mode) from device memory in the device-resident SP2 loop (p.dyn)
    const double alpha = p.dyn ? p.dyn[0] : p.alpha, beta = p.dyn ? p.dyn[1] : p.beta;
    const int old_mode = p.dyn ? (int)p.dyn[2] : p.old_mode;
    const bool a1 = alpha == 1.0, o1 = old_mode == 1;
    int32_t my_max = 0, my_ovf = 0;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = p.row_begin + (int64_t)blockIdx.x * (blockDim.x >> 5) + wi; i < p.row_end; i += nw) {
        const double* srow = S + (size_t)i * np;
        const double* xrow = MODE != 0 ? dOld + (size_t)i * np : nullptr;
        double* cv = p.C.val + (size_t)i * cw;
        int32_t* cc = p.C.col + (size_t)i * cw;
        int kept = 0;
        double ds = 0.0, dc = 0.0, nrm = 0.0;
        const int T = np / kDenseTile;
        const unsigned char* twr = tw + (size_t)(i / tw_rows) * T;
        const unsigned long long* fr = MODE != 0 ? fold + (size_t)(i / kDenseTile) * dense_kbw(np) : nullptr;
        for (int j0 = 0; j0 < n; j0 += 128) {
            // the tile of S was not stored (exactly zero) / the Old row has no entry in these 128
            // columns (its 8 occupancy flags): read zeros; both -> nothing to emit or sum here
            const bool s_ok = twr[j0 >> 7] != 0;
            const bool x_ok = MODE != 0 && ((fr[j0 >> 10] >> ((j0 >> 4) & 63)) & 0xffull) != 0ull;
            if (!s_ok && !x_ok) continue;
            double sv[4], xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = j0 + 32 * u + lane;
                sv[u] = (s_ok && j < n) ? __ldcs(srow + j) : 0.0;  // S is read once: streaming
                xv[u] = (x_ok && j < n) ? xrow[j] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = j0 + 32 * u + lane;
                const double s = sv[u];
                double c;
                if (MODE != 0) {
                    c = __fma_rn(alpha, s, o1 ? __dmul_rn(beta, xv[u]) : 0.0);
                    if (MODE == 2) {
                        const double df = __dsub_rn(s, xv[u]);
                        nrm = __fma_rn(df, df, nrm);
                    }
                } else {
                    c = a1 ? s : __dmul_rn(alpha, s);
                }
                const bool keep = j < n && fabs(c) > tau;
                const unsigned km = __ballot_sync(FULL, keep);
                const int pos = kept + __popc(km & lt);
                if (keep && pos < cw) {
                    cv[pos] = c;
                    cc[pos] = j;
                }
                if ((int64_t)j == i) {
                    ds = s;
                    dc = keep ? c : 0.0;
                }
                kept += __popc(km);
            }
        }
        // the diagonal values live in lane i mod 32
        const int owner = (int)(i & 31);
        ds = __shfl_sync(FULL, ds, owner);
        dc = __shfl_sync(FULL, dc, owner);
        if (MODE == 2) nrm = warp_sum(nrm);
        if (lane == 0) {
            p.C.nnz[i] = kept < cw ? kept : cw;
            if (p.diag_s) p.diag_s[i] = ds;
            if (p.diag_c) p.diag_c[i] = dc;
            if (p.diag_a) p.diag_a[i] = dA[(size_t)i * np + i];
            if (MODE == 2) p.normsq[i] = nrm;
        }
        my_max = max(my_max, kept);
        if (kept > cw) ++my_ovf;
    }
    if (lane == 0) {
        if (my_ovf) atomicAdd(p.status + 0, my_ovf);
        if (my_max) atomicMax(p.status + 1, my_max);
    }
}

cudaError_t launch_dense_emit(const double* S, int np, const RowOpParams& p, const double* dA, const double* dOld,
                              const unsigned char* tw, int tw_rows, const unsigned long long* fold, int num_sms,
                              cudaStream_t s) {
    const int64_t rows = p.row_end - p.row_begin;
    if (rows <= 0) return cudaSuccess;
    if (p.old_mode != 0 && (!dOld || !fold)) return cudaErrorInvalidValue;
    int64_t blocks = (rows + 7) / 8;
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    const int mode = p.old_mode == 0 ? 0 : (p.normsq ? 2 : 1);  // as the row kernels' MODE
    if (mode == 0) dense_emit_kernel<0><<<(unsigned)blocks, 256, 0, s>>>(S, np, p, dA, dOld, tw, tw_rows, fold);
    else if (mode == 1) dense_emit_kernel<1><<<(unsigned)blocks, 256, 0, s>>>(S, np, p, dA, dOld, tw, tw_rows, fold);
    else dense_emit_kernel<2><<<(unsigned)blocks, 256, 0, s>>>(S, np, p, dA, dOld, tw, tw_rows, fold);
    return cudaGetLastError();
}

}  // namespace ell
