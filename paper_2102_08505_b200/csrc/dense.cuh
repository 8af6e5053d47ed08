// dense.cuh — the dense-regime step of libellpack: when an SP2 iterate has filled in (cfg3 reaches
// width 12096 of N = 12288 by iteration 45, profiles/r01_sp2_full_cfg3.json), the sparse row kernels
// pay a shared-memory read-modify-write per product for work a dense FP64 GEMM does from registers.
// The product is the same bit for bit: every output entry is still ONE fma chain over k ascending,
// and the chain's extra terms are exact zeros (fma(a, +-0, s) == s for s != -0; an accumulator that
// starts at +0 never becomes -0 under round-to-nearest), so the values, the pattern (|c| > tau drops
// every structural zero) and the traces equal the oracle's (readings R3, R5, R12).
#pragma once
#include "internal.cuh"

namespace ell {

constexpr int kDenseTile = 128;  // rows and columns of S per CTA
constexpr int kDenseK = 16;      // k rows per pipeline stage

// 64-bit words of one k-block bitset (np / 16 bits)
__host__ __device__ inline int dense_kbw(int np) { return (np / kDenseK + 63) / 64; }

// D (np x np doubles, zeroed by the caller) <- the stored entries of rows [i0, i1) of a:
// D[i][j] = a_ij, or D[j][i] = a_ij with transpose. Occupancy flags (nullable, zeroed by the caller):
// fa[(i / 128) * (np / 16) + j / 16] = 1 (a as the left operand: (m-block, k-block)),
// fb[(i / 16) * (np / 128) + j / 128] = 1 (a as the right operand: (k-block, n-block)).
cudaError_t launch_densify(KMat a, int64_t i0, int64_t i1, int np, bool transpose, double* D, unsigned char* fa,
                           unsigned char* fb, cudaStream_t s);

// S = A B over the k blocks whose flags are both set (nullable flags: every block), k ascending:
// At is A transposed (At[k][m] = a_mk); sym: A B is symmetric (A = B = B^T), only tiles bi <= bj are
// computed and each is also stored transposed. exec (nullable) += FMAs executed.
// fa, fb byte flags (as launch_densify's) -> bitsets Fa[T][kbw] (k blocks of each 128-row block) and
// Fb[T][kbw] (k blocks of each 128-column tile), kbw = dense_kbw(np).
cudaError_t launch_pack_flags(const unsigned char* fa, const unsigned char* fb, int np, unsigned long long* Fa,
                              unsigned long long* Fb, int num_sms, cudaStream_t s);

// Rows [row0, row1) of S (multiples of 128; sym: all rows, tiles bi <= bj mirrored) in tiles of
// bm = dense_tile_rows(np, rows, sym, SMs) rows x 128 columns: 128 while they fill most SMs, else 16
// (small N). A tile with no occupied k block is not stored: tw[(row / bm) * (np / 128) + column / 128]
// = 0 for it, 1 for a stored tile (every entry written by the launch).
int dense_tile_rows(int np, int64_t rows, bool sym, int num_sms);
// mma: 128-row tiles on the FP64 MMA (mma.sync m8n8k4) instead of FP64 FMAs (reading R23; callers
// pass dense_mma_ok()).
cudaError_t launch_dense_gemm(const double* At, const double* B, int np, bool sym, const unsigned long long* Fa,
                              const unsigned long long* Fb, double* S, unsigned char* tw, unsigned long long* exec,
                              int64_t row0, int64_t row1, int bm, bool mma, cudaStream_t s);
// 1 when the FP64 MMA computes the ascending fma chain bit for bit on this device (checked once per
// device on adversarial inputs; reading R23), else 0.
int dense_mma_ok(cudaStream_t s);

// D <- 0 given that D is zero outside the 128 x 16 blocks fa flags (the previous densify's).
cudaError_t launch_dense_clear(double* D, int np, const unsigned char* fa, int num_sms, cudaStream_t s);

// Rows [p.row_begin, p.row_end) of C from the dense S (row stride np): combine with Old (p.old_mode),
// drop, compact, write, diagonals, norm and status as the row kernels do (RowOpParams).
// dA (row stride np; read only with p.diag_a): a dense copy of A whose diagonal is the stored a_ii;
// dOld (row stride np; required when p.old_mode != 0): the dense copy of Old, zero outside the
// 128 x 16 blocks its bitsets fold (Fa of launch_pack_flags) mark. S is read only where tw (tile rows
// tw_rows) says the GEMM stored it.
cudaError_t launch_dense_emit(const double* S, int np, const RowOpParams& p, const double* dA, const double* dOld,
                              const unsigned char* tw, int tw_rows, const unsigned long long* fold, int num_sms,
                              cudaStream_t s);

// The symmetric GEMM's exact work for a symmetric x (the next step's operand), without densifying
// it: occupancy bitsets F ([np/128][ceil(np/16/64)] words, zeroed by the caller), then
// out += the number of (tile bi <= bj, k block) pairs occupied on both sides.
cudaError_t launch_occupancy(KMat x, int64_t n, int np, unsigned long long* F, int num_sms, cudaStream_t s);
cudaError_t launch_dense_work(const unsigned long long* F, int np, unsigned long long* out, int num_sms,
                              cudaStream_t s);

size_t dense_gemm_smem(int np);

}  // namespace ell
