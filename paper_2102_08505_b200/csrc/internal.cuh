// internal.cuh — device-side types and launcher prototypes of libellpack
// (the B200 hot path of arXiv 2102.08505; public ABI in include/ellpack.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ell {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kTraceBlock = 256;  // canonical-sum block

// Read-only view of an ELLPACK matrix (D1: row-major val/col [n][w], nnz [n]).
struct KMat {
    const double* val;
    const int32_t* col;
    const int32_t* nnz;
    int32_t w;
};

// Writable view.
struct KOut {
    double* val;
    int32_t* col;
    int32_t* nnz;
    int32_t w;
};

// One launch of the fused row kernel computes, for rows i in [row_begin, row_end):
//   s_j   = fma chain over k ascending in A_i of a_ik * b_kj
//   c_j   = fma(alpha, s_j, old_mode == 1 ? beta*old_ij : +0)        (§8a-a3)
//   keep iff |c_j| > tau, write ascending into C row i (<= C.w)       (§8a-a3)
// over the union of the product pattern and (old_mode != 0 ? Old_i : {}).
// old_mode: 0 = no Old operand; 1 = Old enters the value (beta*old);
//           2 = Old enters only the union and the norm (SP2 SQUARE step).
struct RowOpParams {
    KMat A, B, Old;
    KOut C;
    int64_t row_begin, row_end;
    double alpha, beta, tau;
    int32_t old_mode;
    int32_t stash_a;    // C aliases A -> stash A row when the row needs > 1 pass
    int32_t stash_old;  // C aliases Old -> stash Old row when the row needs > 1 pass
    int32_t S;          // dense-window capacity (doubles) per warp
    int32_t fast;       // 1: ring fast path (S = ring slots >= 2 hB + 33, B rows <= 256 entries)
    int32_t hB;         // max half-bandwidth of B (probe)
    int64_t ncols;      // matrix dimension N (columns >= N never exist)
    // fast path: bank-balanced copy of B (balance_kernel): [N][bt_w] values / columns
    // (column -1 = padding) and NB(k) = ceil(nnz_B(k) / 16) used half-instruction bins
    const unsigned char* bt;  // row k: int32 slot8[bt_w] (8 (j mod S), padding: 8 (S + r)), f64 val[bt_w]
    const int32_t* bt_nbin;
    int32_t bt_w;             // 64 G
    const int32_t* bp;        // general path: breakpoints [N][bp_np] of B at multiples of S
    int32_t bp_np;
    int32_t ablate;           // timing experiments only (ELLPACK_OPT_ABLATE bit mask, include/ellpack.h)
    // optional per-row outputs, indexed by global row (nullable)
    double* diag_a;   // stored a_ii
    double* diag_s;   // pre-combine s_ii  (tr(X^2) pre-drop, R5)
    double* diag_c;   // stored output c_ii (tr of the new iterate)
    double* normsq;   // sum over the union of (s_ij - old_ij)^2   (old_mode != 0)
    int32_t* status;  // [0] overflow rows, [1] max kept count
    unsigned long long* row_ticket;  // fast kernel: dynamic row counter (zeroed before each launch)
    int32_t row_chunk;               // fast kernel: consecutive rows per ticket (4; 1 for small launches)
    int32_t upper;                   // general kernel: columns j >= i only (symmetric SP2 step, f4 ii)
    KOut C_upper;                    // upper-triangle output when the general path takes `upper`
    const double* dyn;                  // general kernel (nullable): (alpha, beta, old_mode) read from
                                        // device memory (device-resident SP2 loop, f3)
    unsigned long long* exec_products;  // general kernel (nullable): += products it executes (B entries
                                        // accumulated; the symmetric step's count, about P / 2)
    // per-warp global scratch: in-place rows are copied aside (stash) before they are rewritten
    double* st_val;
    int32_t* st_col;
    int64_t st_stride;
};

struct LaunchCfg {
    int S;               // window doubles per warp
    int warps_per_cta;
    int grid;
    size_t smem;
    int R;               // fast path: 64-entry B groups per step (1..4)
    int bps;             // resident CTAs per SM at this configuration
};

// spgemm.cu
// groups = ceil(max nnz_B / 64): the fast path processes every B row as `groups` 64-entry groups
cudaError_t plan_row_op(const RowOpParams& p, int S, int groups, int warps_opt, int num_sms, LaunchCfg* cfg);
cudaError_t launch_row_op(const RowOpParams& p, const LaunchCfg& cfg, cudaStream_t s);
size_t row_op_warp_smem(int S, bool has_old, bool fast);
// bank-balanced copy of B for the fast path (wt = 64 G >= 16 ceil(nnz/16) for every row)
// (S: the ring size of the launch that consumes it; slots are precomputed as 8 (j mod S))
// (rows k0 <= k < k1 only: the B rows the launch's A rows reference)
cudaError_t launch_balance(KMat b, int64_t k0, int64_t k1, int wt, int S, unsigned char* bt, int32_t* bt_nbin,
                           int num_sms, cudaStream_t s);
// out[0..2] = max half-bandwidth of a (rows r0..r1), b (rows b0..b1), c (rows r0..r1); out[3] = max nnz
// of b (rows b0..b1); out[4] = max chunk-parity half of those B rows; A's rows r0..r1 reference B rows
// [INT_MAX - out[5], out[6] - 1] (out[0..6] zeroed by the caller)
cudaError_t launch_bandwidth(KMat a, KMat b, KMat c, int64_t r0, int64_t r1, int64_t b0, int64_t b1, int64_t n,
                             int count_sub, int32_t* out, cudaStream_t s);

// sp2_graph.cu: device-resident SP2 control (§8f-f3). The loop state lives in device memory; a
// one-thread control kernel at the end of every captured iteration applies the stop rule, the
// GROW/FAIL width rule and the branch rule (the host loop's decisions, same expressions), records
// the iteration, writes (alpha, beta, old_mode) of the next step for row_general_dyn_kernel and
// sets the condition of the graph's WHILE node.
struct Sp2Dev {
    // constants (host)
    double tol, stag_gate, nocc;
    int32_t min_iter, max_iter, on_overflow, closest, maxw, pad0;
    // state
    double dyn[3];  // alpha, beta, old_mode of the next step
    double trX, t2, e2, e1;  // tr X_n, T2 of X_n (trace-closest rule), e_{n-2}, e_{n-1}
    int32_t it, stop, wy, regrows, fail_iter, required, branch, pad1;
    int64_t overflow_rows;
};
// count rows of [0, n) with nnz > dev->wy into *out (the FAIL report over the logical width)
cudaError_t launch_count_over_dev(const int32_t* nnz, int64_t n, const Sp2Dev* dev, int32_t* out, cudaStream_t s);
// one thread: the loop's decisions after a step (sums: trS, trX_{n+1}, ||S - X||^2 [, T2 of X_{n+1}];
// status[1]: max kept; ovf: rows over the logical width; prod: products of the step); also zeroes
// ovf and prod for the next iteration. rec: the caller's sp2_iter_rec array (device).
cudaError_t launch_sp2_ctl(Sp2Dev* dev, const double* sums, const int32_t* status, int32_t* ovf,
                           unsigned long long* prod, void* rec, unsigned long long cond_handle, cudaStream_t s);

// tiny.cu: the small-matrix kernel (N <= 1024, one rank, no Old operand, B rows <= 64 slots,
// diag_a and diag_s set): rows, status and (sums != nullptr) the canonical sums of diag_a, diag_s
bool tiny_eligible(const RowOpParams& p, int64_t n);
size_t tiny_smem(int64_t n);
cudaError_t launch_tiny(const RowOpParams& p, int64_t n, unsigned int* counter, int32_t* part, int32_t* status,
                        double* sums, cudaStream_t s);

// split.cu: the split-row ring kernel (W warps per row, 16-bit balanced sub-records)
cudaError_t plan_split(const RowOpParams& p, int S, int W, int G, int num_sms, LaunchCfg* cfg);
cudaError_t launch_split(const RowOpParams& p, const LaunchCfg& cfg, cudaStream_t s);
size_t split_row_smem(int S, int W, bool has_old, int G);
// the warp-specialized ring kernel (accumulator warp + emitter warp per row, W = 1 records)
cudaError_t plan_ws(const RowOpParams& p, int S, int G, int num_sms, LaunchCfg* cfg);
cudaError_t launch_ws(const RowOpParams& p, const LaunchCfg& cfg, cudaStream_t s);
cudaError_t launch_balance_split(KMat b, int64_t k0, int64_t k1, int W, int G, int S, unsigned char* bt,
                                 int32_t* bt_nbin, int num_sms, cudaStream_t s);

// symmetric SP2 step (f4 ii): is h bitwise symmetric (ok[0] stays 0); reach of U's rows
cudaError_t launch_sym_check(KMat h, int64_t r0, int64_t r1, int32_t* bad, cudaStream_t s);
cudaError_t launch_upper_reach(KMat u, int64_t r0, int64_t r1, int32_t* reach, cudaStream_t s);
// row i of Y = L_i (column i of the rows j < i of U, ascending j) followed by U_i; status as the
// row kernel (rows over Y.w, max kept); normsq (nullable): upper-triangle norm -> full norm
cudaError_t launch_sym_assemble(KMat u, KMat x, KOut y, int64_t r0, int64_t r1, const int32_t* reach,
                                const double* diag_s, double* normsq, int32_t* status, int num_sms,
                                cudaStream_t s);

// reduce.cu
cudaError_t launch_block_partials(const double* const* arrays, int narr, int64_t row_begin,
                                  int64_t row_end, int64_t n, double* partials, cudaStream_t s);
cudaError_t launch_canonical_small(const double* const* arrays, int narr, int64_t n, double* out, cudaStream_t s);
cudaError_t launch_final_sums(const double* partials, int narr, int64_t nblocks, double* out,
                              cudaStream_t s);
cudaError_t launch_stored_diag(KMat a, int64_t row_begin, int64_t row_end, double* out,
                               cudaStream_t s);
cudaError_t launch_gershgorin(KMat h, int64_t row_begin, int64_t row_end,
                              unsigned long long* minmax_keys, cudaStream_t s);
cudaError_t launch_fnorm_rows(KMat a, KMat b, int64_t row_begin, int64_t row_end, double* out,
                              cudaStream_t s);
cudaError_t launch_sumsq_rows(KMat a, int64_t row_begin, int64_t row_end, double* out, cudaStream_t s);
cudaError_t launch_validate(KMat a, int64_t n, int32_t* bad, cudaStream_t s);
cudaError_t launch_identity(int64_t n, KOut id, cudaStream_t s);
cudaError_t launch_copy_rows(KMat src, KOut dst, int64_t row_begin, int64_t row_end,
                             int32_t* status, cudaStream_t s);
cudaError_t launch_breakpoints(KMat b, int64_t n, int S, int np, int32_t* bp, int num_sms, cudaStream_t s);
// out[0] = min first column, out[1] = max last column of a's rows r0..r1 (caller initialises
// out to {INT64_MAX, -1})
cudaError_t launch_col_range(KMat a, int64_t r0, int64_t r1, long long* out, cudaStream_t s);
cudaError_t launch_products(KMat a, const int32_t* nnz_b, int64_t r0, int64_t r1, unsigned long long* out,
                            cudaStream_t s);
cudaError_t launch_count_over(const int32_t* nnz, int64_t r0, int64_t r1, int32_t w, int32_t* out,
                              cudaStream_t s);
cudaError_t launch_max_nnz(const int32_t* nnz, int64_t row_begin, int64_t row_end,
                           int32_t* out, cudaStream_t s);

// Resident CTAs per SM of a kernel at (threads, dynamic smem), memoized per device: the first query
// raises the kernel's dynamic-shared-memory limit as needed; later calls are a table lookup (the
// runtime queries cost tens of microseconds, which a cfg1-sized call cannot afford).
cudaError_t occupancy_cached(const void* kern, int threads, size_t smem, int* bps);

// order-preserving double <-> u64 keys for exact atomic min/max
__host__ __device__ inline unsigned long long dkey(double x) {
    unsigned long long b;
#ifdef __CUDA_ARCH__
    b = (unsigned long long)__double_as_longlong(x);
#else
    __builtin_memcpy(&b, &x, 8);
#endif
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double dkey_inv(unsigned long long k) {
    unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    double x;
#ifdef __CUDA_ARCH__
    x = __longlong_as_double((long long)b);
#else
    __builtin_memcpy(&x, &b, 8);
#endif
    return x;
}

}  // namespace ell
