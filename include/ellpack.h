/*
 * ellpack.h — C ABI of libellpack, the B200 (sm_100a) hot path of arXiv 2102.08505:
 * the BML ELLPACK sparse matrix-matrix multiply with drop threshold and its use
 * inside the SP2 density-matrix purification loop of ExaSP2.
 *
 * Citations: P:Lnn = /root/reference/PAPER.md line nn; S:Lnn = SPEC.md line nn;
 * "§8x" = SURVEY.md section 8(x); "Rn" = reading n listed in DESIGN.md §Readings.
 *
 * GENERAL CONVENTIONS (every entry point)
 *  - Plain C types only. Return value: an ellpack_status (0 = ELLPACK_OK).
 *    No exception or abort crosses the ABI; CUDA errors become ELLPACK_ERR_CUDA.
 *  - Matrices are square N x N in canonical row-major ELLPACK (D1, §8a-a0;
 *    S:L28-35): val[N][w] float64, col[N][w] int32, nnz[N] int32, all in DEVICE
 *    memory of the context's device. Row i holds nnz[i] <= w entries in slots
 *    0..nnz[i]-1 with column indices strictly ascending in [0, N); slots >=
 *    nnz[i] are never read. Values must be finite. Inputs that violate this are
 *    undefined behaviour (release build trusts them; tests check them).
 *  - Pointers must be 16-byte aligned and w even (vectorised loads).
 *  - All work is ordered on the context's stream. Functions that return host
 *    scalars (status, traces, bounds, norms) synchronise that stream.
 *  - The drop rule (§8c-c3, "entries ... dropped after accumulation"):
 *    an output entry is stored iff |value| > threshold, threshold >= 0 finite,
 *    applied once to the final combined value (R3). threshold = 0 keeps exactly
 *    the nonzeros.
 *  - Arithmetic (R12): IEEE binary64, round-to-nearest-even. For every output
 *    entry the products a_ik*b_kj are accumulated as an fma chain s <- fma(a,b,s)
 *    from s = +0.0 in ascending k (the order of A's row), then combined once as
 *    c = fma(alpha, s, beta*c_old). Results are bitwise reproducible and equal
 *    to the CPU oracle's (oracle/oracle.c). Traces use the canonical sum
 *    (§8c-c7): sequential within 256-row blocks, then sequential over blocks.
 *  - OVERFLOW (§8c-c4): if some output row keeps more entries than
 *    the output width, the call returns ELLPACK_ERR_OVERFLOW; the output's rows
 *    are then truncated (contents unspecified beyond validity) but
 *    ellpack_overflow_info() reports the exact required width (max kept count)
 *    and the number of overflowing rows. Host out-params are written only on OK.
 *  - Multi-GPU (optional, ellpack_ctx_attach_nccl): every descriptor is a full
 *    N-row replica on every rank; each rank computes only its rows
 *    [row_begin, row_end) of every output, traces are assembled from
 *    all-gathered 256-row block partials (bitwise equal to one rank), and
 *    status/width decisions are all-reduced so all ranks agree.
 */
#ifndef ELLPACK_B200_H_
#define ELLPACK_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ellpack_status {
    ELLPACK_OK = 0,
    ELLPACK_ERR_ARG = 1,      /* invalid argument, aliasing, NaN/negative threshold */
    ELLPACK_ERR_DIM = 2,      /* dimension mismatch (S:L64 DimensionMismatch) */
    ELLPACK_ERR_OVERFLOW = 3, /* an output row exceeds its width (S:L46 OverflowError) */
    ELLPACK_ERR_BOUNDS = 4,   /* degenerate spectral bounds (S:L368 DegenerateBounds) */
    ELLPACK_ERR_NOCONV = 5,   /* SP2 hit max_iter (S:L374 NoConvergence); outputs valid */
    ELLPACK_ERR_NOMEM = 6,    /* device allocation failed */
    ELLPACK_ERR_CUDA = 7,     /* CUDA runtime / launch error */
    ELLPACK_ERR_NCCL = 8,     /* NCCL error */
    ELLPACK_ERR_STATE = 9     /* call not valid in the context's state */
} ellpack_status;

/* Non-owning view of one N x N ELLPACK matrix on the context's device (D1).
 * n: dimension N (> 0); w: width M (> 0, even); val/col: N*w entries; nnz: N. */
typedef struct ellpack_desc {
    int64_t n;
    int32_t w;
    int32_t reserved; /* must be 0 */
    double* val;
    int32_t* col;
    int32_t* nnz;
} ellpack_desc;

typedef struct ellpack_ctx_s* ellpack_ctx;

/* ---------------------------------------------------------------- context */

/* Bind device `device` and CUDA stream `stream` (a cudaStream_t, may be NULL =
 * legacy default stream, e.g. torch.cuda.current_stream().cuda_stream).
 * The context owns a device workspace pool (grown on demand), a small status
 * block and, optionally, an NCCL communicator. One context per host thread;
 * not thread-safe. Errors: ARG (out NULL / bad device), CUDA, NOMEM. */
int ellpack_ctx_create(int device, void* stream, ellpack_ctx* out);
int ellpack_ctx_destroy(ellpack_ctx ctx);
/* Re-bind the stream used by subsequent calls. */
int ellpack_ctx_set_stream(ellpack_ctx ctx, void* stream);

/* Tuning / fault-injection knobs (key, value). Unknown key -> ARG.
 *  ELLPACK_OPT_WINDOW      dense-window accumulator capacity per row, in
 *                          doubles (0 = automatic). Rows whose column span
 *                          exceeds it are processed in several passes.
 *  ELLPACK_OPT_WARPS       warps (rows in flight) per CTA (0 = automatic).
 *  ELLPACK_OPT_SP2_WIDTH0  fault injection: sp2_run starts its iterates at this
 *                          width (exercises GROW), 0 = off.
 *  ELLPACK_OPT_PROFILE     1 = bracket every launch of the fused row kernel (in the dense
 *                          regime: of the dense GEMM) with CUDA events on the context
 *                          stream and accumulate its device time (ellpack_ctx_kernel_time);
 *                          setting it resets the accumulators. 0 = off (default).
 *  ELLPACK_OPT_ABLATE      timing experiments only, results are WRONG when set (bit mask):
 *                          1 = the ring kernel skips its output-row stores, 2 = its
 *                          accumulator updates, 4 = its B gathers, 8 = its emission.
 *                          0 = off (default). Only builds with -DELL_ABLATE=1 accept a
 *                          nonzero mask (ELLPACK_ERR_ARG otherwise).
 *  ELLPACK_OPT_GENERAL_WINDOW  window (doubles, multiple of 32) of the general path that
 *                          wide rows (dense SP2 iterates) use; 0 = automatic (1024).
 *  ELLPACK_OPT_VALIDATE    nonzero: every entry point first checks its input operands
 *                          for canonical form on the device (0 <= nnz <= w; columns in
 *                          [0, N), strictly ascending; values finite; §8c-c1) and returns
 *                          ELLPACK_ERR_ARG on a violation (one extra kernel and one
 *                          synchronising read-back per operand set). 0 = inputs trusted
 *                          (default).
 *  ELLPACK_OPT_SP2_SYMMETRIC  1 (default): sp2_run with the GROW policy (any number of ranks) checks H for
 *                          bitwise symmetry; if symmetric, every SP2 step that runs on the general
 *                          (wide-row) path computes only the upper triangle of X_{n+1} (columns
 *                          j >= i) and mirrors it (§8f-f4 ii; X_n symmetric => X_n^2 bitwise
 *                          symmetric, P4), about half the products. Results are bitwise those of
 *                          the full computation. 0: always compute whole rows.
 *  ELLPACK_OPT_SP2_MEM_CAP fault injection: sp2_run treats an iterate allocation as not fitting
 *                          in device memory when the value arrays of its live iterates (X_n, X_{n+1},
 *                          the symmetric step's upper triangle) would exceed this many bytes
 *                          (exercises the fallback from the headroom width to the exact width and the
 *                          symmetric step's whole-row fallback); the dense regime's two N^2 arrays
 *                          "do not fit" when they exceed it (the run falls back to the sparse
 *                          kernels); 0 = off (default).
 *  ELLPACK_OPT_RING_KERNEL which kernel runs rows on the ring (narrow-band) path: 0 = automatic
 *                          (the split-row kernel with 1 warp per row whenever the output does not
 *                          alias an input and the ring fits 16-bit offsets, else the legacy ring
 *                          kernel), 1 = always the legacy ring kernel, 2 = the split-row kernel
 *                          with 1 warp per row, 3 = with 2 warps per row. Results are bitwise the
 *                          same for every choice (A/B experiments and tests).
 *  ELLPACK_OPT_SP2_DEVICE_LOOP  0 (default) = automatic: on one rank, for N <= 8192, sp2_run runs its
 *                          loop as ONE launch of a CUDA graph with a conditional WHILE node (branch,
 *                          stop and width rules decided on the device): no host
 *                          synchronisation per iteration; both iterates at the physical width
 *                          max_width, every step on the general path. 1 = always the host loop
 *                          (one synchronisation per iteration), 2 = the device loop whenever it
 *                          applies (one rank). Results are bitwise the same either way.
 *                          With the dense regime available (ELLPACK_OPT_DENSE 0), automatic picks
 *                          the device loop (every step dense) for N <= 1024 and otherwise the host
 *                          loop, whose steps switch to the dense GEMM when it is predicted faster.
 *  ELLPACK_OPT_DENSE       the dense-regime step (one rank, N <= 65536, X X only): X_n is scattered
 *                          into an N x N array and S = X_n^2 runs as a dense FP64 GEMM (k blocks
 *                          empty on either side skipped; only the upper triangle of tiles when X_n
 *                          is symmetric), then one warp per row combines, drops and compacts S into
 *                          X_{n+1}. Every output is still one fma chain over k ascending -- the
 *                          extra terms are exact zeros -- so results are bitwise those of the
 *                          sparse kernels. 0 (default) = automatic: an SP2 step goes dense when its
 *                          predicted time (FMAs of the k blocks inside X_n's band at the last dense
 *                          step's rate) is below 0.85 x the sparse prediction (the step's estimated
 *                          products at the last sparse step's rate), and the 2 (symmetric X) or 3
 *                          N^2-double arrays fit in 60% of the free device memory; 1 = never;
 *                          2 = always when they fit (every SP2 step on one rank and every
 *                          ellpack_multiply_x2; tests).
 *  ELLPACK_OPT_DENSE_KERNEL the dense GEMM's 128-row tiles: 0 (default) = on the FP64 MMA
 *                          (mma.sync m8n8k4) when a per-device self-check confirms it computes the
 *                          ascending fma chain bit for bit, else on FP64 FMAs; 1 = FP64 FMAs;
 *                          2 = the FP64 MMA (tests). Results are bitwise the same either way.
 *  ELLPACK_OPT_SMALL_KERNEL 0 (default) = ellpack_multiply_x2 on a small matrix (N <= 1024, one
 *                          rank, input width <= 64) runs the small-matrix kernel: 16 B rows' gathers
 *                          in flight per warp, status and the canonical trace sums finished by the
 *                          last CTA, one launch; 1 = the general path (row kernel + trace-sum kernel).
 *                          Results are bitwise the same either way. */
enum { ELLPACK_OPT_WINDOW = 1, ELLPACK_OPT_WARPS = 2, ELLPACK_OPT_SP2_WIDTH0 = 3, ELLPACK_OPT_PROFILE = 4,
       ELLPACK_OPT_ABLATE = 5, ELLPACK_OPT_GENERAL_WINDOW = 6, ELLPACK_OPT_VALIDATE = 7,
       ELLPACK_OPT_SP2_SYMMETRIC = 8, ELLPACK_OPT_SP2_MEM_CAP = 9, ELLPACK_OPT_RING_KERNEL = 10,
       ELLPACK_OPT_SP2_DEVICE_LOOP = 11, ELLPACK_OPT_DENSE = 12, ELLPACK_OPT_DENSE_KERNEL = 13,
       ELLPACK_OPT_SMALL_KERNEL = 14 };
int ellpack_ctx_set_option(ellpack_ctx ctx, int key, int64_t value);

/* Accumulated device time (ms, CUDA events on the ctx stream) and launch count of
 * the fused row kernel since ELLPACK_OPT_PROFILE was last set. */
int ellpack_ctx_kernel_time(ellpack_ctx ctx, double* row_kernel_ms, int64_t* row_kernel_launches);

/* Number of kernels this context launched since creation (evidence counter). */
int64_t ellpack_ctx_kernel_launches(ellpack_ctx ctx);

/* Number of blocking host synchronisations of the context stream since creation (evidence
 * counter for the SP2 control path: sp2_run waits once per iteration). */
int64_t ellpack_ctx_host_syncs(ellpack_ctx ctx);

/* Launch geometry of the last fused row-kernel launch on this context (what bench.py reports
 * beside its roofline): out[0] path (5 the small-matrix kernel of ellpack_multiply_x2, 4 dense regime -- out[1..7] then stale, 3 warp-specialized ring
 * kernel, 2 split-row ring kernel, 1 one-warp ring kernel, 0 general path), out[1] G (64-entry B groups per step, ring paths), out[2] S (ring / window doubles per
 * row), out[3] warps per CTA (split kernel: warps per row),
 * out[4] grid, out[5] dynamic shared memory bytes per CTA, out[6] resident CTAs per SM,
 * out[7] B half-bandwidth of the probe. Errors: ARG. */
int ellpack_ctx_last_launch(ellpack_ctx ctx, int32_t out[8]);

/* --------------------------------------------------------------- storage */

/* ellpack_create(N, M) (BJ north_star): allocate an N x M matrix on
 * the ctx device (stream-ordered cudaMallocAsync), all rows empty, padding 0.
 * Library-owned: release with ellpack_destroy. Errors: ARG (N <= 0, M <= 0 or
 * odd, M > N rounded up to even), NOMEM. */
int ellpack_create(ellpack_ctx ctx, int64_t n, int32_t m, ellpack_desc* out);
int ellpack_destroy(ellpack_ctx ctx, ellpack_desc* desc);

/* --------------------------------------------------------------- the ops */

/* C <- drop_tau(alpha*A*B + beta*C)  (BJ north_star (1); §8c-c2..c4;
 * P:L95-96 "sparse matrix-matrix multiply", P:L445-457 ELLPACK X^2).
 * Row i: s_j = fma chain over k ascending in A's row, then for j in the union of
 * the product pattern and (beta != 0 ? C_old row i : {}):
 * c = fma(alpha, s_j, beta*c_old_j or +0), kept iff |c| > threshold.
 * alpha == 0: no products are formed (NaN/Inf in A, B cannot leak); beta == 0:
 * C_old is never read (its NaNs cannot leak) (R13). C is updated in place row by
 * row; C must not alias A or B (checked by pointer -> ARG). A, B, C must share n
 * (DIM). On OVERFLOW C's rows are truncated to C.w; see ellpack_overflow_info. */
int ellpack_multiply(ellpack_ctx ctx, const ellpack_desc* a, const ellpack_desc* b,
                     ellpack_desc* c, double alpha, double beta, double threshold);

/* X2 <- drop_tau(X*X) with tr(X) and tr(X^2) from the same pass (
 * P:L493-494 "SP2 Loop X2"; §8c-c5). *trace_x = canonical sum of X's stored
 * diagonal; *trace_x2 = canonical sum of the PRE-drop diagonal of X*X (R5).
 * Either trace pointer may be NULL. X2 must not alias X. */
int ellpack_multiply_x2(ellpack_ctx ctx, const ellpack_desc* x, ellpack_desc* x2,
                        double threshold, double* trace_x, double* trace_x2);

/* A <- drop_tau(alpha*A + beta*B) (S:L78-86 add_scaled, BML argument order; §8c-c6).
 * Per entry of the union pattern: fma(alpha, a_j or 0, beta*(b_j or 0)).
 * In place on A, row by row. B may be the same descriptor as A ((alpha+beta)A). */
int ellpack_add(ellpack_ctx ctx, ellpack_desc* a, const ellpack_desc* b,
                double alpha, double beta, double threshold);

/* A <- drop_tau(A + beta*I) (BJ north_star "add_identity"; §8c-c6): the diagonal
 * becomes a_ii + beta in one rounding (inserted if absent). OVERFLOW if a full
 * row lacks its diagonal. */
int ellpack_add_identity(ellpack_ctx ctx, ellpack_desc* a, double beta, double threshold);

/* A <- drop_tau(alpha*A + beta*I): off-diagonal alpha*a_ij, diagonal
 * fma(alpha, a_ii or 0, beta). The SP2 X0 map (§8c-c9). */
int ellpack_scale_add_identity(ellpack_ctx ctx, ellpack_desc* a, double alpha, double beta,
                               double threshold);

/* *out = canonical sum of A's stored diagonal (§8c-c7). Syncs. */
int ellpack_trace(ellpack_ctx ctx, const ellpack_desc* a, double* out);

/* *out = ||A - B||_F over the union pattern (S:L91-96 fnorm_diff; P:L494
 * "SP2 Loop Norm"; §8c-c11). A diagnostic: its summation order is
 * deterministic but not the oracle's. Errors: DIM. Syncs. */
int ellpack_fnorm_diff(ellpack_ctx ctx, const ellpack_desc* a, const ellpack_desc* b, double* out);

/* Gershgorin bounds (§8c-c8): r_i = sequential sum of |h_ij|, j != i,
 * in slot order; *emin = min(h_ii - r_i), *emax = max(h_ii + r_i). Syncs. */
int ellpack_gershgorin(ellpack_ctx ctx, const ellpack_desc* h, double* emin, double* emax);

/* Details of the last ELLPACK_ERR_OVERFLOW returned on this context
 * (required width = max kept count over rows; overflow rows = #rows kept > w, exact, also
 * for sp2_run's FAIL at X0 (rows of X0 over the initial width) and inside the loop (rows of
 * X_{n+1} over the current width), §8c-c4). */
int ellpack_overflow_info(ellpack_ctx ctx, int64_t* overflow_rows, int32_t* required_width);

/* ------------------------------------------------------------------ SP2 */

enum { SP2_FAIL = 0, SP2_GROW = 1 };
enum { SP2_CONVERGED = 0, SP2_STAGNATED = 1, SP2_MAXITER = 2, SP2_OVERFLOWED = 3 };
enum { SP2_SQUARE = 0, SP2_EXPAND = 1 };
/* Branch rules. TRACE_SIGN: SQUARE iff tr(X_n) > nocc (tie -> EXPAND).
 * TRACE_CLOSEST (§8f-f4 (i); P:L52 cites Niklasson 2002; reading R19):
 * SQUARE iff |T2 - nocc| < |(2 tr(X_n) - T2) - nocc| (tie -> EXPAND), where
 * T2 = canonical sum over rows of q_i, q_i = fma chain q <- fma(x, x, q) over the
 * stored slots of row i in ascending order from +0: for symmetric X_n (every
 * iterate of a symmetric H) T2 = sum_ij x_ij^2 = tr(X_n^2) in exact arithmetic,
 * so the rule is decided before the fused step. T2 of X_{n+1} is computed right
 * after step n and fetched with that step's traces (no extra synchronisation). */
enum { SP2_RULE_TRACE_SIGN = 0, SP2_RULE_TRACE_CLOSEST = 1 };

typedef struct sp2_opts {
    double threshold;      /* tau, drop threshold of every iterate (default 0) */
    int32_t max_iter;      /* default 100 */
    int32_t min_iter;      /* stagnation test active from iteration min_iter (default 20) */
    double stag_gate;      /* stagnation test active only when e_n <= stag_gate (1e-3) */
    double emin, emax;     /* spectral bounds; NaN -> Gershgorin */
    int32_t on_overflow;   /* SP2_FAIL | SP2_GROW (default GROW) */
    int32_t max_width;     /* GROW ceiling (<= 0 -> N) */
    int32_t initial_width; /* width of X0 (<= 0 -> H.w) */
    int32_t branch_rule;   /* SP2_RULE_TRACE_SIGN (default) | SP2_RULE_TRACE_CLOSEST */
} sp2_opts;

typedef struct sp2_iter_rec {
    double trX, trS, e, fnorm; /* tr(X_n), tr(X_n^2) pre-drop, e_n = trX-trS, ||X_n^2-X_n||_F */
    int32_t branch;            /* SP2_SQUARE | SP2_EXPAND */
    int32_t width;             /* width of X_{n+1} */
    int32_t required;          /* max kept count of X_{n+1} */
    int32_t regime;            /* 0: the sparse row kernels; 1: the dense regime (ELLPACK_OPT_DENSE) */
    int64_t products;          /* scalar products of this X^2 (pattern count) */
    double frob2;              /* TRACE_CLOSEST: T2 of X_n that decided the branch; else 0 */
    int64_t products_exec;     /* products the GPU executed for this step: = products, or about half
                                  of them when the symmetric step (ELLPACK_OPT_SP2_SYMMETRIC) ran;
                                  dense regime: the FMAs of the GEMM's non-empty k blocks */
    double step_ms;            /* host loop: device time of the step (X^2 + combine, CUDA events on the
                                  ctx stream); device loop: NaN (the loop is one graph launch) */
} sp2_iter_rec;

typedef struct sp2_report {
    int32_t iterations, stop_reason, final_width, regrows;
    double emin, emax, trD;
    int64_t overflow_rows;
    int32_t required_width, fail_iter;
    /* phase seconds (P:L491-495 phase names) */
    double t_read_hamiltonian, t_init_misc, t_sp2_loop_x2, t_sp2_loop_norm, t_sp2_loop_misc;
    sp2_iter_rec* iters;       /* caller-provided array of >= max_iter records, or NULL */
} sp2_report;

/* SP2-Basic purification (BJ north_star (2); P:L52,
 * P:L368-371; §8c-c9..c10):
 *   bounds (Gershgorin unless given), X0 = drop(alpha*H + beta*I) with
 *   alpha = -1/(emax-emin), beta = emax/(emax-emin); then per iteration n:
 *   branch = tr(X_n) > nocc ? SQUARE : EXPAND (tie -> EXPAND), or the
 *   trace-closest rule above when opts->branch_rule = SP2_RULE_TRACE_CLOSEST;
 *   ONE fused pass computes S = X_n^2 and writes X_{n+1} = drop(S) or
 *   drop(2X_n - S) with tr(S), tr(X_{n+1}) and ||S - X_n||_F^2 partials;
 *   stop when |tr(X_n) - tr(S)| <= tol (CONVERGED), on gated stagnation
 *   (STAGNATED) or at max_iter (ELLPACK_ERR_NOCONV). Overflow: FAIL returns
 *   OVERFLOW; GROW re-creates X_{n+1} at round_up32(required) and redoes step n.
 * D (caller-owned, width D->w) receives the final iterate; OVERFLOW if too
 * narrow. rep may be NULL. Errors: ARG (nocc not in [0,N], tol < 0), BOUNDS,
 * OVERFLOW, NOCONV (D and rep still valid), NOMEM, CUDA, NCCL; STATE if the context's rows are
 * restricted (ellpack_ctx_set_rows) without a communicator. Iterates live in context-owned
 * buffers that are reused across calls. */
int sp2_run(ellpack_ctx ctx, const ellpack_desc* h, int64_t nocc, double tol,
            const sp2_opts* opts, ellpack_desc* d, sp2_report* rep);

/* Fill *opts with the defaults listed above. */
void sp2_opts_default(sp2_opts* opts);

/* ------------------------------------------------------- host-buffer path */

/* End-to-end X^2 through HOST memory (the bench's e2e leg): copies X (host
 * arrays, n x wx) to the device, runs ellpack_multiply_x2 into a device buffer of
 * width wx2, copies X2 back into the host arrays (n x wx2) -- with a communicator
 * only this rank's rows [row_begin, row_end) of X2 (X is copied whole: it is the B
 * operand). Host arrays should be pinned for full PCIe bandwidth. Device scratch is
 * owned by the context and reused across calls. Errors as ellpack_multiply_x2. */
int ellpack_multiply_x2_host(ellpack_ctx ctx, int64_t n,
                             int32_t wx, const double* x_val, const int32_t* x_col, const int32_t* x_nnz,
                             int32_t wx2, double* x2_val, int32_t* x2_col, int32_t* x2_nnz,
                             double threshold, double* trace_x, double* trace_x2);

/* ------------------------------------------------------------ multi-GPU */

/* NCCL bootstrap: rank 0 calls ellpack_nccl_unique_id and broadcasts the 128
 * bytes (e.g. torch.distributed.broadcast_object_list); every rank then calls
 * ellpack_ctx_attach_nccl (collective). Rows [row_begin,row_end) are this
 * rank's block. The blocks of all ranks are all-gathered and checked: they must be
 * contiguous, ascending with rank, EQUAL, a multiple of 256 rows each (canonical
 * trace blocks and equal all-gather counts, §8c-c7/c12, reading R17) and cover
 * [0, N) with N = nranks * block; otherwise every rank returns ELLPACK_ERR_ARG and
 * no communicator is attached. Afterwards every operand of every call must have
 * n == N (ELLPACK_ERR_DIM otherwise). Errors: ARG, NCCL, CUDA, STATE (already attached). */
int ellpack_nccl_unique_id(uint8_t id[128]);
int ellpack_ctx_attach_nccl(ellpack_ctx ctx, int nranks, int rank, const uint8_t id[128],
                            int64_t row_begin, int64_t row_end);

/* Restrict this context's outputs to rows [row_begin, row_end) WITHOUT a
 * communicator (single-process emulation of one rank; used by tests). */
int ellpack_ctx_set_rows(ellpack_ctx ctx, int64_t row_begin, int64_t row_end);

/* All-gather the row blocks of a replicated matrix in place over the attached
 * communicator (the B-operand exchange of BJ north_star (3)). No-op without one. */
int ellpack_allgather_rows(ellpack_ctx ctx, ellpack_desc* m);

/* Band-aware halo exchange, the alternative to the full all-gather when the
 * operands are banded: the rows [row_begin,row_end) of `a` on this rank reference only the B rows
 * [lo, hi] (lo = min first column, hi = max last column of those rows), so each rank needs just
 * those rows of `b`. In place over the attached communicator: every rank's [lo, hi] is
 * all-gathered (16 bytes per rank), then the rows of the plan below travel by NCCL send/recv
 * (val, col, nnz). a and b may be the same matrix (X^2, SP2). Rows of b outside this rank's
 * block and its [lo, hi] are left untouched (not valid for this rank). No-op without a
 * communicator. Errors: ARG, DIM, CUDA, NCCL. sp2_run uses it between iterations and all-gathers
 * only the final iterate. */
int ellpack_halo_rows(ellpack_ctx ctx, const ellpack_desc* a, ellpack_desc* b);

/* X2 <- drop_tau(X*X) for this rank's rows when X holds only this rank's block valid (as an SP2
 * iterate or a row-distributed input does): the band-aware halo of X (the rows of other ranks this
 * rank's rows reference, ellpack_halo_rows) travels by NCCL on a second stream WHILE the interior
 * rows -- rows i with [i - h, i + h] inside the rank's block, h the all-reduced half-bandwidth of
 * X's rows -- are computed from the rank's own rows; the boundary rows follow once the halo is in
 * (SURVEY §8f-f1 "exchange that halo ... while computing interior rows whose k's are all local").
 * Traces and status as ellpack_multiply_x2; X's halo rows are received into X. Without a
 * communicator nothing is exchanged (X must then hold every row the block references) and the
 * rows are computed in the same interior / boundary launches. Errors as ellpack_multiply_x2. */
int ellpack_multiply_x2_halo(ellpack_ctx ctx, ellpack_desc* x, ellpack_desc* x2, double threshold,
                             double* trace_x, double* trace_x2);

/* The row split of ellpack_multiply_x2_halo (host only): block [r0, r1), half-bandwidth h ->
 * out[0..1] interior rows [i0, i1) = [min(r1, r0 + h), max(i0, r1 - h)), out[2..3] and out[4..5]
 * the boundary rows [r0, i0) and [i1, r1). Errors: ARG. */
int ellpack_row_split(int64_t r0, int64_t r1, int64_t h, int64_t out[6]);

/* The halo plan (host only, no context; the same function both sides of every pair evaluate):
 * equal contiguous blocks of `per` rows (block q = [q per, min(n, (q+1) per))) and every rank's
 * referenced rows need[2q] .. need[2q+1] (inclusive; need[2q] > need[2q+1] = none). This rank
 * sends (peer, row_begin, row_end) = its block ∩ the peer's range, and receives the peer's block
 * ∩ its own range, peers ascending, into send[3k..3k+2] (k < *n_send) and recv[3k..3k+2]
 * (k < *n_recv); both arrays hold 3 nranks entries. Errors: ARG. */
int ellpack_halo_plan(int64_t n, int nranks, int rank, int64_t per, const int64_t* need,
                      int32_t* n_send, int64_t* send, int32_t* n_recv, int64_t* recv);

const char* ellpack_strerror(int status);

#ifdef __cplusplus
}
#endif
#endif /* ELLPACK_B200_H_ */
