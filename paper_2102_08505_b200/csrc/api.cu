// api.cu — the C ABI of libellpack (include/ellpack.h): context, validation, the
// ELLPACK ops, the SP2-Basic driver and the NCCL row-block exchange.
//
// Every op is one launch of the fused row kernel (spgemm.cu) plus, where traces
// are returned, the canonical block-sum kernels (reduce.cu):
//   multiply            A x B,  Old = C (beta != 0), C in place
//   multiply_x2         X x X,  diag_a/diag_s -> tr(X), tr(X^2)
//   add                 A x I,  Old = B (old_mode 1), C = A in place   -> fma(alpha, a, beta*b)
//   (scale_)add_identity A x I, Old = I                                -> fma(alpha, a_ii, beta)
//   sp2 step            X x X,  Old = X, C = X_{n+1}                   (BJ north_star (2))
// A x I reproduces a exactly (fma(a, 1, +0) = a), so add/identity share the
// kernel's single-rounding combine instead of a second code path.
#include "internal.cuh"
#include "dense.cuh"
#include "../../include/ellpack.h"

#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only: ranges are no-ops unless a profiler is attached

#include <algorithm>
#include <chrono>
#include <climits>
#include <initializer_list>
#include <cstdio>
#include <vector>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>

using namespace ell;

// Dense-window limits (doubles per row): rows whose centred window needs more than
// kFastWindowMax use the multi-pass general path with kGeneralWindow.
constexpr int64_t kFastWindowMax = 12288;  // 96 KB + stage per warp
constexpr int kFastMinRows = 4;            // ring path only with >= 4 rows resident per SM
constexpr int64_t kGeneralWindow = 1024;
constexpr int kProbe = 7;  // bandwidth-probe words (launch_bandwidth)
#ifndef ELL_ROW_CHUNK
#define ELL_ROW_CHUNK 4  // rows per ticket of the ring kernels (large launches)
#endif
constexpr int64_t kNoProbeN = 1024;  // up to this N a row op runs unprobed on one general-path window
constexpr int64_t kSplitRingMax = 8064;  // split kernel: ring slots (16-bit byte offsets incl. trash)  // measured best for cfg3/cfg4 SP2 (512..4096 swept)

namespace {

struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
};

// NCCL entry points resolved at attach time (torch's libnccl.so.2), so the
// library loads on machines without NCCL.
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
};

NcclApi g_nccl;

bool load_nccl() {
    if (g_nccl.ok) return true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        const char* envp = getenv("ELLPACK_NCCL_LIB");
        if (envp) h = dlopen(envp, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) return false;
#define LOADSYM(field, name) g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
    if (!g_nccl.field) return false;
    LOADSYM(GetUniqueId, "ncclGetUniqueId");
    LOADSYM(CommInitRank, "ncclCommInitRank");
    LOADSYM(CommDestroy, "ncclCommDestroy");
    LOADSYM(AllGather, "ncclAllGather");
    LOADSYM(AllReduce, "ncclAllReduce");
    LOADSYM(GroupStart, "ncclGroupStart");
    LOADSYM(GroupEnd, "ncclGroupEnd");
    LOADSYM(Send, "ncclSend");
    LOADSYM(Recv, "ncclRecv");
    LOADSYM(CommGetAsyncError, "ncclCommGetAsyncError");
#undef LOADSYM
    g_nccl.ok = true;
    return true;
}

}  // namespace

struct ellpack_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    int window_opt = 0, warps_opt = 0, sp2_width0 = 0, ablate = 0, general_s = 0, validate = 0;
    int sp2_sym = 1;     // ELLPACK_OPT_SP2_SYMMETRIC
    int last_upper = 0;  // the last row op computed the upper triangle only
    int64_t launches = 0;
    int64_t host_syncs = 0;   // blocking stream synchronisations (evidence counter, f3)
    int64_t sp2_mem_cap = 0;  // ELLPACK_OPT_SP2_MEM_CAP: max bytes of the live SP2 iterate value arrays
    int64_t it_live[4] = {0, 0, 0, 0};  // value-array bytes of each live SP2 iterate slot
    int sym_nomem = 0;        // the symmetric step's U buffer did not fit (whole rows instead)
    // small device/pinned blocks
    int32_t* d_status = nullptr;              // [0] ovf rows, [1] max kept
    unsigned long long* d_keys = nullptr;     // gershgorin min/max keys; [2] SP2 product count
    double* d_sums = nullptr;                 // final sums (<= 8)
    int32_t* d_bw = nullptr;                  // bandwidth probe [0..5]; [8] agreed width (comm)
    LaunchCfg last_cfg{};
    int32_t last_fast = 0, last_hB = 0, last_split = 0;
    int ring_kernel = 0;  // ELLPACK_OPT_RING_KERNEL
    int small_kernel = 0;  // ELLPACK_OPT_SMALL_KERNEL
    int sp2_loop = 0;     // ELLPACK_OPT_SP2_DEVICE_LOOP
    int force_general_s = 0;  // device SP2 loop: every row op on the general path with this window
    Buf sp2dev, sp2rec;       // device SP2 loop: control block, iteration records
    cudaGraphExec_t x2_exec = nullptr;   // small unprobed X^2: the captured launch sequence, replayed
    uint64_t x2_exec_key = 0;
    int x2_exec_launches = 0;
    bool x2_exec_ok = false;             // cleared by every option change (the launch plan depends on them)
    LaunchCfg x2_cfg{};                  // the captured call's launch record (ellpack_ctx_last_launch)
    int x2_fast = 0, x2_split = 0, x2_hB = 0, x2_small = 0;
    cudaGraphExec_t sp2_exec = nullptr;  // device SP2 loop: the instantiated graph and what it captured
    uint64_t sp2_exec_key = 0;
    int sp2_exec_launches = 0;
    bool last_step_general = false;
    int dense_opt = 0;     // ELLPACK_OPT_DENSE
    int dense_kernel = 0;  // ELLPACK_OPT_DENSE_KERNEL
    Buf dense[3];          // dense regime: X (or B), X^T (non-symmetric A), S -- np x np doubles each
    Buf dflags;            // dense regime: k-block occupancy of the left and right operands
    Buf docc;              // dense regime: occupancy bitsets of the next SP2 operand (exact GEMM work)
    Buf old_val, old_col, old_nnz;  // ellpack_multiply with beta != 0: the scratch copy of C_old
    int last_dense = 0;    // the last SP2 step / X^2 ran in the dense regime
    int last_small = 0;    // the last X^2 ran the small-matrix kernel (tiny.cu)
    int64_t dense_clean_np = 0;  // dense[0] is zero outside the blocks dflags' fa marks (for this N_p)
    int64_t dense_fit_key = -1;  // dense_fits: the cached free-memory answer (N_p, arrays)
    bool dense_fit_ok = false;
    bool dense_full_clear = false;  // the last dense step zeroed the whole array (one-time cost)
    struct Host {
        int32_t bw[8];
        int32_t status_u[2];
        int32_t status[4];
        unsigned long long keys[4];
        double sums[8];
        int32_t imax;
    }* h = nullptr;
    Host* h_dev = nullptr;  // the same pinned block as the device addresses it (mapped; nullable)
    // workspace
    Buf rows[4];      // per-row double arrays
    Buf partials;     // canonical block partials
    Buf stash_val, stash_col;
    Buf ident_val, ident_col, ident_nnz;
    int64_t ident_n = 0;
    Buf hx_val, hx_col, hx_nnz, hy_val, hy_col, hy_nnz;  // host-path device copies
    Buf bt, bt_nbin, bp;
    Buf halo;  // all ranks' referenced row ranges (halo exchange)
    Buf vflag; // ELLPACK_OPT_VALIDATE violation flag
    Buf symaux; // symmetric SP2 step: [0] H asymmetric flag, [1] U reach, [2..3] U status
    Buf tiny;   // small-matrix kernel (tiny.cu): [0] last-CTA counter (kept zero), [4..) 2 ints per CTA
    Buf it[4][3];  // SP2 iterate buffers (val, col, nnz) x 4 slots
    int32_t* h_reach = nullptr;  // pinned: every rank's probe reach (2 per rank), fetched with a step
    // ring sizing cache: (hB, G, mode) -> (S, rows resident per SM)
    int64_t ring_key = -1;
    int ring_S = 0;
    bool ring_ok = true;
    // overflow info of the last OVERFLOW
    int64_t last_ovf_rows = 0;
    int32_t last_req = 0;
    // row partition
    int64_t row_begin = 0, row_end = -1;
    int64_t comm_n = 0;  // with a communicator: N of every operand (ranks' equal blocks cover [0, N))
    int nranks = 1, rank = 0;
    ncclComm_t comm = nullptr;
    cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    // row-kernel profiling (ELLPACK_OPT_PROFILE)
    bool profile = false, prof_pending = false;
    int prof_n = 0;                                    // row-kernel launches awaiting collection
    cudaEvent_t pev[4][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
    cudaStream_t side = nullptr;                       // halo exchange beside the interior rows (f1)
    cudaEvent_t sev[2] = {nullptr, nullptr};
    double prof_ms = 0.0;
    int64_t prof_launches = 0;
};

namespace {

int from_cuda(cudaError_t e) {
    if (e == cudaSuccess) return ELLPACK_OK;
    if (e == cudaErrorMemoryAllocation) return ELLPACK_ERR_NOMEM;
    return ELLPACK_ERR_CUDA;
}

#define CK(x)                                  \
    do {                                       \
        cudaError_t e_ = (x);                  \
        if (e_ != cudaSuccess) return from_cuda(e_); \
    } while (0)
#define RK(x)                                  \
    do {                                       \
        int r_ = (x);                          \
        if (r_ != ELLPACK_OK) return r_;       \
    } while (0)
#define NK(x)                                  \
    do {                                       \
        if ((x) != ncclSuccess) return ELLPACK_ERR_NCCL; \
    } while (0)

// every blocking wait on the context stream goes through here (counted: ellpack_ctx_host_syncs)
int host_sync(ellpack_ctx c) {
    c->host_syncs++;
    CK(cudaStreamSynchronize(c->stream));
    if (c->comm) {
        // a failed or aborted communicator (peer lost, network error) surfaces here, not as a hang
        ncclResult_t ae = ncclSuccess;
        if (g_nccl.CommGetAsyncError(c->comm, &ae) != ncclSuccess || ae != ncclSuccess) return ELLPACK_ERR_NCCL;
    }
    return ELLPACK_OK;
}

// hash combine for the keys of cached CUDA graphs
uint64_t mix64(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
}

// NVTX range over a scope (the paper's phase names), visible in nsys / ncu timelines
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    void next(const char* name) { nvtxRangePop(); nvtxRangePushA(name); }  // the next phase
    ~NvtxRange() { nvtxRangePop(); }
};

// With a communicator every operand must be the N x N matrix the ranks' blocks partition.
int check_comm_n(ellpack_ctx c, int64_t n) {
    return (c->comm && n != c->comm_n) ? ELLPACK_ERR_DIM : ELLPACK_OK;
}

int grow(ellpack_ctx c, Buf& b, size_t bytes) {
    if (b.bytes >= bytes) return ELLPACK_OK;
    if (b.p) CK(cudaFreeAsync(b.p, c->stream));
    b.p = nullptr;
    b.bytes = 0;
    size_t want = bytes + bytes / 8 + 256;
    CK(cudaMallocAsync(&b.p, want, c->stream));
    b.bytes = want;
    return ELLPACK_OK;
}

void release(ellpack_ctx c, Buf& b) {
    if (b.p) cudaFreeAsync(b.p, c->stream);
    b.p = nullptr;
    b.bytes = 0;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int check_desc(const ellpack_desc* d) {
    if (!d || d->n <= 0 || d->w <= 0 || (d->w & 1) || !d->val || !d->col || !d->nnz)
        return ELLPACK_ERR_ARG;
    if (d->n > INT32_MAX) return ELLPACK_ERR_ARG;
    if (!aligned16(d->val) || !aligned16(d->col) || (reinterpret_cast<uintptr_t>(d->nnz) & 3))
        return ELLPACK_ERR_ARG;
    return ELLPACK_OK;
}

bool valid_tau(double t) { return t >= 0.0 && std::isfinite(t); }

// ELLPACK_OPT_VALIDATE: canonical-form check of input operands on the device (one thread per
// row, one synchronising read-back); ARG on any violation. Off: inputs are trusted (§8b).
int validate_inputs(ellpack_ctx c, std::initializer_list<const ellpack_desc*> ds) {
    if (!c->validate) return ELLPACK_OK;
    RK(grow(c, c->vflag, sizeof(int32_t)));
    int32_t* flag = (int32_t*)c->vflag.p;
    CK(cudaMemsetAsync(flag, 0, sizeof(int32_t), c->stream));
    for (const ellpack_desc* d : ds) {
        CK(launch_validate(KMat{d->val, d->col, d->nnz, d->w}, d->n, flag, c->stream));
        c->launches++;
    }
    int32_t bad = 0;
    CK(cudaMemcpyAsync(&bad, flag, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
    RK(host_sync(c));
    return bad ? ELLPACK_ERR_ARG : ELLPACK_OK;
}

KMat kmat(const ellpack_desc* d) { return KMat{d->val, d->col, d->nnz, d->w}; }
KOut kout(const ellpack_desc* d) { return KOut{d->val, d->col, d->nnz, d->w}; }

bool same(const ellpack_desc* a, const ellpack_desc* b) {
    return a->val == b->val || a->col == b->col || a->nnz == b->nnz;
}

void rows_of(ellpack_ctx c, int64_t n, int64_t* r0, int64_t* r1) {
    if (c->row_end < 0) { *r0 = 0; *r1 = n; }
    else { *r0 = c->row_begin < n ? c->row_begin : n; *r1 = c->row_end < n ? c->row_end : n; }
}

int ensure_identity(ellpack_ctx c, int64_t n) {
    if (c->ident_n >= n) return ELLPACK_OK;
    RK(grow(c, c->ident_val, sizeof(double) * 2 * n));
    RK(grow(c, c->ident_col, sizeof(int32_t) * 2 * n));
    RK(grow(c, c->ident_nnz, sizeof(int32_t) * n));
    CK(launch_identity(n, KOut{(double*)c->ident_val.p, (int32_t*)c->ident_col.p,
                               (int32_t*)c->ident_nnz.p, 2}, c->stream));
    c->launches++;
    c->ident_n = n;
    return ELLPACK_OK;
}

KMat identity(ellpack_ctx c) {
    return KMat{(const double*)c->ident_val.p, (const int32_t*)c->ident_col.p,
                (const int32_t*)c->ident_nnz.p, 2};
}

// all-reduce of the status block (sum overflow rows, max kept) over the comm
int reduce_status(ellpack_ctx c) {
    if (!c->comm) return ELLPACK_OK;
    NK(g_nccl.GroupStart());
    NK(g_nccl.AllReduce(c->d_status, c->d_status, 1, ncclInt32, ncclSum, c->comm, c->stream));
    NK(g_nccl.AllReduce(c->d_status + 1, c->d_status + 1, 1, ncclInt32, ncclMax, c->comm, c->stream));
    NK(g_nccl.GroupEnd());
    return ELLPACK_OK;
}

// Bandwidth probe of a row op, enqueued only (d_bw[0..kProbe), see launch_bandwidth). With a
// communicator each rank probes its own rows of every operand and the maxima (half-bandwidths,
// max nnz and max chunk-parity sub-row of B: d_bw[0..4]) are all-reduced, so every rank plans the
// same launch from the global values even when it holds only its block + halo of B; the reach
// (d_bw[5..6]) stays per rank.
int enqueue_probe(ellpack_ctx c, const RowOpParams& p, int64_t n) {
    const bool has_old = p.old_mode != 0;
    CK(cudaMemsetAsync(c->d_bw, 0, kProbe * sizeof(int32_t), c->stream));
    const KMat none{nullptr, nullptr, nullptr, 0};
    const int64_t b0 = c->comm ? p.row_begin : 0, b1 = c->comm ? p.row_end : n;
    CK(launch_bandwidth(p.alpha != 0.0 ? p.A : none, p.B, has_old ? p.Old : none, p.row_begin, p.row_end,
                        b0, b1, n, c->ring_kernel == 3, c->d_bw, c->stream));
    c->launches++;
    if (c->comm) NK(g_nccl.AllReduce(c->d_bw, c->d_bw, 5, ncclInt32, ncclMax, c->comm, c->stream));
    return ELLPACK_OK;
}

// Enqueue one row op (kernel + scratch management). Status is left in d_status.
// The launch geometry comes from a bandwidth probe (one tiny kernel + a 24-byte read-back, or
// `bw`: the probe values of these operands already on the host, e.g. fetched by the previous SP2
// step with its status -- then nothing here waits on the device): with half-bandwidths hA, hB,
// hOld every row's products and Old entries lie within i +- h, h = max(hA + hB, hOld), so a
// ring of S >= 2 hB + 33 doubles holds the live part of every row ("fast path", progressive
// emission). Wider rows use the multi-pass general path.
// alloc_upper (nullable): called when a launch takes the symmetric (upper-triangle) route, to
// provide p.C_upper; a NOMEM there falls back to whole rows (c->sym_nomem = 1).
// Per-launch extras of a row op split into several launches (the halo-overlapped multiply, f1):
// which B rows the balance pass prepares (nbal ranges [k0, k1); default: every row the launch's A
// rows reference) and whether the status block accumulates over the previous launch.
struct RowOpExtra {
    int nbal = -1;
    int64_t bal[4] = {0, 0, 0, 0};
    bool keep_status = false;
};

int enqueue_row_op(ellpack_ctx c, RowOpParams& p, int64_t n, const int32_t* bw = nullptr,
                   int (*alloc_upper)(ellpack_ctx, void*, KOut*) = nullptr, void* alloc_arg = nullptr,
                   const RowOpExtra* ex = nullptr) {
    p.ncols = n;
    c->last_dense = 0;
    c->last_small = 0;
    const bool has_old = p.old_mode != 0;
    // A small matrix (N <= kNoProbeN, one rank) needs no probe: one general-path window covers every
    // column, so nothing depends on the bandwidths and the call waits on the device once, at the end
    // (the cfg1-sized calls are launch- and synchronisation-bound).
    int32_t bwv[kProbe] = {0, 0, 0, 0, 0, INT_MAX, (int32_t)std::min<int64_t>(n, INT_MAX)};
    const bool no_probe = !bw && n <= kNoProbeN && !c->comm && c->window_opt == 0 && c->ring_kernel == 0;
    if (!bw && !no_probe) {
        RK(enqueue_probe(c, p, n));
        CK(cudaMemcpyAsync(c->h->bw, c->d_bw, kProbe * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
        RK(host_sync(c));
        bw = c->h->bw;
    }
    if (bw) memcpy(bwv, bw, sizeof bwv);
    const int64_t hB = bwv[1];
    const int64_t hprod = p.alpha != 0.0 ? (int64_t)bwv[0] + hB : 0;
    const int64_t h = has_old ? (hprod > bwv[2] ? hprod : bwv[2]) : hprod;
    const int64_t nr = (n + 31) & ~int64_t(31);
    const int maxnb = p.alpha != 0.0 ? bwv[3] : 0;
    const int groups = maxnb <= 64 ? 1 : (maxnb + 63) / 64;
    p.hB = (int32_t)hB;
    p.ablate = c->ablate;
    // ring fast path: S >= 2 hB + 33 slots (progressive emission), B rows <= 256 entries
    int64_t ring = (2 * hB + 33 + 31) & ~int64_t(31);
    if (ring > nr) ring = nr < 32 ? 32 : nr;
    int64_t S;
    // split-row ring kernel (split.cu): W warps per row, 128-column emission blocks, 16-bit slots:
    // the default ring path whenever C does not alias an input (no stash) and the ring's byte
    // offsets fit 16 bits (S + 16 <= 8192 slots)
    int split_w = 0, split_g = 0;
    LaunchCfg scfg{};
    {
        const int rk = c->ring_kernel;
        const int64_t sring = (2 * hB + 129 + 127) & ~int64_t(127);
        const bool stash = p.stash_a || p.stash_old;
        if (c->window_opt == 0 && c->force_general_s == 0 && !no_probe && rk != 1 && !stash && groups <= 4 &&
            sring <= kSplitRingMax) {
            // W = 0: the warp-specialized kernel (accumulator + emitter warps, W = 1 records)
            // automatic: one warp per row; the warp-specialized experiment has no Old operand
            const int W = rk == 3 ? 2 : ((rk == 4 && !has_old) ? 0 : 1);
            const int maxsub = p.alpha != 0.0 ? bwv[4] : 0;
            const int G = W != 2 ? (groups < 1 ? 1 : groups) : std::max(1, (maxsub + 63) / 64);
            const int mode = !has_old ? 0 : (p.normsq ? 2 : 1);
            const int64_t key = (((sring * 8 + G) * 4 + mode) * 4 + W) * 2 + 1;
            auto plan = [&](int64_t S_, LaunchCfg* t_) {
                return W == 0 ? plan_ws(p, (int)S_, G, c->num_sms, t_) : plan_split(p, (int)S_, W, G, c->num_sms, t_);
            };
            if (key != c->ring_key) {
                LaunchCfg t;
                CK(plan(sring, &t));
                c->ring_ok = t.bps >= kFastMinRows;  // rows in flight per SM
                int64_t grown = sring;
                // slack: emission every few halves instead of every half, at the same rows per SM
                for (int64_t s2 = sring + 128; s2 <= sring + 512 && s2 <= kSplitRingMax; s2 += 128) {
                    LaunchCfg u;
                    if (plan(s2, &u) != cudaSuccess) break;
                    if (u.bps < t.bps) break;
                    grown = s2;
                }
                c->ring_key = key;
                c->ring_S = (int)grown;
            }
            if (c->ring_ok) {
                split_w = W == 0 ? -1 : W;
                split_g = G;
                CK(plan(c->ring_S, &scfg));
            }
        }
    }
    if (split_w) {
        p.fast = 1;
        S = scfg.S;
    } else if (c->window_opt > 0 || c->force_general_s > 0 || no_probe) {
        // forced general path (tests; the device SP2 loop; small matrices: one window of N columns)
        S = c->window_opt > 0 ? c->window_opt : (no_probe ? nr : c->force_general_s);
        p.fast = 0;
    } else if (ring <= kFastWindowMax && groups <= 4) {
        // Grow the ring by slack while the rows resident per SM stay the same: slack lets the
        // emission run in 4-chunk blocks every few steps instead of one chunk per step.
        p.fast = 1;
        const int mode = !has_old ? 0 : (p.normsq ? 2 : 1);
        const int64_t key = (((ring * 8 + groups) * 4 + mode) * 64 + c->warps_opt) * 2;
        if (key != c->ring_key) {
            LaunchCfg t;
            CK(plan_row_op(p, (int)ring, groups, c->warps_opt, c->num_sms, &t));
            // a ring too wide for kFastMinRows rows per SM leaves the SM latency-bound: the
            // general path (1024-double windows, ~16 warps/SM) is faster there (SP2 cfg4 it 1:
            // 2 rows/SM ring 29.7 ms)
            c->ring_ok = t.bps * t.warps_per_cta >= kFastMinRows;
            const int64_t rows0 = (int64_t)t.grid * t.warps_per_cta;  // resident rows (full grid)
            int64_t grown = ring;
            for (int64_t s2 = ring + 32; s2 <= ring + 512 && s2 <= kFastWindowMax && s2 <= nr; s2 += 32) {
                LaunchCfg u;
                if (plan_row_op(p, (int)s2, groups, c->warps_opt, c->num_sms, &u) != cudaSuccess) break;
                if ((int64_t)u.grid * u.warps_per_cta < rows0) break;
                grown = s2;
            }
            c->ring_key = key;
            c->ring_S = (int)grown;
        }
        S = c->ring_S;
        if (!c->ring_ok) {
            S = c->general_s > 0 ? c->general_s : kGeneralWindow;
            p.fast = 0;
        }
    } else {
        S = c->general_s > 0 ? c->general_s : kGeneralWindow;
        p.fast = 0;
    }
    (void)h;
    LaunchCfg cfg;
    if (split_w) {
        cfg = scfg;
    } else {
        if (S > nr) S = nr;
        if (S < 32) S = 32;
        CK(plan_row_op(p, (int)S, groups, c->warps_opt, c->num_sms, &cfg));
    }
    p.S = cfg.S;
    // symmetric SP2 step (f4 ii): a general-path launch computes only the upper triangle, into
    // C_upper; the ring path computes whole rows
    c->last_upper = 0;
    c->sym_nomem = 0;
    if (p.upper) {
        int rc = (p.fast || !alloc_upper) ? ELLPACK_ERR_ARG : alloc_upper(c, alloc_arg, &p.C_upper);
        if (rc == ELLPACK_OK) {
            p.C = p.C_upper;
            c->last_upper = 1;
        } else {
            p.upper = 0;
            if (rc == ELLPACK_ERR_NOMEM) {
                cudaGetLastError();
                c->sym_nomem = 1;  // whole rows this time; the caller stops asking
            } else if (!p.fast) {
                return rc;
            }
        }
    }
    if (split_w) {
        // per-owner bank-balanced copy of B, 16-bit ring byte offsets for this S
        const int rw = split_w < 0 ? 1 : split_w;  // records per B row
        const int64_t k0 = std::max<int64_t>(0, (int64_t)INT_MAX - bwv[5]);
        const int64_t k1 = std::min<int64_t>(n, (int64_t)bwv[6]);
        RK(grow(c, c->bt, (size_t)640 * split_g * rw * n));
        RK(grow(c, c->bt_nbin, sizeof(int32_t) * (size_t)rw * n));
        const int nbal = ex && ex->nbal >= 0 ? ex->nbal : 1;
        for (int q = 0; q < nbal; ++q) {
            const int64_t b0 = ex && ex->nbal >= 0 ? ex->bal[2 * q] : k0;
            const int64_t b1 = ex && ex->nbal >= 0 ? ex->bal[2 * q + 1] : k1;
            CK(launch_balance_split(p.B, b0, b1, rw, split_g, p.S, (unsigned char*)c->bt.p,
                                    (int32_t*)c->bt_nbin.p, c->num_sms, c->stream));
            c->launches++;
        }
        p.bt = (const unsigned char*)c->bt.p;
        p.bt_nbin = (const int32_t*)c->bt_nbin.p;
        p.bt_w = 64 * split_g;
    } else if (p.fast) {
        // bank-balanced copy of B with ring slots precomputed for this S (all N rows: B is the
        // full operand on every rank)
        const int wt = 64 * (groups < 1 ? 1 : groups);
        RK(grow(c, c->bt, (size_t)12 * n * wt));
        RK(grow(c, c->bt_nbin, sizeof(int32_t) * (size_t)n));
        // only the B rows this launch's A rows reference (a rank's block plus its halo; rows a halo
        // exchange did not deliver are never read)
        const int64_t k0 = std::max<int64_t>(0, (int64_t)INT_MAX - bwv[5]);
        const int64_t k1 = std::min<int64_t>(n, (int64_t)bwv[6]);
        const int nbal = ex && ex->nbal >= 0 ? ex->nbal : 1;
        for (int q = 0; q < nbal; ++q) {
            const int64_t b0 = ex && ex->nbal >= 0 ? ex->bal[2 * q] : k0;
            const int64_t b1 = ex && ex->nbal >= 0 ? ex->bal[2 * q + 1] : k1;
            CK(launch_balance(p.B, b0, b1, wt, p.S, (unsigned char*)c->bt.p, (int32_t*)c->bt_nbin.p,
                              c->num_sms, c->stream));
            c->launches++;
        }
        p.bt = (const unsigned char*)c->bt.p;
        p.bt_nbin = (const int32_t*)c->bt_nbin.p;
        p.bt_w = wt;
    } else if (p.S >= n) {
        // one window covers every column: no breakpoints (the kernel takes whole B rows)
        p.bp = nullptr;
        p.bp_np = 0;
    } else {
        // breakpoints of B at the aligned window starts (general path)
        const int np = (int)((n + p.S - 1) / p.S) + 1;
        RK(grow(c, c->bp, sizeof(int32_t) * (size_t)n * np));
        CK(launch_breakpoints(p.B, n, p.S, np, (int32_t*)c->bp.p, c->num_sms, c->stream));
        c->launches++;
        p.bp = (const int32_t*)c->bp.p;
        p.bp_np = np;
    }
    c->last_cfg = cfg;
    c->last_fast = p.fast;
    c->last_split = split_w;
    c->last_hB = (int32_t)hB;
    const int64_t total_warps = (int64_t)cfg.grid * cfg.warps_per_cta;
    const bool may_multi = n > cfg.S;
    p.st_val = nullptr;
    p.st_col = nullptr;
    if (may_multi || p.fast) {
        // in-place rows are stashed on the ring path (progressive emission) and on multi-pass rows
        if (p.stash_a || p.stash_old) {
            p.st_stride = (p.stash_a ? p.A.w : 0) + (p.stash_old ? p.Old.w : 0);
            RK(grow(c, c->stash_val, sizeof(double) * (size_t)total_warps * p.st_stride));
            RK(grow(c, c->stash_col, sizeof(int32_t) * (size_t)total_warps * p.st_stride));
            p.st_val = (double*)c->stash_val.p;
            p.st_col = (int32_t*)c->stash_col.p;
        }
    }
    p.status = c->d_status;
    if (!(ex && ex->keep_status)) CK(cudaMemsetAsync(c->d_status, 0, 2 * sizeof(int32_t), c->stream));
    p.row_ticket = c->d_keys + 3;  // d_keys[3]: the fast kernel's row counter
    {
        // rows per ticket: 4 (fewer atomics, neighbouring rows share B records in L2) unless the
        // launch has fewer than 64 rows per resident warp, where one-row tickets keep the tail short
        const int64_t rows = p.row_end - p.row_begin;
        const int64_t in_flight = split_w ? (int64_t)cfg.grid : total_warps;  // rows being worked on
        p.row_chunk = rows >= 64 * in_flight ? ELL_ROW_CHUNK : 1;
    }
    CK(cudaMemsetAsync(p.row_ticket, 0, 8, c->stream));
    const int pk = c->prof_n < 4 ? c->prof_n : 3;
    if (c->profile) CK(cudaEventRecord(c->pev[pk][0], c->stream));
    if (split_w < 0) CK(launch_ws(p, cfg, c->stream));
    else if (split_w) CK(launch_split(p, cfg, c->stream));
    else CK(launch_row_op(p, cfg, c->stream));
    if (c->profile) {
        CK(cudaEventRecord(c->pev[pk][1], c->stream));
        c->prof_n = pk + 1;
        c->prof_pending = true;
    }
    c->launches++;
    return ELLPACK_OK;
}

// called after a stream sync: fold the pending row-kernel event pair into the profile
void prof_collect(ellpack_ctx c) {
    if (!c->prof_pending) return;
    float ms = 0.f;
    for (int q = 0; q < c->prof_n; ++q) {
        if (cudaEventElapsedTime(&ms, c->pev[q][0], c->pev[q][1]) == cudaSuccess) c->prof_ms += ms;
    }
    c->prof_n = 0;
    {
        c->prof_launches++;  // one multiply (its row-kernel launches summed)
    }
    c->prof_pending = false;
}

// Canonical sums of `narr` per-row arrays over all n rows (partials exchanged over ranks).
int enqueue_canonical(ellpack_ctx c, const double* const* arrays, int narr, int64_t n) {
    int64_t r0, r1;
    rows_of(c, n, &r0, &r1);
    const int64_t nb = (n + kTraceBlock - 1) / kTraceBlock;
    if (!c->comm && nb * narr <= 16) {  // small: both levels in one launch
        CK(launch_canonical_small(arrays, narr, n, c->d_sums, c->stream));
        c->launches++;
        return ELLPACK_OK;
    }
    RK(grow(c, c->partials, sizeof(double) * (size_t)nb * narr));
    double* part = (double*)c->partials.p;
    CK(launch_block_partials(arrays, narr, r0, r1, n, part, c->stream));
    c->launches++;
    if (c->comm) {
        const int64_t per = (r1 - r0) / kTraceBlock;  // equal 256-aligned blocks (checked at attach)
        NK(g_nccl.GroupStart());
        for (int a = 0; a < narr; ++a) {
            double* base = part + (size_t)a * nb;
            NK(g_nccl.AllGather(base + (size_t)c->rank * per, base, (size_t)per, ncclFloat64, c->comm,
                                c->stream));
        }
        NK(g_nccl.GroupEnd());
    }
    CK(launch_final_sums(part, narr, nb, c->d_sums, c->stream));
    c->launches++;
    return ELLPACK_OK;
}

// ---- dense regime (dense.cu): S = A B as a dense FP64 GEMM, then the row epilogue
constexpr int64_t kDenseMaxN = 65536;

int64_t dense_np(int64_t n) { return (n + kDenseTile - 1) / kDenseTile * kDenseTile; }

// can this context run a dense step of dimension n (buffers for `bufs` np x np arrays)?
bool dense_fits(ellpack_ctx c, int64_t n, int bufs) {
    if (c->comm || c->dense_opt == 1 || n > kDenseMaxN || n <= 0) return false;
    const int64_t np = dense_np(n);
    const double one = 8.0 * (double)np * (double)np;
    // the arrays this step uses (dense[0] X or B, dense[2] S, dense[1] A^T when not symmetric) that
    // are not already large enough: only then ask the driver for free memory (cudaMemGetInfo costs
    // milliseconds)
    double need = 0.0;
    for (int b : {0, 2, 1}) {
        if (b == 1 && bufs < 3) break;
        if ((double)c->dense[b].bytes < one) need += one;
    }
    if (need == 0.0) return true;
    // one driver query per (N_p, arrays) until the context's dense arrays change (sp2_run resets it)
    const int64_t key = np * 4 + bufs;
    if (c->dense_fit_key == key) return c->dense_fit_ok;
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); return false; }
    if (need > 0.6 * (double)fr) {
        // memory freed with cudaFreeAsync (an earlier context's dense arrays) stays in the device's
        // default pool until trimmed: return it and ask again
        cudaMemPool_t pool;
        if (cudaStreamSynchronize(c->stream) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, c->device) == cudaSuccess &&
            cudaMemPoolTrimTo(pool, 0) == cudaSuccess && cudaMemGetInfo(&fr, &tot) != cudaSuccess)
            fr = 0;
        cudaGetLastError();
    }
    c->dense_fit_key = key;
    c->dense_fit_ok = need <= 0.6 * (double)fr;
    if (getenv("ELLPACK_DEBUG_REGIME"))
        fprintf(stderr, "[regime] dense arrays %.2f GB, free %.2f GB -> %s\n", need * 1e-9, (double)fr * 1e-9,
                c->dense_fit_ok ? "fit" : "do not fit");
    return c->dense_fit_ok;
}

// FMAs the symmetric dense GEMM runs on X^2 for X of half-bandwidth h (every 128 x 16 block within
// the band counted as occupied: an upper bound of the flags' count), the model the regime choice
// times with the measured dense rate.
double dense_band_fmas(int64_t n, int64_t h, bool sym) {
    const int64_t np = dense_np(n), T = np / kDenseTile;
    double blocks = 0.0;
    for (int64_t bi = 0; bi < T; ++bi) {
        const int64_t rlo = std::max<int64_t>(0, bi * kDenseTile - h);
        const int64_t rhi = std::min<int64_t>(n - 1, bi * kDenseTile + kDenseTile - 1 + h);
        for (int64_t bj = sym ? bi : 0; bj < T; ++bj) {
            const int64_t clo = std::max<int64_t>(0, bj * kDenseTile - h);
            const int64_t chi = std::min<int64_t>(n - 1, bj * kDenseTile + kDenseTile - 1 + h);
            const int64_t lo = std::max(rlo, clo), hi = std::min(rhi, chi);
            if (lo > hi) {
                if (bj * kDenseTile > bi * kDenseTile + 2 * h + kDenseTile) break;  // past the band
                continue;
            }
            blocks += (double)(hi / kDenseK - lo / kDenseK + 1);
        }
    }
    return blocks * kDenseK * kDenseTile * kDenseTile;
}

// p as for enqueue_row_op (A, B, Old, C, alpha, beta, old_mode, tau, diagonals, norm, exec_products);
// C must not alias A, B or Old; Old (when old_mode != 0) must be B. sym: A = B and bitwise
// symmetric (one dense array, half the tiles).
int enqueue_dense_op(ellpack_ctx c, RowOpParams& p, int64_t n, bool sym, const int32_t* bwv = nullptr,
                     bool halo = false) {
    // the dense regime computes X X (A = B; Old, when present, is X too)
    if (p.A.val != p.B.val || p.A.col != p.B.col || p.A.nnz != p.B.nnz) return ELLPACK_ERR_ARG;
    if (p.old_mode != 0 && (p.Old.val != p.B.val || p.Old.col != p.B.col || p.Old.nnz != p.B.nnz))
        return ELLPACK_ERR_ARG;
    p.ncols = n;
    const int64_t np = dense_np(n);
    const size_t bytes = sizeof(double) * (size_t)np * (size_t)np;
    const int64_t T = np / kDenseTile, KB = np / kDenseK;
    // a rank's row block (communicator): S rows [r0, r1) from the X rows they reference -- its own
    // and the halo rows [k0, k1) the probe's reach names (symmetric X: X^T = X, one dense copy)
    const int64_t r0 = p.row_begin, r1 = p.row_end;
    const bool part = r0 != 0 || r1 != n;
    if (part && (!sym || r0 % kDenseTile || (r1 - r0) % kDenseTile)) return ELLPACK_ERR_ARG;
    int64_t x0 = 0, x1 = n;  // rows of X densified (without a probe: every row is local)
    if (part && bwv) {
        x0 = std::min<int64_t>(r0, std::max<int64_t>(0, (int64_t)INT_MAX - bwv[5]));
        x1 = std::max<int64_t>(r1, std::min<int64_t>(n, (int64_t)bwv[6]));
    }
    // ELLPACK_OPT_SP2_MEM_CAP fault injection: the dense arrays "do not fit" either
    if (c->sp2_mem_cap > 0 && (int64_t)(2 * bytes) > c->sp2_mem_cap) return ELLPACK_ERR_NOMEM;
    const void* d0 = c->dense[0].p;
    const void* f0 = c->dflags.p;
    RK(grow(c, c->dense[0], bytes));
    RK(grow(c, c->dense[2], bytes));
    if (!sym) RK(grow(c, c->dense[1], bytes));
    const size_t fbytes = 2 * (size_t)T * KB;                      // fa | fb (bytes)
    const size_t bbytes = 2 * (size_t)T * dense_kbw((int)np) * 8;   // Fa | Fb (bitsets)
    const size_t tbytes = (size_t)(np / 16) * T;                    // tw (16-row tiles at most)
    RK(grow(c, c->dflags, fbytes + bbytes + tbytes));
    if (c->dense[0].p != d0 || c->dflags.p != f0) c->dense_clean_np = 0;  // reallocated: contents unknown
    unsigned char* fa = (unsigned char*)c->dflags.p;
    unsigned char* fb = fa + (size_t)T * KB;
    unsigned long long* Fa = (unsigned long long*)(fa + fbytes);
    unsigned long long* Fb = Fa + (size_t)T * dense_kbw((int)np);
    unsigned char* tw = fa + fbytes + bbytes;
    double* D = (double*)c->dense[0].p;                    // X (row-major): B, Old
    double* Dt = sym ? D : (double*)c->dense[1].p;         // X^T: A
    double* S = (double*)c->dense[2].p;
    // D is zero outside the blocks fa flags (the last densify's) when dense_clean_np == np: clearing
    // those costs the previous iterate's band instead of N^2
    c->dense_full_clear = c->dense_clean_np != np;
    if (!c->dense_full_clear) {
        CK(launch_dense_clear(D, (int)np, fa, c->num_sms, c->stream));
        c->launches++;
    } else {
        CK(cudaMemsetAsync(D, 0, bytes, c->stream));
    }
    CK(cudaMemsetAsync(c->dflags.p, 0, fbytes, c->stream));
    if (!sym) CK(cudaMemsetAsync(Dt, 0, bytes, c->stream));
    if (halo) CK(cudaStreamWaitEvent(c->stream, c->sev[1], 0));  // the halo rows of X_n have landed
    if (sym) {
        CK(launch_densify(p.B, x0, x1, (int)np, false, D, fa, fb, c->stream));
        c->launches++;
    } else {
        CK(launch_densify(p.A, 0, n, (int)np, true, Dt, fa, nullptr, c->stream));
        CK(launch_densify(p.B, 0, n, (int)np, false, D, nullptr, fb, c->stream));
        c->launches += 2;
    }
    c->dense_clean_np = np;  // D = X, nonzero only in fa's blocks (A = B = X)
    CK(launch_pack_flags(fa, fb, (int)np, Fa, Fb, c->num_sms, c->stream));
    c->launches++;
    // ELLPACK_OPT_PROFILE: the GEMM is this op's "row kernel" (ellpack_ctx_kernel_time)
    const int pk = c->prof_n < 4 ? c->prof_n : 3;
    if (c->profile) CK(cudaEventRecord(c->pev[pk][0], c->stream));
    const bool sym_tiles = sym && !part;
    const int64_t g0 = part ? r0 : 0, g1 = part ? r1 : np;
    const int bm = dense_tile_rows((int)np, g1 - g0, sym_tiles, c->num_sms);
    const bool mma = c->dense_kernel == 2 || (c->dense_kernel == 0 && dense_mma_ok(c->stream));
    CK(launch_dense_gemm(Dt, D, (int)np, sym_tiles, Fa, Fb, S, tw, p.exec_products, g0, g1, bm, mma, c->stream));
    if (c->profile) {
        CK(cudaEventRecord(c->pev[pk][1], c->stream));
        c->prof_n = pk + 1;
        c->prof_pending = true;
    }
    c->launches++;
    p.status = c->d_status;
    CK(cudaMemsetAsync(c->d_status, 0, 2 * sizeof(int32_t), c->stream));
    // stored a_ii of A: the diagonal of either dense copy of A; Old = X: its dense copy D and flags fa
    const double* dA = sym ? D : Dt;
    CK(launch_dense_emit(S, (int)np, p, dA, p.old_mode != 0 ? D : nullptr, tw,
                         bm, Fa, c->num_sms, c->stream));
    c->launches++;
    c->last_upper = 0;
    c->last_dense = 1;
    c->last_small = 0;
    p.fast = 0;
    return ELLPACK_OK;
}

// One read-back: status, `nsums` canonical sums and, with probe, the bandwidth probe d_bw[0..5]
// (+ every rank's reach with a communicator); then the one host synchronisation.
int fetch_copies(ellpack_ctx c, int nsums) {
    CK(cudaMemcpyAsync(c->h->status, c->d_status, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    if (nsums > 0)
        CK(cudaMemcpyAsync(c->h->sums, c->d_sums, nsums * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    return ELLPACK_OK;
}

int fetch(ellpack_ctx c, int nsums, bool probe = false) {
    RK(fetch_copies(c, nsums));
    if (probe) {
        CK(cudaMemcpyAsync(c->h->bw, c->d_bw, kProbe * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
        if (c->comm)
            CK(cudaMemcpyAsync(c->h_reach, c->halo.p, 2 * sizeof(int32_t) * c->nranks, cudaMemcpyDeviceToHost,
                               c->stream));
    }
    RK(host_sync(c));
    prof_collect(c);
    return ELLPACK_OK;
}

int finish_status(ellpack_ctx c) {
    if (c->h->status[0] > 0) {
        c->last_ovf_rows = c->h->status[0];
        c->last_req = c->h->status[1];
        return ELLPACK_ERR_OVERFLOW;
    }
    return ELLPACK_OK;
}

RowOpParams base_params(ellpack_ctx c, int64_t n) {
    RowOpParams p;
    memset(&p, 0, sizeof p);
    rows_of(c, n, &p.row_begin, &p.row_end);
    return p;
}

int allgather_desc(ellpack_ctx c, const ellpack_desc* m) {
    if (!c->comm) return ELLPACK_OK;
    int64_t r0, r1;
    rows_of(c, m->n, &r0, &r1);
    const size_t per = (size_t)(r1 - r0);
    const size_t w = (size_t)m->w;
    NK(g_nccl.GroupStart());
    NK(g_nccl.AllGather(m->val + (size_t)r0 * w, m->val, per * w, ncclFloat64, c->comm, c->stream));
    NK(g_nccl.AllGather(m->col + (size_t)r0 * w, m->col, per * w, ncclInt32, c->comm, c->stream));
    NK(g_nccl.AllGather(m->nnz + r0, m->nnz, per, ncclInt32, c->comm, c->stream));
    NK(g_nccl.GroupEnd());
    return ELLPACK_OK;
}

// Band-aware halo exchange (§8f-f1): this rank's rows of `a` reference B rows [lo, hi]; the
// ranges of all ranks are all-gathered (16 bytes each), then every rank sends the part of its own
// block of `b` each peer reads and receives the parts of the peers' blocks it reads (NCCL
// point-to-point in one group; the plan is ellpack_halo_plan, identical on both sides of a pair).
// The send/recv half of the halo exchange, from every rank's referenced rows need[2q..2q+1]
// (host values, inclusive; need[2q] > need[2q+1] = none). Enqueue only: no host wait.
int halo_exec(ellpack_ctx c, ellpack_desc* b, const int64_t* need) {
    const int64_t n = b->n;
    int64_t r0, r1;
    rows_of(c, n, &r0, &r1);
    const int P = c->nranks;
    std::vector<int64_t> snd(3 * (size_t)P), rcv(3 * (size_t)P);
    int32_t ns = 0, nr = 0;
    RK(ellpack_halo_plan(n, P, c->rank, r1 - r0, need, &ns, snd.data(), &nr, rcv.data()));
    const size_t w = (size_t)b->w;
    NK(g_nccl.GroupStart());
    for (int q = 0; q < ns; ++q) {
        const int peer = (int)snd[3 * q];
        const size_t s0 = (size_t)snd[3 * q + 1], cnt = (size_t)(snd[3 * q + 2] - snd[3 * q + 1]);
        NK(g_nccl.Send(b->val + s0 * w, cnt * w, ncclFloat64, peer, c->comm, c->stream));
        NK(g_nccl.Send(b->col + s0 * w, cnt * w, ncclInt32, peer, c->comm, c->stream));
        NK(g_nccl.Send(b->nnz + s0, cnt, ncclInt32, peer, c->comm, c->stream));
    }
    for (int q = 0; q < nr; ++q) {
        const int peer = (int)rcv[3 * q];
        const size_t t0 = (size_t)rcv[3 * q + 1], cnt = (size_t)(rcv[3 * q + 2] - rcv[3 * q + 1]);
        NK(g_nccl.Recv(b->val + t0 * w, cnt * w, ncclFloat64, peer, c->comm, c->stream));
        NK(g_nccl.Recv(b->col + t0 * w, cnt * w, ncclInt32, peer, c->comm, c->stream));
        NK(g_nccl.Recv(b->nnz + t0, cnt, ncclInt32, peer, c->comm, c->stream));
    }
    NK(g_nccl.GroupEnd());
    return ELLPACK_OK;
}

int halo_desc(ellpack_ctx c, const ellpack_desc* a, ellpack_desc* b) {
    if (!c->comm) return ELLPACK_OK;
    const int64_t n = b->n;
    int64_t r0, r1;
    rows_of(c, n, &r0, &r1);
    const int P = c->nranks;
    RK(grow(c, c->halo, sizeof(long long) * 2 * (size_t)P));
    long long* d_need = (long long*)c->halo.p;
    long long* mine = d_need + 2 * c->rank;
    const long long init[2] = {LLONG_MAX, -1};
    CK(cudaMemcpyAsync(mine, init, sizeof init, cudaMemcpyHostToDevice, c->stream));
    CK(launch_col_range(kmat(a), r0, r1, mine, c->stream));
    c->launches++;
    NK(g_nccl.AllGather(mine, d_need, 2, ncclInt64, c->comm, c->stream));
    std::vector<long long> need(2 * (size_t)P);
    CK(cudaMemcpyAsync(need.data(), d_need, sizeof(long long) * 2 * P, cudaMemcpyDeviceToHost, c->stream));
    RK(host_sync(c));
    std::vector<int64_t> needl(need.begin(), need.end());
    return halo_exec(c, b, needl.data());
}

// The halo of `b` (need: every rank's referenced rows) sent and received on the side stream, after
// everything already on the context stream; sev[1] marks its completion. With a communicator only.
int start_halo(ellpack_ctx c, ellpack_desc* b, const int64_t* need) {
    if (!c->side) {
        CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->sev[0], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->sev[1], cudaEventDisableTiming));
    }
    CK(cudaEventRecord(c->sev[0], c->stream));
    CK(cudaStreamWaitEvent(c->side, c->sev[0], 0));
    cudaStream_t main = c->stream;
    c->stream = c->side;
    const int rc = halo_exec(c, b, need);
    c->stream = main;
    RK(rc);
    CK(cudaEventRecord(c->sev[1], c->side));
    return ELLPACK_OK;
}

// One row op over this rank's rows [r0, r1) in up to three launches (§8f-f1): the interior rows --
// [r0 + h, r1 - h), h = the all-reduced half-bandwidth of A (bwv[0]), whose B rows are all the
// rank's own -- first; then, once the halo started by start_halo is in (halo = true: the context
// stream waits for sev[1]), the boundary rows [r0, r0 + h) and [r1 - h, r1). The balance pass of
// the ring paths prepares the own B rows for the interior launch and the halo rows for the
// boundary ones; the status block accumulates over the launches.
int enqueue_row_op_split(ellpack_ctx c, RowOpParams& p, int64_t n, const int32_t* bwv, bool halo,
                         int (*alloc_upper)(ellpack_ctx, void*, KOut*) = nullptr, void* alloc_arg = nullptr) {
    bool upper = false;
    const int64_t r0 = p.row_begin, r1 = p.row_end;
    int64_t sp[6];
    RK(ellpack_row_split(r0, r1, bwv[0], sp));
    const int64_t k0 = std::max<int64_t>(0, (int64_t)INT_MAX - bwv[5]);
    const int64_t k1 = std::min<int64_t>(n, (int64_t)bwv[6]);
    bool any = false;
    if (sp[0] < sp[1]) {
        RowOpParams q = p;
        q.row_begin = sp[0];
        q.row_end = sp[1];
        RowOpExtra ex;
        ex.nbal = 1;
        ex.bal[0] = std::max(k0, r0);
        ex.bal[1] = std::max(ex.bal[0], std::min(k1, r1));
        RK(enqueue_row_op(c, q, n, bwv, alloc_upper, alloc_arg, &ex));
        p.fast = q.fast;
        upper = upper || c->last_upper;
        any = true;
    }
    if (halo) CK(cudaStreamWaitEvent(c->stream, c->sev[1], 0));
    bool halo_balanced = false;
    for (int b = 0; b < 2; ++b) {
        const int64_t b0 = sp[2 + 2 * b], b1 = sp[3 + 2 * b];
        if (b0 >= b1) continue;
        RowOpParams q = p;
        q.row_begin = b0;
        q.row_end = b1;
        RowOpExtra ex;
        ex.keep_status = any;
        if (!any) {  // nothing balanced yet: every referenced row
            ex.nbal = 1;
            ex.bal[0] = k0;
            ex.bal[1] = k1;
        } else if (!halo_balanced) {  // the halo rows, once
            ex.nbal = 2;
            ex.bal[0] = k0;
            ex.bal[1] = std::max(k0, std::min(k1, r0));
            ex.bal[2] = std::min(k1, std::max(k0, r1));
            ex.bal[3] = k1;
        } else {
            ex.nbal = 0;
        }
        RK(enqueue_row_op(c, q, n, bwv, alloc_upper, alloc_arg, &ex));
        p.fast = q.fast;
        upper = upper || c->last_upper;
        any = true;
        halo_balanced = true;
    }
    if (!any) CK(cudaMemsetAsync(c->d_status, 0, 2 * sizeof(int32_t), c->stream));
    c->last_upper = upper;  // every launch takes the same route (one plan)
    return ELLPACK_OK;
}

}  // namespace

// =========================================================================== ABI

extern "C" {

const char* ellpack_strerror(int s) {
    switch (s) {
        case ELLPACK_OK: return "ok";
        case ELLPACK_ERR_ARG: return "invalid argument";
        case ELLPACK_ERR_DIM: return "dimension mismatch";
        case ELLPACK_ERR_OVERFLOW: return "output row exceeds ELLPACK width";
        case ELLPACK_ERR_BOUNDS: return "degenerate spectral bounds";
        case ELLPACK_ERR_NOCONV: return "SP2 did not converge within max_iter";
        case ELLPACK_ERR_NOMEM: return "device allocation failed";
        case ELLPACK_ERR_CUDA: return "CUDA error";
        case ELLPACK_ERR_NCCL: return "NCCL error";
        case ELLPACK_ERR_STATE: return "invalid context state";
        default: return "unknown status";
    }
}

int ellpack_ctx_create(int device, void* stream, ellpack_ctx* out) {
    if (!out) return ELLPACK_ERR_ARG;
    *out = nullptr;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return ELLPACK_ERR_ARG;
    CK(cudaSetDevice(device));
    ellpack_ctx c = new (std::nothrow) ellpack_ctx_s();
    if (!c) return ELLPACK_ERR_NOMEM;
    c->device = device;
    c->stream = (cudaStream_t)stream;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    {
        // keep freed stream-ordered allocations in the device pool: SP2 re-creates iterates of
        // growing width every few iterations, and returning them to the driver at each sync
        // costs milliseconds per GB
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    cudaError_t e = cudaMalloc(&c->d_status, 64);
    if (!e) e = cudaMalloc(&c->d_keys, 64);
    if (!e) e = cudaMalloc(&c->d_sums, 64);
    if (!e) e = cudaMalloc(&c->d_bw, 64);
    if (!e) e = cudaMallocHost(&c->h, sizeof(ellpack_ctx_s::Host));
    if (!e) {  // the device's view of the pinned block: the small-matrix kernel writes its status and
               // sums there directly (no read-back copies); null when the device cannot map it
        void* hd = nullptr;
        if (cudaHostGetDevicePointer(&hd, c->h, 0) == cudaSuccess) c->h_dev = (ellpack_ctx_s::Host*)hd;
        cudaGetLastError();
    }
    for (int k = 0; k < 6 && !e; ++k) e = cudaEventCreate(&c->ev[k]);
    for (int k = 0; k < 4 && !e; ++k) {
        e = cudaEventCreate(&c->pev[k][0]);
        if (!e) e = cudaEventCreate(&c->pev[k][1]);
    }
    if (e) { ellpack_ctx_destroy(c); return from_cuda(e); }
    *out = c;
    return ELLPACK_OK;
}

int ellpack_ctx_destroy(ellpack_ctx c) {
    if (!c) return ELLPACK_ERR_ARG;
    cudaSetDevice(c->device);
    Buf* bufs[] = {&c->rows[0], &c->rows[1], &c->rows[2], &c->rows[3], &c->partials,
                   &c->stash_val, &c->stash_col, &c->ident_val, &c->ident_col, &c->ident_nnz,
                   &c->hx_val, &c->hx_col, &c->hx_nnz, &c->hy_val, &c->hy_col, &c->hy_nnz,
                   &c->bt, &c->bt_nbin, &c->bp, &c->halo, &c->vflag, &c->symaux, &c->sp2dev, &c->sp2rec, &c->tiny,
                   &c->dense[0], &c->dense[1], &c->dense[2], &c->dflags, &c->docc,
                   &c->old_val, &c->old_col, &c->old_nnz};
    if (c->sp2_exec) cudaGraphExecDestroy(c->sp2_exec);
    if (c->x2_exec) cudaGraphExecDestroy(c->x2_exec);
    for (auto& sl : c->it)
        for (Buf& b : sl) release(c, b);
    for (Buf* b : bufs) release(c, *b);
    cudaStreamSynchronize(c->stream);
    {
        // hand the freed workspace (up to two 34 GB dense arrays) back to the device, not to the pool
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, c->device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
        cudaGetLastError();
    }
    if (c->comm && g_nccl.ok) g_nccl.CommDestroy(c->comm);
    cudaFree(c->d_status);
    cudaFree(c->d_keys);
    cudaFree(c->d_sums);
    cudaFree(c->d_bw);
    if (c->h) cudaFreeHost(c->h);
    if (c->h_reach) cudaFreeHost(c->h_reach);
    for (int k = 0; k < 6; ++k) if (c->ev[k]) cudaEventDestroy(c->ev[k]);
    for (int k = 0; k < 4; ++k)
        for (int q = 0; q < 2; ++q) if (c->pev[k][q]) cudaEventDestroy(c->pev[k][q]);
    for (int q = 0; q < 2; ++q) if (c->sev[q]) cudaEventDestroy(c->sev[q]);
    if (c->side) cudaStreamDestroy(c->side);
    delete c;
    return ELLPACK_OK;
}

int ellpack_ctx_set_stream(ellpack_ctx c, void* stream) {
    if (!c) return ELLPACK_ERR_ARG;
    c->stream = (cudaStream_t)stream;
    return ELLPACK_OK;
}

int ellpack_ctx_set_option(ellpack_ctx c, int key, int64_t v) {
    if (!c || v < 0) return ELLPACK_ERR_ARG;
    c->x2_exec_ok = false;
    switch (key) {
        case ELLPACK_OPT_WINDOW: c->window_opt = (int)v; return ELLPACK_OK;
        case ELLPACK_OPT_VALIDATE: c->validate = v != 0; return ELLPACK_OK;
        case ELLPACK_OPT_SP2_SYMMETRIC: c->sp2_sym = v != 0; return ELLPACK_OK;
        case ELLPACK_OPT_WARPS: c->warps_opt = (int)v; return ELLPACK_OK;
        case ELLPACK_OPT_SP2_WIDTH0: c->sp2_width0 = (int)v; return ELLPACK_OK;
        case ELLPACK_OPT_SP2_MEM_CAP: c->sp2_mem_cap = v; return ELLPACK_OK;
        case ELLPACK_OPT_SP2_DEVICE_LOOP:
            if (v > 2) return ELLPACK_ERR_ARG;
            c->sp2_loop = (int)v;
            return ELLPACK_OK;
        case ELLPACK_OPT_DENSE:
            if (v > 2) return ELLPACK_ERR_ARG;
            c->dense_opt = (int)v;
            return ELLPACK_OK;
        case ELLPACK_OPT_DENSE_KERNEL:
            if (v > 2) return ELLPACK_ERR_ARG;
            c->dense_kernel = (int)v;
            return ELLPACK_OK;
        case ELLPACK_OPT_SMALL_KERNEL:
            if (v > 1) return ELLPACK_ERR_ARG;
            c->small_kernel = (int)v;
            return ELLPACK_OK;
        case ELLPACK_OPT_RING_KERNEL:
            if (v > 4) return ELLPACK_ERR_ARG;
            c->ring_kernel = (int)v;
            c->ring_key = -1;
            return ELLPACK_OK;
        case ELLPACK_OPT_ABLATE:
#if defined(ELL_ABLATE) && ELL_ABLATE
            c->ablate = (int)v;
            return ELLPACK_OK;
#else
            return v == 0 ? ELLPACK_OK : ELLPACK_ERR_ARG;  // experiments not compiled in
#endif
        case ELLPACK_OPT_GENERAL_WINDOW:
            if (v < 0 || v > kFastWindowMax || (v & 31)) return ELLPACK_ERR_ARG;
            c->general_s = (int)v;
            return ELLPACK_OK;
        case ELLPACK_OPT_PROFILE:
            c->profile = v != 0;
            c->prof_ms = 0.0;
            c->prof_launches = 0;
            c->prof_pending = false;
            c->prof_n = 0;
            return ELLPACK_OK;
        default: return ELLPACK_ERR_ARG;
    }
}

int64_t ellpack_ctx_kernel_launches(ellpack_ctx c) { return c ? c->launches : -1; }

int64_t ellpack_ctx_host_syncs(ellpack_ctx c) { return c ? c->host_syncs : -1; }

int ellpack_ctx_last_launch(ellpack_ctx c, int32_t out[8]) {
    if (!c || !out) return ELLPACK_ERR_ARG;
    const LaunchCfg& g = c->last_cfg;
    out[0] = c->last_fast;
    out[1] = g.R;
    out[2] = g.S;
    out[3] = g.warps_per_cta;
    out[4] = g.grid;
    out[5] = (int32_t)g.smem;
    out[6] = g.bps;
    out[7] = c->last_hB;
    // 3: warp-specialized ring kernel, 2: split-row ring kernel (out[3] = W warps per row)
    out[0] = c->last_split < 0 ? 3 : (c->last_split ? 2 : c->last_fast);
    if (c->last_dense) out[0] = 4;  // dense regime (dense.cu): out[1..7] describe no row kernel
    if (c->last_small) out[0] = 5;  // small-matrix kernel (tiny.cu)
    return ELLPACK_OK;
}

int ellpack_ctx_kernel_time(ellpack_ctx c, double* ms, int64_t* launches) {
    if (!c) return ELLPACK_ERR_ARG;
    if (ms) *ms = c->prof_ms;
    if (launches) *launches = c->prof_launches;
    return ELLPACK_OK;
}

int ellpack_ctx_set_rows(ellpack_ctx c, int64_t r0, int64_t r1) {
    if (!c || r0 < 0 || (r1 >= 0 && r1 < r0)) return ELLPACK_ERR_ARG;
    if (c->comm) return ELLPACK_ERR_STATE;
    c->row_begin = r0;
    c->row_end = r1;
    return ELLPACK_OK;
}

int ellpack_create(ellpack_ctx c, int64_t n, int32_t m, ellpack_desc* out) {
    if (!c || !out || n <= 0 || n > INT32_MAX || m <= 0 || (m & 1)) return ELLPACK_ERR_ARG;
    CK(cudaSetDevice(c->device));
    ellpack_desc d{};
    d.n = n;
    d.w = m;
    const size_t cells = (size_t)n * (size_t)m;
    cudaError_t e = cudaMallocAsync((void**)&d.val, cells * sizeof(double), c->stream);
    if (!e) e = cudaMallocAsync((void**)&d.col, cells * sizeof(int32_t), c->stream);
    if (!e) e = cudaMallocAsync((void**)&d.nnz, (size_t)n * sizeof(int32_t), c->stream);
    if (!e) e = cudaMemsetAsync(d.nnz, 0, (size_t)n * sizeof(int32_t), c->stream);
    if (!e) e = cudaMemsetAsync(d.val, 0, cells * sizeof(double), c->stream);
    if (!e) e = cudaMemsetAsync(d.col, 0, cells * sizeof(int32_t), c->stream);
    if (e) {
        if (d.val) cudaFreeAsync(d.val, c->stream);
        if (d.col) cudaFreeAsync(d.col, c->stream);
        if (d.nnz) cudaFreeAsync(d.nnz, c->stream);
        return from_cuda(e);
    }
    *out = d;
    return ELLPACK_OK;
}

int ellpack_destroy(ellpack_ctx c, ellpack_desc* d) {
    if (!c || !d) return ELLPACK_ERR_ARG;
    if (d->val) cudaFreeAsync(d->val, c->stream);
    if (d->col) cudaFreeAsync(d->col, c->stream);
    if (d->nnz) cudaFreeAsync(d->nnz, c->stream);
    memset(d, 0, sizeof *d);
    return ELLPACK_OK;
}

int ellpack_overflow_info(ellpack_ctx c, int64_t* rows, int32_t* req) {
    if (!c) return ELLPACK_ERR_ARG;
    if (rows) *rows = c->last_ovf_rows;
    if (req) *req = c->last_req;
    return ELLPACK_OK;
}

int ellpack_multiply(ellpack_ctx c, const ellpack_desc* a, const ellpack_desc* b, ellpack_desc* cm,
                     double alpha, double beta, double tau) {
    if (!c) return ELLPACK_ERR_ARG;
    RK(check_desc(a));
    RK(check_desc(b));
    RK(check_desc(cm));
    if (a->n != b->n || a->n != cm->n) return ELLPACK_ERR_DIM;
    RK(check_comm_n(c, a->n));
    if (!valid_tau(tau) || !std::isfinite(alpha) || !std::isfinite(beta)) return ELLPACK_ERR_ARG;
    if (same(cm, a) || same(cm, b)) return ELLPACK_ERR_ARG;
    NvtxRange nv("ellpack_multiply");
    CK(cudaSetDevice(c->device));
    if (beta != 0.0) RK(validate_inputs(c, {a, b, cm})); else RK(validate_inputs(c, {a, b}));
    RowOpParams p = base_params(c, a->n);
    p.A = kmat(a);
    p.B = kmat(b);
    p.C = kout(cm);
    p.alpha = alpha;
    p.beta = beta;
    p.tau = tau;
    if (beta != 0.0) {
        p.old_mode = 1;
        // C_old is C itself (updated in place): its live entries go to a scratch copy first (one
        // kernel, 12 B per live entry), so the row kernels read Old from memory the output never
        // overwrites -- the split ring kernel then applies (it does not stash aliased rows)
        const int64_t nn = a->n;
        RK(grow(c, c->old_val, sizeof(double) * (size_t)nn * cm->w));
        RK(grow(c, c->old_col, sizeof(int32_t) * (size_t)nn * cm->w));
        RK(grow(c, c->old_nnz, sizeof(int32_t) * (size_t)nn));
        KOut oc{(double*)c->old_val.p, (int32_t*)c->old_col.p, (int32_t*)c->old_nnz.p, cm->w};
        CK(launch_copy_rows(kmat(cm), oc, p.row_begin, p.row_end, c->d_status + 4, c->stream));
        c->launches++;
        p.Old = KMat{oc.val, oc.col, oc.nnz, oc.w};
        p.stash_old = 0;
    }
    RK(enqueue_row_op(c, p, a->n));
    RK(reduce_status(c));
    RK(fetch(c, 0));
    return finish_status(c);
}

int ellpack_multiply_x2(ellpack_ctx c, const ellpack_desc* x, ellpack_desc* x2, double tau,
                        double* trace_x, double* trace_x2) {
    if (!c) return ELLPACK_ERR_ARG;
    RK(check_desc(x));
    RK(check_desc(x2));
    if (x->n != x2->n) return ELLPACK_ERR_DIM;
    RK(check_comm_n(c, x->n));
    if (!valid_tau(tau)) return ELLPACK_ERR_ARG;
    if (same(x, x2)) return ELLPACK_ERR_ARG;
    NvtxRange nv("ellpack_multiply_x2 (SP2 Loop X2)");
    CK(cudaSetDevice(c->device));
    RK(validate_inputs(c, {x}));
    const int64_t n = x->n;
    RK(grow(c, c->rows[0], sizeof(double) * n));
    RK(grow(c, c->rows[1], sizeof(double) * n));
    RowOpParams p = base_params(c, n);
    p.A = kmat(x);
    p.B = kmat(x);
    p.C = kout(x2);
    p.alpha = 1.0;
    p.beta = 0.0;
    p.tau = tau;
    p.diag_a = (double*)c->rows[0].p;
    p.diag_s = (double*)c->rows[1].p;
    // forced dense regime (ELLPACK_OPT_DENSE 2): X's symmetry decides one or two dense copies
    int dense_sym = -1;
    if (c->dense_opt == 2 && dense_fits(c, n, 3)) {
        RK(grow(c, c->symaux, 4 * sizeof(int32_t)));
        int32_t* aux = (int32_t*)c->symaux.p;
        CK(cudaMemsetAsync(aux, 0, sizeof(int32_t), c->stream));
        CK(launch_sym_check(kmat(x), 0, n, aux, c->stream));
        c->launches++;
        int32_t asym = 1;
        CK(cudaMemcpyAsync(&asym, aux, sizeof asym, cudaMemcpyDeviceToHost, c->stream));
        RK(host_sync(c));
        dense_sym = asym == 0 ? 1 : 0;
        // a row block (ellpack_ctx_set_rows) runs dense only for a symmetric X (X^T = X: one copy)
        if ((p.row_begin != 0 || p.row_end != n) && dense_sym != 1) dense_sym = -1;
    }
    c->last_dense = 0;
    // a small matrix on one rank: the small-matrix kernel (tiny.cu) -- one launch that also writes
    // the status and the canonical sums of tr X, tr X^2
    const bool tiny = dense_sym < 0 && n <= kNoProbeN && !c->comm && c->window_opt == 0 && c->ring_kernel == 0 &&
                      c->small_kernel == 0 && !c->profile && tiny_eligible(p, n);
    if (tiny) {
        // counter + 2 ints per CTA, zeroed once here (the kernel leaves the counter zero); grown
        // outside any graph capture
        const size_t tb = 16 + 8 * (size_t)((n + 3) / 4);
        if (c->tiny.bytes < tb) {
            RK(grow(c, c->tiny, tb));
            CK(cudaMemsetAsync(c->tiny.p, 0, c->tiny.bytes, c->stream));
        }
    }
    auto enqueue = [&]() -> int {
        if (tiny) {
            p.ncols = n;
            p.status = c->d_status;  // written whole by the last CTA (no memset)
            // status and sums straight into the pinned host block when it is mapped (the read-back
            // copies are then not needed), else into the device status/sums
            CK(launch_tiny(p, n, (unsigned int*)c->tiny.p, (int32_t*)((char*)c->tiny.p + 16),
                           c->h_dev ? c->h_dev->status : c->d_status, c->h_dev ? c->h_dev->sums : c->d_sums,
                           c->stream));
            c->launches++;
            c->last_cfg = LaunchCfg{(int)((n + 31) & ~int64_t(31)), 4, (int)((n + 3) / 4), tiny_smem(n), 0, 0};
            c->last_fast = 0;
            c->last_split = 0;
            c->last_hB = 0;
            c->last_small = 1;
            return ELLPACK_OK;
        }
        if (dense_sym >= 0) RK(enqueue_dense_op(c, p, n, dense_sym == 1));
        else RK(enqueue_row_op(c, p, n));
        const double* arrs[2] = {p.diag_a, p.diag_s};
        RK(enqueue_canonical(c, arrs, 2, n));
        return reduce_status(c);
    };
    // A small matrix runs unprobed on one general-path window: its launch sequence depends only on the
    // shapes and pointers, so it is captured once as a CUDA graph and replayed (one launch instead of
    // a breakpoints kernel, two memsets, the row kernel and two reduction kernels -- the cfg1-sized
    // call is launch-latency bound)
    const bool graphable = dense_sym < 0 && n <= kNoProbeN && !c->comm && c->window_opt == 0 && c->ring_kernel == 0 &&
                           !c->profile && !c->validate && c->row_end < 0;
    if (graphable) {
        uint64_t key = 0x78325f67ull, tb;
        memcpy(&tb, &tau, 8);
        for (uint64_t v : {(uint64_t)(uintptr_t)x->val, (uint64_t)(uintptr_t)x->col, (uint64_t)(uintptr_t)x->nnz,
                           (uint64_t)x->w, (uint64_t)(uintptr_t)x2->val, (uint64_t)(uintptr_t)x2->col,
                           (uint64_t)(uintptr_t)x2->nnz, (uint64_t)x2->w, (uint64_t)n, tb,
                           (uint64_t)(uintptr_t)c->rows[0].p, (uint64_t)(uintptr_t)c->rows[1].p,
                           (uint64_t)(uintptr_t)c->partials.p, (uint64_t)(uintptr_t)c->bp.p})
            key = mix64(key, v);
        if (!c->x2_exec || !c->x2_exec_ok || c->x2_exec_key != key) {
            if (c->x2_exec) { cudaGraphExecDestroy(c->x2_exec); c->x2_exec = nullptr; }
            // grow the workspace outside the capture (the bp and partials buffers of this shape)
            const int np = (int)((n + 31) / 32) + 1;  // any window S >= 32 the plan picks
            RK(grow(c, c->bp, sizeof(int32_t) * (size_t)n * np));
            RK(grow(c, c->partials, sizeof(double) * 2 * (size_t)((n + kTraceBlock - 1) / kTraceBlock)));
            cudaStream_t cs = nullptr;
            CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            cudaStream_t saved = c->stream;
            const int64_t l0 = c->launches;
            cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed);
            int rc = ELLPACK_OK;
            cudaGraph_t g = nullptr;
            if (!e) {
                c->stream = cs;
                rc = enqueue();
                // the read-back copies are graph nodes too (none when the small-matrix kernel
                // wrote to the mapped host block)
                if (rc == ELLPACK_OK && !(tiny && c->h_dev)) rc = fetch_copies(c, 2);
                c->stream = saved;
                e = cudaStreamEndCapture(cs, &g);
            }
            c->x2_exec_launches = (int)(c->launches - l0);
            c->launches = l0;
            if (!e && rc == ELLPACK_OK) e = cudaGraphInstantiate(&c->x2_exec, g, 0);
            if (g) cudaGraphDestroy(g);
            cudaStreamDestroy(cs);
            RK(rc);
            CK(e);
            // the key covers the buffers the capture saw (they may have grown inside it)
            key = 0x78325f67ull;
            for (uint64_t v : {(uint64_t)(uintptr_t)x->val, (uint64_t)(uintptr_t)x->col, (uint64_t)(uintptr_t)x->nnz,
                               (uint64_t)x->w, (uint64_t)(uintptr_t)x2->val, (uint64_t)(uintptr_t)x2->col,
                               (uint64_t)(uintptr_t)x2->nnz, (uint64_t)x2->w, (uint64_t)n, tb,
                               (uint64_t)(uintptr_t)c->rows[0].p, (uint64_t)(uintptr_t)c->rows[1].p,
                               (uint64_t)(uintptr_t)c->partials.p, (uint64_t)(uintptr_t)c->bp.p})
                key = mix64(key, v);
            c->x2_exec_key = key;
            c->x2_exec_ok = true;
            c->x2_cfg = c->last_cfg;
            c->x2_fast = c->last_fast;
            c->x2_split = c->last_split;
            c->x2_hB = c->last_hB;
            c->x2_small = c->last_small;
        }
        CK(cudaGraphLaunch(c->x2_exec, c->stream));
        c->launches += c->x2_exec_launches;
        c->last_cfg = c->x2_cfg;
        c->last_fast = c->x2_fast;
        c->last_split = c->x2_split;
        c->last_hB = c->x2_hB;
        c->last_small = c->x2_small;
        RK(host_sync(c));
    } else {
        RK(enqueue());
        if (tiny && c->h_dev) RK(host_sync(c));
        else RK(fetch(c, 2));
    }
    RK(finish_status(c));
    if (trace_x) *trace_x = c->h->sums[0];
    if (trace_x2) *trace_x2 = c->h->sums[1];
    return ELLPACK_OK;
}

static int add_via_identity(ellpack_ctx c, ellpack_desc* a, const KMat& old, bool old_is_a,
                            double alpha, double beta, double tau) {
    RK(check_comm_n(c, a->n));
    CK(cudaSetDevice(c->device));
    RK(ensure_identity(c, a->n));
    RowOpParams p = base_params(c, a->n);
    p.A = kmat(a);
    p.B = identity(c);
    p.Old = old;
    p.old_mode = 1;
    p.C = kout(a);
    p.alpha = alpha;
    p.beta = beta;
    p.tau = tau;
    p.stash_a = 1;
    p.stash_old = old_is_a ? 1 : 0;
    RK(enqueue_row_op(c, p, a->n));
    RK(reduce_status(c));
    RK(fetch(c, 0));
    return finish_status(c);
}

int ellpack_add(ellpack_ctx c, ellpack_desc* a, const ellpack_desc* b, double alpha, double beta,
                double tau) {
    if (!c) return ELLPACK_ERR_ARG;
    RK(check_desc(a));
    RK(check_desc(b));
    if (a->n != b->n) return ELLPACK_ERR_DIM;
    if (!valid_tau(tau) || !std::isfinite(alpha) || !std::isfinite(beta)) return ELLPACK_ERR_ARG;
    const bool ident = a->val == b->val && a->col == b->col && a->nnz == b->nnz && a->w == b->w;
    if (!ident && same(a, b)) return ELLPACK_ERR_ARG;  // partial aliasing
    CK(cudaSetDevice(c->device));
    RK(validate_inputs(c, {a, b}));
    return add_via_identity(c, a, kmat(b), ident, alpha, beta, tau);
}

int ellpack_scale_add_identity(ellpack_ctx c, ellpack_desc* a, double alpha, double beta, double tau) {
    if (!c) return ELLPACK_ERR_ARG;
    RK(check_desc(a));
    if (!valid_tau(tau) || !std::isfinite(alpha) || !std::isfinite(beta)) return ELLPACK_ERR_ARG;
    CK(cudaSetDevice(c->device));
    RK(validate_inputs(c, {a}));
    RK(ensure_identity(c, a->n));
    return add_via_identity(c, a, identity(c), false, alpha, beta, tau);
}

int ellpack_add_identity(ellpack_ctx c, ellpack_desc* a, double beta, double tau) {
    return ellpack_scale_add_identity(c, a, 1.0, beta, tau);
}

int ellpack_trace(ellpack_ctx c, const ellpack_desc* a, double* out) {
    if (!c || !out) return ELLPACK_ERR_ARG;
    RK(check_desc(a));
    RK(check_comm_n(c, a->n));
    CK(cudaSetDevice(c->device));
    RK(validate_inputs(c, {a}));
    const int64_t n = a->n;
    RK(grow(c, c->rows[0], sizeof(double) * n));
    int64_t r0, r1;
    rows_of(c, n, &r0, &r1);
    CK(launch_stored_diag(kmat(a), r0, r1, (double*)c->rows[0].p, c->stream));
    c->launches++;
    const double* arrs[1] = {(const double*)c->rows[0].p};
    RK(enqueue_canonical(c, arrs, 1, n));
    CK(cudaMemsetAsync(c->d_status, 0, 8, c->stream));
    RK(fetch(c, 1));
    *out = c->h->sums[0];
    return ELLPACK_OK;
}

int ellpack_fnorm_diff(ellpack_ctx c, const ellpack_desc* a, const ellpack_desc* b, double* out) {
    if (!c || !out) return ELLPACK_ERR_ARG;
    RK(check_desc(a));
    RK(check_desc(b));
    if (a->n != b->n) return ELLPACK_ERR_DIM;
    RK(check_comm_n(c, a->n));
    CK(cudaSetDevice(c->device));
    RK(validate_inputs(c, {a, b}));
    const int64_t n = a->n;
    RK(grow(c, c->rows[0], sizeof(double) * n));
    int64_t r0, r1;
    rows_of(c, n, &r0, &r1);
    CK(launch_fnorm_rows(kmat(a), kmat(b), r0, r1, (double*)c->rows[0].p, c->stream));
    c->launches++;
    const double* arrs[1] = {(const double*)c->rows[0].p};
    RK(enqueue_canonical(c, arrs, 1, n));
    CK(cudaMemsetAsync(c->d_status, 0, 8, c->stream));
    RK(fetch(c, 1));
    *out = std::sqrt(c->h->sums[0]);
    return ELLPACK_OK;
}

static int gershgorin_impl(ellpack_ctx c, const ellpack_desc* h, double* emin, double* emax) {
    const int64_t n = h->n;
    int64_t r0, r1;
    rows_of(c, n, &r0, &r1);
    const unsigned long long init[2] = {~0ull, 0ull};
    c->h->keys[0] = init[0];
    c->h->keys[1] = init[1];
    CK(cudaMemcpyAsync(c->d_keys, c->h->keys, 16, cudaMemcpyHostToDevice, c->stream));
    CK(launch_gershgorin(kmat(h), r0, r1, c->d_keys, c->stream));
    c->launches++;
    if (c->comm) {
        NK(g_nccl.GroupStart());
        NK(g_nccl.AllReduce(c->d_keys, c->d_keys, 1, ncclUint64, ncclMin, c->comm, c->stream));
        NK(g_nccl.AllReduce(c->d_keys + 1, c->d_keys + 1, 1, ncclUint64, ncclMax, c->comm, c->stream));
        NK(g_nccl.GroupEnd());
    }
    CK(cudaMemcpyAsync(c->h->keys, c->d_keys, 16, cudaMemcpyDeviceToHost, c->stream));
    RK(host_sync(c));
    *emin = dkey_inv(c->h->keys[0]);
    *emax = dkey_inv(c->h->keys[1]);
    return ELLPACK_OK;
}

int ellpack_gershgorin(ellpack_ctx c, const ellpack_desc* h, double* emin, double* emax) {
    if (!c || !emin || !emax) return ELLPACK_ERR_ARG;
    RK(check_desc(h));
    RK(check_comm_n(c, h->n));
    CK(cudaSetDevice(c->device));
    RK(validate_inputs(c, {h}));
    return gershgorin_impl(c, h, emin, emax);
}

int ellpack_allgather_rows(ellpack_ctx c, ellpack_desc* m) {
    if (!c) return ELLPACK_ERR_ARG;
    RK(check_desc(m));
    RK(check_comm_n(c, m->n));
    return allgather_desc(c, m);
}

int ellpack_halo_plan(int64_t n, int nranks, int rank, int64_t per, const int64_t* need, int32_t* n_send,
                      int64_t* send, int32_t* n_recv, int64_t* recv) {
    if (n < 0 || nranks < 1 || rank < 0 || rank >= nranks || per < 1 || !need || !n_send || !send || !n_recv ||
        !recv)
        return ELLPACK_ERR_ARG;
    // block q = [q per, min(n, (q + 1) per)); need[2q..2q+1] = rank q's referenced rows (inclusive)
    auto blk0 = [&](int q) { return std::min<int64_t>(n, (int64_t)q * per); };
    auto blk1 = [&](int q) { return std::min<int64_t>(n, (int64_t)(q + 1) * per); };
    int32_t ns = 0, nr = 0;
    for (int q = 0; q < nranks; ++q) {
        if (q == rank) continue;
        const int64_t s0 = std::max(blk0(rank), std::max<int64_t>(0, need[2 * q]));
        const int64_t s1 = std::min(blk1(rank), need[2 * q + 1] + 1);
        if (s0 < s1) { send[3 * ns] = q; send[3 * ns + 1] = s0; send[3 * ns + 2] = s1; ++ns; }
        const int64_t t0 = std::max(blk0(q), std::max<int64_t>(0, need[2 * rank]));
        const int64_t t1 = std::min(blk1(q), need[2 * rank + 1] + 1);
        if (t0 < t1) { recv[3 * nr] = q; recv[3 * nr + 1] = t0; recv[3 * nr + 2] = t1; ++nr; }
    }
    *n_send = ns;
    *n_recv = nr;
    return ELLPACK_OK;
}

int ellpack_halo_rows(ellpack_ctx c, const ellpack_desc* a, ellpack_desc* b) {
    if (!c) return ELLPACK_ERR_ARG;
    RK(check_desc(a));
    RK(check_desc(b));
    if (a->n != b->n) return ELLPACK_ERR_DIM;
    RK(check_comm_n(c, a->n));
    CK(cudaSetDevice(c->device));
    return halo_desc(c, a, b);
}

int ellpack_nccl_unique_id(uint8_t id[128]) {
    if (!id) return ELLPACK_ERR_ARG;
    if (!load_nccl()) return ELLPACK_ERR_NCCL;
    ncclUniqueId u;
    NK(g_nccl.GetUniqueId(&u));
    memcpy(id, &u, 128);
    return ELLPACK_OK;
}

int ellpack_ctx_attach_nccl(ellpack_ctx c, int nranks, int rank, const uint8_t id[128],
                            int64_t row_begin, int64_t row_end) {
    if (!c || !id || nranks < 1 || rank < 0 || rank >= nranks || row_begin < 0 || row_end < row_begin)
        return ELLPACK_ERR_ARG;
    if (row_begin % kTraceBlock) return ELLPACK_ERR_ARG;
    if (c->comm) return ELLPACK_ERR_STATE;
    if (!load_nccl()) return ELLPACK_ERR_NCCL;
    CK(cudaSetDevice(c->device));
    ncclUniqueId u;
    memcpy(&u, id, 128);
    NK(g_nccl.CommInitRank(&c->comm, nranks, u, rank));
    // Every rank's block, all-gathered (collective, so every rank takes the same decision): the
    // blocks must be contiguous, ascending with rank, equal, multiples of 256 rows (canonical
    // trace blocks and equal all-gather counts, §8c-c7/c12, reading R17) and cover [0, N).
    long long* d_rng = nullptr;
    std::vector<long long> rng(2 * (size_t)nranks);
    const long long mine[2] = {(long long)row_begin, (long long)row_end};
    cudaError_t e = cudaMalloc(&d_rng, sizeof(long long) * 2 * (nranks + 1));
    if (!e) e = cudaMemcpyAsync(d_rng + 2 * nranks, mine, sizeof mine, cudaMemcpyHostToDevice, c->stream);
    ncclResult_t ne = ncclSuccess;
    if (!e) ne = g_nccl.AllGather(d_rng + 2 * nranks, d_rng, 2, ncclInt64, c->comm, c->stream);
    if (!e && ne == ncclSuccess)
        e = cudaMemcpyAsync(rng.data(), d_rng, sizeof(long long) * 2 * nranks, cudaMemcpyDeviceToHost, c->stream);
    if (!e) { c->host_syncs++; e = cudaStreamSynchronize(c->stream); }
    if (d_rng) cudaFree(d_rng);
    int rc = e ? from_cuda(e) : (ne != ncclSuccess ? ELLPACK_ERR_NCCL : ELLPACK_OK);
    const long long per = rng[1] - rng[0];
    if (rc == ELLPACK_OK) {
        bool ok = per > 0 && per % kTraceBlock == 0;
        for (int q = 0; q < nranks && ok; ++q)
            ok = rng[2 * q] == (long long)q * per && rng[2 * q + 1] == (long long)(q + 1) * per;
        if (!ok) rc = ELLPACK_ERR_ARG;
    }
    if (rc != ELLPACK_OK) {
        g_nccl.CommDestroy(c->comm);
        c->comm = nullptr;
        return rc;
    }
    c->nranks = nranks;
    c->rank = rank;
    c->row_begin = row_begin;
    c->row_end = row_end;
    c->comm_n = per * nranks;
    if (c->h_reach) cudaFreeHost(c->h_reach);
    c->h_reach = nullptr;
    CK(cudaMallocHost(&c->h_reach, 2 * sizeof(int32_t) * nranks));
    return ELLPACK_OK;
}

void sp2_opts_default(sp2_opts* o) {
    if (!o) return;
    memset(o, 0, sizeof *o);
    o->threshold = 0.0;
    o->max_iter = 100;
    o->min_iter = 20;
    o->stag_gate = 1e-3;
    o->emin = NAN;
    o->emax = NAN;
    o->on_overflow = SP2_GROW;
    o->max_width = 0;
    o->initial_width = 0;
}

// ------------------------------------------------------------------------- SP2

namespace {

// SP2 iterates live in context-owned buffers (c->it[slot]) that only grow: repeated runs and
// regrows reuse them, no allocation or zero-fill in the loop (padding slots are never read).
struct DevMatrix {
    ellpack_desc d{};
    bool owned = false;
    int slot = 0;
};

int dm_alloc(ellpack_ctx c, DevMatrix& m, int64_t n, int32_t w) {
    // ELLPACK_OPT_SP2_MEM_CAP (fault injection): the live iterates' value arrays above the cap
    // "do not fit"
    if (c->sp2_mem_cap > 0) {
        int64_t live = (int64_t)sizeof(double) * n * w;
        for (int q = 0; q < 4; ++q) live += q == m.slot ? 0 : c->it_live[q];
        if (live > c->sp2_mem_cap) return ELLPACK_ERR_NOMEM;
    }
    Buf* b = c->it[m.slot];
    RK(grow(c, b[0], sizeof(double) * (size_t)n * w));
    RK(grow(c, b[1], sizeof(int32_t) * (size_t)n * w));
    RK(grow(c, b[2], sizeof(int32_t) * (size_t)n));
    m.d.n = n;
    m.d.w = w;
    m.d.reserved = 0;
    m.d.val = (double*)b[0].p;
    m.d.col = (int32_t*)b[1].p;
    m.d.nnz = (int32_t*)b[2].p;
    // rows are reinterpreted at the new width: empty them (with a halo exchange, rows outside a
    // rank's block and halo are never written and must read as valid rows)
    CK(cudaMemsetAsync(m.d.nnz, 0, sizeof(int32_t) * (size_t)n, c->stream));
    m.owned = true;
    c->it_live[m.slot] = (int64_t)sizeof(double) * n * w;
    return ELLPACK_OK;
}

void dm_free(ellpack_ctx c, DevMatrix& m) {
    m.owned = false;
    c->it_live[m.slot] = 0;
}

// give the slot's device memory back (grow() never shrinks: a failed retry must not keep a
// partially grown, oversized value array)
void dm_release(ellpack_ctx c, DevMatrix& m) {
    for (Buf& b : c->it[m.slot]) release(c, b);
    dm_free(c, m);
}

int32_t round_up32(int64_t x) { return (int32_t)((x + 31) & ~int64_t(31)); }

// MIN over ranks of a width (0 = "did not fit" on some rank); identity without a communicator.
int agree_width(ellpack_ctx c, int32_t mine, int32_t* out) {
    if (!c->comm) { *out = mine; return ELLPACK_OK; }
    int32_t* d = c->d_bw + 8;
    c->h->imax = mine;
    CK(cudaMemcpyAsync(d, &c->h->imax, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
    NK(g_nccl.AllReduce(d, d, 1, ncclInt32, ncclMin, c->comm, c->stream));
    CK(cudaMemcpyAsync(&c->h->imax, d, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    RK(host_sync(c));
    *out = c->h->imax;
    return ELLPACK_OK;
}

// Physical iterate width `want` (headroom), falling back to `need` when the headroom does not
// fit in device memory (large N densifying iterates). The slot is released before the retry, so
// the retry is not charged for a partial oversized allocation. With a communicator every rank
// ends with the same physical width (MIN over ranks: the halo send/recv counts are cnt * w on
// both sides) and a NOMEM on any rank is a NOMEM on every rank.
int dm_alloc_headroom(ellpack_ctx c, DevMatrix& m, int64_t n, int32_t& want, int32_t need) {
    int rc = dm_alloc(c, m, n, want);
    int32_t got = want;
    if (rc == ELLPACK_ERR_NOMEM && need < want) {
        cudaGetLastError();  // clear the failed allocation
        dm_release(c, m);
        rc = dm_alloc(c, m, n, need);
        got = need;
    }
    if (rc == ELLPACK_ERR_NOMEM) {
        cudaGetLastError();
        got = 0;
    } else if (rc != ELLPACK_OK) {
        return rc;
    }
    int32_t agreed = got;
    RK(agree_width(c, got, &agreed));
    if (agreed <= 0) {
        dm_release(c, m);
        return ELLPACK_ERR_NOMEM;
    }
    m.d.w = agreed;  // a wider local buffer is viewed at the agreed (smaller) width
    want = agreed;
    return ELLPACK_OK;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Exact number of (this rank's, then all-reduced) rows of m with more than w entries (the FAIL
// report, §8c-c4: overflow_rows = #{i : kept_i > W}); m's stored counts must not be truncated
// below w + 1 (physical width >= logical width). One kernel + one synchronising read-back.
int count_rows_over(ellpack_ctx c, const ellpack_desc* m, int32_t w, int64_t* out) {
    int64_t r0, r1;
    rows_of(c, m->n, &r0, &r1);
    int32_t* d = c->d_status + 2;
    CK(cudaMemsetAsync(d, 0, sizeof(int32_t), c->stream));
    CK(launch_count_over(m->nnz, r0, r1, w, d, c->stream));
    c->launches++;
    if (c->comm) NK(g_nccl.AllReduce(d, d, 1, ncclInt32, ncclSum, c->comm, c->stream));
    CK(cudaMemcpyAsync(&c->h->imax, d, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    RK(host_sync(c));
    *out = c->h->imax;
    return ELLPACK_OK;
}

// X (width w) <- drop(alpha*H + beta*I) computed at a safe width first (H.w + 1),
// then copied at width w; returns required width in *req.
int sp2_make_x0(ellpack_ctx c, const ellpack_desc* h, double alpha, double beta, double tau,
                DevMatrix& tmp, int32_t* req) {
    const int64_t n = h->n;
    const int32_t wt = (h->w + 2) & ~1;
    RK(dm_alloc(c, tmp, n, wt));
    int64_t r0, r1;
    rows_of(c, n, &r0, &r1);
    // tmp <- H (own rows), then tmp <- alpha*tmp + beta*I in place
    CK(cudaMemsetAsync(c->d_status, 0, 8, c->stream));
    CK(launch_copy_rows(kmat(h), kout(&tmp.d), r0, r1, c->d_status, c->stream));
    c->launches++;
    RK(ensure_identity(c, n));
    RowOpParams p = base_params(c, n);
    p.A = kmat(&tmp.d);
    p.B = identity(c);
    p.Old = identity(c);
    p.old_mode = 1;
    p.C = kout(&tmp.d);
    p.alpha = alpha;
    p.beta = beta;
    p.tau = tau;
    p.stash_a = 1;
    RK(enqueue_row_op(c, p, n));
    RK(reduce_status(c));
    RK(fetch(c, 0));
    *req = c->h->status[1];
    return ELLPACK_OK;
}

// symmetric step: U (the upper triangle of X_{n+1}) is allocated only when a launch takes the
// general path's upper route, at the physical width of the iterate it mirrors into
struct UpperAlloc {
    DevMatrix* U;
    int64_t n;
    int32_t w;
};
int alloc_upper(ellpack_ctx c, void* arg, KOut* out) {
    UpperAlloc* a = (UpperAlloc*)arg;
    if (!a->U->owned || a->U->d.w < a->w) {
        int rc = dm_alloc(c, *a->U, a->n, a->w);
        if (rc != ELLPACK_OK) {
            if (rc == ELLPACK_ERR_NOMEM) { cudaGetLastError(); dm_release(c, *a->U); }
            return rc;
        }
    }
    *out = kout(&a->U->d);
    return ELLPACK_OK;
}

// Probe of the next SP2 operand X (A = B = Old = X) enqueued right after the step that wrote it,
// fetched with that step's status: the next step plans its launch with no read-back of its own.
// With a communicator each rank's reach (the X rows its rows reference) is all-gathered too, so
// the halo exchange of X needs no read-back either.
int enqueue_next_probe(ellpack_ctx c, const ellpack_desc* x) {
    RowOpParams q = base_params(c, x->n);
    q.A = kmat(x);
    q.B = kmat(x);
    q.Old = kmat(x);
    q.alpha = 1.0;
    q.old_mode = 1;
    RK(enqueue_probe(c, q, x->n));
    if (c->comm) {
        RK(grow(c, c->halo, sizeof(long long) * 2 * (size_t)c->nranks));
        NK(g_nccl.AllGather(c->d_bw + 5, (int32_t*)c->halo.p, 2, ncclInt32, c->comm, c->stream));
    }
    return ELLPACK_OK;
}

// host copies of the prefetched probe (bw) and every rank's reach, as halo_exec's need ranges
void take_probe(ellpack_ctx c, int32_t* bw, std::vector<int64_t>& need) {
    memcpy(bw, c->h->bw, kProbe * sizeof(int32_t));
    for (int q = 0; c->comm && q < c->nranks; ++q) {
        need[2 * q] = (int64_t)INT_MAX - c->h_reach[2 * q];
        need[2 * q + 1] = (int64_t)c->h_reach[2 * q + 1] - 1;
    }
}


// ---------------------------------------------------------------- device-resident SP2 loop

constexpr int64_t kDevLoopMaxN = 8192;         // automatic: the device loop for N up to this
constexpr int kDevLoopWindow = 1024;           // its general-path window (every iterate width)

// The device loop keeps both iterates at the physical width max_width (no regrow inside the
// graph), single rank, and the automatic choice takes it for small N only: there the host
// synchronisation and the launch sequence are the iteration's cost.
constexpr int64_t kDevLoopDenseN = 1024;  // the device loop's steps are all dense up to this N

// the device loop's steps run dense: forced, or small N where a dense step costs about as much as a
// narrow sparse one (N = 512: 31 us GEMM) and the run is bound by per-iteration host work
bool device_loop_dense(ellpack_ctx c, int64_t n, bool sym) {
    if (c->dense_opt == 1 || !dense_fits(c, n, sym ? 2 : 3)) return false;
    return c->dense_opt == 2 || n <= kDevLoopDenseN;
}

bool use_device_loop(ellpack_ctx c, int64_t n, int32_t maxw, bool sym) {
    if (c->comm || c->sp2_loop == 1) return false;
    const double bytes = 2.0 * 12.0 * (double)n * (double)maxw;
    if (c->sp2_loop == 2) return bytes <= 64e9;
    // automatic. With the dense regime available: the device loop when all its steps go dense, else
    // the host loop, whose steps switch to dense as the iterates fill in
    if (c->dense_opt != 1 && n <= kDenseMaxN) return device_loop_dense(c, n, sym) && bytes <= 4e9;
    return n <= kDevLoopMaxN && bytes <= 4e9;
}


// SP2 iterations as ONE launch of a CUDA graph: a WHILE node whose body is one iteration
// (products, breakpoints, the fused step on the general path with (alpha, beta, old_mode) from the
// control block, [T2], canonical sums, rows over the logical width, the control kernel, X <- Y).
// The host waits once, after the loop. X (width maxw) holds X0 on entry and the final iterate on
// exit. Fills the report fields the host loop fills and returns an ellpack status.
int sp2_device_loop(ellpack_ctx c, const sp2_opts& o, int64_t n, int64_t nocc, double tol, int32_t w, int32_t maxw,
                    bool closest, bool sym, double& trX, double t2, DevMatrix& X, DevMatrix& Y, sp2_report& R,
                    sp2_iter_rec* iters, int32_t& wx, int& stop, int& it, double& t_loop) {
    // every step dense (dense.cu) or every step on the general path
    const bool dense = device_loop_dense(c, n, sym);
    // iterates at the physical width maxw
    if (X.d.w < maxw) {
        RK(dm_alloc(c, Y, n, maxw));
        CK(cudaMemsetAsync(c->d_status, 0, 8, c->stream));
        CK(launch_copy_rows(kmat(&X.d), kout(&Y.d), 0, n, c->d_status, c->stream));
        c->launches++;
        std::swap(X, Y);
    }
    if (!Y.owned || Y.d.w < maxw) RK(dm_alloc(c, Y, n, maxw));
    // workspace the captured launches use, grown before capture (no allocation inside the graph)
    const int S = (int)std::min<int64_t>(kDevLoopWindow, (n + 31) & ~int64_t(31));
    const int np = (int)((n + S - 1) / S) + 1;
    RK(grow(c, c->bp, sizeof(int32_t) * (size_t)n * np));
    for (int a = 0; a < 4; ++a) RK(grow(c, c->rows[a], sizeof(double) * n));
    RK(grow(c, c->partials, sizeof(double) * 4 * (size_t)((n + kTraceBlock - 1) / kTraceBlock)));
    RK(grow(c, c->sp2dev, sizeof(Sp2Dev)));
    RK(grow(c, c->sp2rec, sizeof(sp2_iter_rec) * (size_t)o.max_iter));
    if (dense) {
        const int64_t np = dense_np(n);
        const size_t bytes = sizeof(double) * (size_t)np * (size_t)np;
        RK(grow(c, c->dense[0], bytes));
        RK(grow(c, c->dense[2], bytes));
        if (!sym) RK(grow(c, c->dense[1], bytes));
        RK(grow(c, c->dflags, 2 * (size_t)(np / kDenseTile) * (size_t)(np / kDenseK) +
                                  2 * (size_t)(np / kDenseTile) * dense_kbw((int)np) * 8 +
                                  (size_t)(np / 16) * (size_t)(np / kDenseTile)));
        (void)dense_mma_ok(c->stream);  // the once-per-device check synchronises: not inside the capture
        // the captured steps clear D by the previous step's flags: start from D = 0, flags = 0
        CK(cudaMemsetAsync(c->dense[0].p, 0, bytes, c->stream));
        CK(cudaMemsetAsync(c->dflags.p, 0, c->dflags.bytes, c->stream));
        c->dense_clean_np = np;
    }
    Sp2Dev* dev = (Sp2Dev*)c->sp2dev.p;
    Sp2Dev hd;
    memset(&hd, 0, sizeof hd);
    hd.tol = tol;
    hd.stag_gate = o.stag_gate;
    hd.nocc = (double)nocc;
    hd.min_iter = o.min_iter;
    hd.max_iter = o.max_iter;
    hd.on_overflow = o.on_overflow;
    hd.closest = closest;
    hd.maxw = maxw;
    hd.pad0 = dense ? 1 : 0;  // recorded as each iteration's regime
    int branch = (trX > (double)nocc) ? SP2_SQUARE : SP2_EXPAND;
    if (closest)
        branch = (std::fabs(t2 - (double)nocc) < std::fabs((2.0 * trX - t2) - (double)nocc)) ? SP2_SQUARE : SP2_EXPAND;
    hd.branch = branch;
    hd.dyn[0] = branch == SP2_SQUARE ? 1.0 : -1.0;
    hd.dyn[1] = branch == SP2_SQUARE ? 0.0 : 2.0;
    hd.dyn[2] = branch == SP2_SQUARE ? 2.0 : 1.0;
    hd.trX = trX;
    hd.t2 = t2;
    hd.e2 = hd.e1 = NAN;
    hd.stop = -1;
    hd.wy = w;
    CK(cudaMemcpyAsync(dev, &hd, sizeof hd, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->d_status + 2, 0, sizeof(int32_t), c->stream));
    CK(cudaMemsetAsync(c->d_keys + 2, 0, 8, c->stream));

    // the graph: rebuilt only when something it captured changed
    uint64_t key = 0x5350320ull;
    for (uint64_t v : {(uint64_t)(uintptr_t)X.d.val, (uint64_t)(uintptr_t)Y.d.val, (uint64_t)(uintptr_t)c->bp.p,
                       (uint64_t)(uintptr_t)c->rows[0].p, (uint64_t)(uintptr_t)c->rows[3].p,
                       (uint64_t)(uintptr_t)c->partials.p, (uint64_t)(uintptr_t)c->sp2dev.p,
                       (uint64_t)(uintptr_t)c->sp2rec.p, (uint64_t)(uintptr_t)c->stream, (uint64_t)n,
                       (uint64_t)maxw, (uint64_t)closest, (uint64_t)S, (uint64_t)dense, (uint64_t)sym,
                       (uint64_t)(uintptr_t)c->dense[0].p, (uint64_t)(uintptr_t)c->dense[1].p,
                       (uint64_t)(uintptr_t)c->dense[2].p, (uint64_t)(uintptr_t)c->dflags.p})
        key = mix64(key, v);
    uint64_t tb;
    memcpy(&tb, &o.threshold, 8);
    key = mix64(key, tb);
    if (!c->sp2_exec || c->sp2_exec_key != key) {
        if (c->sp2_exec) { cudaGraphExecDestroy(c->sp2_exec); c->sp2_exec = nullptr; }
        cudaGraph_t g = nullptr;
        CK(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle cond;
        cudaError_t e = cudaGraphConditionalHandleCreate(&cond, g, 1u, cudaGraphCondAssignDefault);
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = cond;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t wnode;
        if (!e) e = cudaGraphAddNode(&wnode, g, nullptr, 0, &cp);
        cudaStream_t cs = nullptr;
        if (!e) e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
        int rc = ELLPACK_OK;
        int64_t l0 = c->launches;
        if (!e) e = cudaStreamBeginCaptureToGraph(cs, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                  cudaStreamCaptureModeRelaxed);
        if (!e) {
            cudaStream_t saved = c->stream;
            const bool prof = c->profile;
            c->stream = cs;
            c->profile = false;
            c->force_general_s = S;
            do {
                if ((e = launch_products(kmat(&X.d), X.d.nnz, 0, n, c->d_keys + 2, cs))) break;
                c->launches++;
                RowOpParams p = base_params(c, n);
                p.A = kmat(&X.d);
                p.B = kmat(&X.d);
                p.Old = kmat(&X.d);
                p.C = kout(&Y.d);
                p.tau = o.threshold;
                p.alpha = 1.0;     // placeholders for the planner: the kernel reads p.dyn
                p.old_mode = 2;
                p.dyn = dev->dyn;
                p.diag_s = (double*)c->rows[0].p;
                p.diag_c = (double*)c->rows[1].p;
                p.normsq = (double*)c->rows[2].p;
                int32_t bw0[kProbe] = {0, 0, 0, 0, 0, 0, 0};
                if (dense) rc = enqueue_dense_op(c, p, n, sym);
                else rc = enqueue_row_op(c, p, n, bw0);
                if (rc) break;
                if (closest) {
                    if ((e = launch_sumsq_rows(kmat(&Y.d), 0, n, (double*)c->rows[3].p, cs))) break;
                    c->launches++;
                }
                const double* arrs[4] = {p.diag_s, p.diag_c, p.normsq, (const double*)c->rows[3].p};
                if ((rc = enqueue_canonical(c, arrs, closest ? 4 : 3, n))) break;
                if ((e = launch_count_over_dev(Y.d.nnz, n, dev, c->d_status + 2, cs))) break;
                if ((e = launch_sp2_ctl(dev, c->d_sums, c->d_status, c->d_status + 2, c->d_keys + 2, c->sp2rec.p,
                                        (unsigned long long)cond, cs)))
                    break;
                if ((e = launch_copy_rows(kmat(&Y.d), kout(&X.d), 0, n, c->d_status + 4, cs))) break;
                c->launches += 3;
            } while (false);
            c->stream = saved;
            c->profile = prof;
            c->force_general_s = 0;
            cudaGraph_t body_out = nullptr;
            cudaError_t e2 = cudaStreamEndCapture(cs, &body_out);
            if (!e) e = e2;
        }
        c->sp2_exec_launches = (int)(c->launches - l0);
        c->launches = l0;
        if (!e && rc == ELLPACK_OK) e = cudaGraphInstantiate(&c->sp2_exec, g, 0);
        if (cs) cudaStreamDestroy(cs);
        cudaGraphDestroy(g);
        if (rc != ELLPACK_OK) return rc;
        CK(e);
        c->sp2_exec_key = key;
    }
    cudaEventRecord(c->ev[0], c->stream);
    CK(cudaGraphLaunch(c->sp2_exec, c->stream));
    cudaEventRecord(c->ev[1], c->stream);
    CK(cudaMemcpyAsync(&hd, dev, sizeof hd, cudaMemcpyDeviceToHost, c->stream));
    RK(host_sync(c));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    t_loop = ms * 1e-3;
    it = hd.it;
    c->launches += (int64_t)c->sp2_exec_launches * (hd.it + (hd.stop == SP2_OVERFLOWED ? 1 : 0));
    if (iters && hd.it > 0) {
        CK(cudaMemcpyAsync(iters, c->sp2rec.p, sizeof(sp2_iter_rec) * (size_t)hd.it, cudaMemcpyDeviceToHost,
                           c->stream));
        RK(host_sync(c));
    }
    trX = hd.trX;
    wx = hd.wy;
    R.regrows += hd.regrows;
    if (hd.stop == SP2_OVERFLOWED) {
        R.stop_reason = SP2_OVERFLOWED;
        R.overflow_rows = hd.overflow_rows;
        R.required_width = hd.required;
        R.fail_iter = hd.fail_iter;
        c->last_ovf_rows = hd.overflow_rows;
        c->last_req = hd.required;
        return ELLPACK_ERR_OVERFLOW;
    }
    stop = hd.stop;
    return ELLPACK_OK;
}

}  // namespace

int sp2_run(ellpack_ctx c, const ellpack_desc* h, int64_t nocc, double tol, const sp2_opts* opts_in,
            ellpack_desc* dout, sp2_report* rep) {
    if (!c) return ELLPACK_ERR_ARG;
    RK(check_desc(h));
    RK(check_desc(dout));
    const int64_t n = h->n;
    if (dout->n != n) return ELLPACK_ERR_DIM;
    RK(check_comm_n(c, n));
    if (nocc < 0 || nocc > n || !(tol >= 0.0)) return ELLPACK_ERR_ARG;
    {
        // a row block without a communicator cannot see the other rows of X_{n+1}
        int64_t q0, q1;
        rows_of(c, n, &q0, &q1);
        if (!c->comm && (q0 != 0 || q1 != n)) return ELLPACK_ERR_STATE;
    }
    sp2_opts o;
    if (opts_in) o = *opts_in; else sp2_opts_default(&o);
    c->dense_fit_key = -1;  // free memory is asked again once per run
    if (!valid_tau(o.threshold) || o.max_iter < 1) return ELLPACK_ERR_ARG;
    if (o.branch_rule != SP2_RULE_TRACE_SIGN && o.branch_rule != SP2_RULE_TRACE_CLOSEST) return ELLPACK_ERR_ARG;
    CK(cudaSetDevice(c->device));
    RK(validate_inputs(c, {h}));
    sp2_iter_rec* iters = rep ? rep->iters : nullptr;
    sp2_report R;
    memset(&R, 0, sizeof R);
    R.iters = iters;
    R.fail_iter = 0;
    const double t_start = now_s();

    // ---- Init Misc: bounds, X0, tr(X0)
    NvtxRange phase("SP2 Init Misc");
    double emin = o.emin, emax = o.emax;
    if (std::isnan(emin) || std::isnan(emax)) RK(gershgorin_impl(c, h, &emin, &emax));
    R.emin = emin;
    R.emax = emax;
    const double dl = emax - emin;
    if (!(dl > 0.0) || !std::isfinite(dl)) {
        if (rep) *rep = R;
        return ELLPACK_ERR_BOUNDS;
    }
    const double alpha0 = -1.0 / dl, beta0 = emax / dl;
    const int32_t maxw = o.max_width > 0 ? ((o.max_width + 1) & ~1) : (int32_t)((n + 1) & ~int64_t(1));
    int32_t w = c->sp2_width0 > 0 ? c->sp2_width0 : (o.initial_width > 0 ? o.initial_width : h->w);
    w = (w + 1) & ~1;
    const double t_read_end = now_s();
    DevMatrix X, Y, T, U;
    X.slot = 0;
    Y.slot = 1;
    T.slot = 2;
    U.slot = 3;  // symmetric step: the upper triangle of X_{n+1}
    int status = ELLPACK_OK;
    int32_t req = 0;
    auto cleanup = [&]() { dm_free(c, X); dm_free(c, Y); dm_free(c, T); dm_free(c, U); };
    // Symmetric step (§8f-f4 ii): with H bitwise symmetric every iterate is (P4), so general-path
    // steps compute only the upper triangle and mirror it. GROW policy (FAIL needs the exact
    // overflow row count of a step, which a truncated upper triangle cannot give). With a
    // communicator each rank checks its own rows (the flag is all-reduced) and the U rows of lower
    // ranks its rows mirror arrive by a second halo.
    bool sym = false, sym_off = false;
    if (c->sp2_sym && o.on_overflow == SP2_GROW) {
        RK(grow(c, c->symaux, 4 * sizeof(int32_t)));
        int32_t* aux = (int32_t*)c->symaux.p;
        int64_t q0, q1;
        rows_of(c, n, &q0, &q1);
        CK(cudaMemsetAsync(aux, 0, sizeof(int32_t), c->stream));
        CK(launch_sym_check(kmat(h), q0, q1, aux, c->stream));  // this rank's rows (H is replicated)
        c->launches++;
        if (c->comm) NK(g_nccl.AllReduce(aux, aux, 1, ncclInt32, ncclMax, c->comm, c->stream));
        int32_t asym = 1;
        CK(cudaMemcpyAsync(&asym, aux, sizeof asym, cudaMemcpyDeviceToHost, c->stream));
        RK(host_sync(c));
        sym = asym == 0;
    }
    // the dense regime across ranks (symmetric X): every rank must take the same regime every step,
    // so the choice uses only all-reduced inputs -- here the smallest free memory of any rank
    bool dense_comm_ok = false, dense_comm_alloc = false;
    if (c->comm && sym && c->dense_opt != 1 && n <= kDenseMaxN) {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); fr = 0; }
        unsigned long long f64 = fr;
        CK(cudaMemcpyAsync(c->d_keys + 6, &f64, 8, cudaMemcpyHostToDevice, c->stream));
        NK(g_nccl.AllReduce(c->d_keys + 6, c->d_keys + 6, 1, ncclUint64, ncclMin, c->comm, c->stream));
        CK(cudaMemcpyAsync(&f64, c->d_keys + 6, 8, cudaMemcpyDeviceToHost, c->stream));
        RK(host_sync(c));
        const double npd = (double)dense_np(n);
        dense_comm_ok = 2.0 * 8.0 * npd * npd <= 0.6 * (double)f64;
    }
    int rc = sp2_make_x0(c, h, alpha0, beta0, o.threshold, T, &req);
    if (rc) { cleanup(); return rc; }
    if (req > w) {
        if (o.on_overflow == SP2_FAIL || req > maxw) {
            int64_t ovf = 0;
            if ((rc = count_rows_over(c, &T.d, w, &ovf))) { cleanup(); return rc; }
            R.stop_reason = SP2_OVERFLOWED; R.required_width = req; R.fail_iter = -1;
            R.overflow_rows = ovf;
            c->last_req = req;
            c->last_ovf_rows = ovf;
            cleanup();
            if (rep) *rep = R;
            return ELLPACK_ERR_OVERFLOW;
        }
        w = round_up32(req) < maxw ? round_up32(req) : maxw;
        R.regrows++;
    }
    int64_t r0, r1;
    rows_of(c, n, &r0, &r1);
    if ((rc = dm_alloc(c, X, n, w))) { cleanup(); return rc; }
    CK(cudaMemsetAsync(c->d_status, 0, 8, c->stream));
    CK(launch_copy_rows(kmat(&T.d), kout(&X.d), r0, r1, c->d_status, c->stream));
    c->launches++;
    dm_free(c, T);
    if ((rc = halo_desc(c, &X.d, &X.d))) { cleanup(); return rc; }  // rows X0's rows reference
    double trX;
    if ((rc = ellpack_trace(c, &X.d, &trX))) { cleanup(); return rc; }
    // trace-closest rule (SP2_RULE_TRACE_CLOSEST): T2 of X0 here, of X_{n+1} after step n
    const bool closest = o.branch_rule == SP2_RULE_TRACE_CLOSEST;
    double t2 = 0.0;
    RK(grow(c, c->rows[3], sizeof(double) * n));
    if (closest) {
        CK(launch_sumsq_rows(kmat(&X.d), r0, r1, (double*)c->rows[3].p, c->stream));
        c->launches++;
        const double* arrs[1] = {(const double*)c->rows[3].p};
        if ((rc = enqueue_canonical(c, arrs, 1, n))) { cleanup(); return rc; }
        CK(cudaMemsetAsync(c->d_status, 0, 8, c->stream));
        if ((rc = fetch(c, 1))) { cleanup(); return rc; }
        t2 = c->h->sums[0];
    }
    // the probe of X0 (its halo rows are in place), for the first step's launch plan
    int32_t bwX[kProbe];
    std::vector<int64_t> needX(2 * (size_t)c->nranks);
    if ((rc = enqueue_next_probe(c, &X.d))) { cleanup(); return rc; }
    if ((rc = fetch(c, 0, true))) { cleanup(); return rc; }
    take_probe(c, bwX, needX);
    const double t_init_end = now_s();
    phase.next("SP2 Loop (X2 + Norm + Misc)");

    // ---- SP2 loop
    // One host synchronisation per iteration: the step's status, traces, norm, product count,
    // the probe of X_{n+1} and (with a communicator) every rank's reach arrive in one read-back;
    // the next step's launch plan and halo exchange are computed from them without waiting.
    RK(grow(c, c->rows[0], sizeof(double) * n));
    RK(grow(c, c->rows[1], sizeof(double) * n));
    RK(grow(c, c->rows[2], sizeof(double) * n));
    double t_x2 = 0.0, t_norm = 0.0;
    double e_hist[2] = {NAN, NAN};
    // Widths. The GROW reading (§8c-c10 iv) fixes the LOGICAL width sequence (round_up32 of the
    // required width whenever it is exceeded) that the report records, exactly as the oracle.
    // The PHYSICAL width of the iterate buffer may be larger: it is allocated with headroom
    // (x 8 of the initial width, x 4 of the required width on a physical overflow), so an
    // iteration whose logical width grows is recomputed only when the physical one overflows.
    // Values and patterns do not depend on the storage width.
    int32_t wy = w;       // logical width of X_{n+1}
    int32_t wx = w;       // logical width of X_n
    // physical width of the Y buffer: headroom from the start (gapless fills grow several-fold per
    // early iteration; only FAIL keeps physical == logical so overflow counts stay exact)
    int32_t wcap = o.on_overflow == SP2_FAIL ? w : (int32_t)std::min<int64_t>(maxw, round_up32((int64_t)w * 8));
    int stop = -1;
    int it;
    double p_prev = 0.0, p_prev2 = 0.0;  // products of the last two steps (dense-regime decision)
    // measured rates of the two regimes (pattern products / s of a sparse step; GEMM FMAs / s of a
    // dense step, densify and epilogue included), seeded below the long steps' rates of cfg3 and cfg4
    // (tools/dense_switch.py, profiles/r02_dense_switch_*.log)
    double rate_sparse = 5e11, rate_dense = 1e13;  // (dense: FMAs / s)
    double rate_sparse_seen = 0.0;
    bool dense_tried = false;  // a dense step ran in this run (its rate replaced the seed)
    bool dense_off = false;    // the dense arrays could not be allocated: sparse kernels for the rest
    // X_{n+1}'s exact dense work is measured after every step while the automatic regime may pick dense
    // (symmetric X, one rank): w_next FMAs, 0 = not measured
    const bool measure_work = sym && !c->comm && c->dense_opt == 0 && n <= kDenseMaxN;
    double w_next = 0.0;
    UpperAlloc ua{&U, n, 0};
    bool halo_pending = false;  // the halo of X_n travels on the side stream (communicator only)
    const bool dev_loop = use_device_loop(c, n, maxw, sym);
    if (dev_loop) {
        // (§8f-f3) the whole loop as one graph launch: zero host synchronisations per iteration
        double t_loop = 0.0;
        it = 0;
        rc = sp2_device_loop(c, o, n, nocc, tol, w, maxw, closest, sym, trX, t2, X, Y, R, iters, wx, stop, it,
                             t_loop);
        if (rc) status = rc;
        t_x2 = t_loop;
    }
    if (!dev_loop)
    for (it = 0; it < o.max_iter; ++it) {
        int branch = (trX > (double)nocc) ? SP2_SQUARE : SP2_EXPAND;
        if (closest)  // (same expression as the oracle: tie -> EXPAND)
            branch = (std::fabs(t2 - (double)nocc) < std::fabs((2.0 * trX - t2) - (double)nocc)) ? SP2_SQUARE
                                                                                                : SP2_EXPAND;
        if (!Y.owned || Y.d.w < wy) {
            int32_t want = wcap > wy ? wcap : wy;
            if ((rc = dm_alloc_headroom(c, Y, n, want, wy))) { status = rc; break; }
            if (want < wcap) wcap = want;
        }
        // scalar products of this X^2 (this rank's rows; summed over ranks below)
        CK(cudaMemsetAsync(c->d_keys + 2, 0, 8, c->stream));
        {
            int64_t pr0, pr1;
            rows_of(c, n, &pr0, &pr1);
            CK(launch_products(kmat(&X.d), X.d.nnz, pr0, pr1, c->d_keys + 2, c->stream));
            c->launches++;
            if (c->comm) {
                NK(g_nccl.AllReduce(c->d_keys + 2, c->d_keys + 2, 1, ncclUint64, ncclSum, c->comm, c->stream));
            }
            // read back with the step's status/sums (same stream, no extra synchronisation)
            CK(cudaMemcpyAsync(&c->h->keys[0], c->d_keys + 2, 8, cudaMemcpyDeviceToHost, c->stream));
        }
        // the regime of this step (dense.cu or the sparse kernels): forced, or the one whose predicted
        // time is lower. Sparse: the products P of the step (the last step's, times its growth) at the
        // pattern-product rate the last sparse step achieved. Dense: the GEMM's FMAs over the k blocks
        // inside X_n's band (dense_band_fmas: every 128 x 16 block within the probe's half-bandwidth
        // counted as occupied) at the rate the last dense step achieved on that count.
        bool dense_step = false;
        double w_dense = 0.0, p_est = 0.0;
        if (c->dense_opt != 1 && !dense_off && (c->comm ? dense_comm_ok : dense_fits(c, n, sym ? 2 : 3))) {
            // the GEMM's exact work when the last step measured X_n's block occupancy (symmetric X),
            // else the band model
            // (across ranks every rank computes all tiles of its rows: no mirrored half)
            w_dense = w_next > 0.0 ? w_next : dense_band_fmas(n, std::max(bwX[0], bwX[1]), sym && !c->comm);
            if (c->dense_opt == 2) {
                dense_step = true;
            } else if (p_prev > 0.0) {
                // (growth per step <= 2: cfg3's early steps grow 1.5-1.9x once past X0)
                const double g = p_prev2 > 0.0 ? std::min(2.0, std::max(1.0, p_prev / p_prev2)) : 1.0;
                p_est = p_prev * g;
                const double t_d = w_dense / rate_dense, t_s = p_est / rate_sparse;
                dense_step = t_d < (dense_tried ? 0.95 : 0.85) * t_s;  // (a measured dense rate: a thinner margin)
                // the band model counts every block inside the band as occupied: iterates with holes in
                // their band (cfg4's lattice) run faster than it predicts, which only a measured dense
                // step reveals -- one exploratory dense step per run when the prediction is close
                if (!dense_step && !dense_tried && t_s > 5e-3 && t_d < 1.5 * t_s) dense_step = true;
                if (getenv("ELLPACK_DEBUG_REGIME"))
                    fprintf(stderr, "[regime] it %d w %.3e (%s) rate_d %.3e t_d %.3f ms | P_est %.3e rate_s %.3e t_s %.3f ms -> %s\n",
                            it, w_dense, w_next > 0.0 ? "exact" : "band", rate_dense, t_d * 1e3, p_est, rate_sparse,
                            t_s * 1e3, dense_step ? "dense" : "sparse");
            }
        }
        if (dense_step && c->comm && !dense_comm_alloc) {
            // the first dense step of a run across ranks: every rank allocates, then all agree (MIN of
            // the success flags) -- a rank that could not falls back with the others, never alone
            dense_comm_alloc = true;
            const int64_t np = dense_np(n);
            const size_t bytes = sizeof(double) * (size_t)np * (size_t)np;
            const size_t fl = 2 * (size_t)(np / kDenseTile) * (size_t)(np / kDenseK) +
                              2 * (size_t)(np / kDenseTile) * dense_kbw((int)np) * 8 +
                              (size_t)(np / 16) * (size_t)(np / kDenseTile);
            unsigned long long okv = (grow(c, c->dense[0], bytes) == ELLPACK_OK && grow(c, c->dense[2], bytes) == ELLPACK_OK &&
                                      grow(c, c->dflags, fl) == ELLPACK_OK) ? 1ull : 0ull;
            cudaGetLastError();
            CK(cudaMemcpyAsync(c->d_keys + 6, &okv, 8, cudaMemcpyHostToDevice, c->stream));
            NK(g_nccl.AllReduce(c->d_keys + 6, c->d_keys + 6, 1, ncclUint64, ncclMin, c->comm, c->stream));
            CK(cudaMemcpyAsync(&okv, c->d_keys + 6, 8, cudaMemcpyDeviceToHost, c->stream));
            RK(host_sync(c));
            if (!okv) {
                dense_comm_ok = false;
                dense_step = false;
            }
        }
        c->last_dense = 0;
        bool redo;
        int32_t kept_max = 0;
        double step_ms = 0.0;
        do {
            redo = false;
            RowOpParams p = base_params(c, n);
            p.A = kmat(&X.d);
            p.B = kmat(&X.d);
            p.Old = kmat(&X.d);
            p.C = kout(&Y.d);
            p.tau = o.threshold;
            if (branch == SP2_SQUARE) { p.alpha = 1.0; p.beta = 0.0; p.old_mode = 2; }
            else { p.alpha = -1.0; p.beta = 2.0; p.old_mode = 1; }
            p.diag_s = (double*)c->rows[0].p;
            p.diag_c = (double*)c->rows[1].p;
            p.normsq = (double*)c->rows[2].p;
            p.upper = sym && !sym_off && !dense_step;  // taken only if the general path runs (enqueue_row_op)
            if (p.upper && c->comm && (!U.owned || U.d.w != Y.d.w)) {
                // every rank must take the upper route together: U at the agreed width, or none
                int32_t want = Y.d.w;
                if (dm_alloc_headroom(c, U, n, want, Y.d.w) != ELLPACK_OK || want != Y.d.w) {
                    cudaGetLastError();
                    dm_free(c, U);
                    sym_off = true;
                    p.upper = 0;
                }
            }
            CK(cudaMemsetAsync(c->d_keys + 4, 0, 8, c->stream));
            p.exec_products = c->d_keys + 4;
            ua.w = Y.d.w;
            cudaEventRecord(c->ev[0], c->stream);
            // with a communicator the halo of X_n (started after the previous step) is in flight:
            // the interior rows run beside it, the boundary rows after it (§8f-f1)
            if (dense_step) {
                rc = enqueue_dense_op(c, p, n, sym, bwX, halo_pending);
                if (rc == ELLPACK_ERR_NOMEM && !c->comm) {
                    // the dense arrays did not fit after all (fragmentation): this step and the rest of
                    // the run on the sparse kernels (same bits). With a communicator the arrays were
                    // allocated and agreed on before the first dense step.
                    cudaGetLastError();
                    release(c, c->dense[0]);
                    release(c, c->dense[1]);
                    release(c, c->dense[2]);
                    c->dense_clean_np = 0;
                    c->dense_fit_key = -2;  // (a key no (N_p, arrays) pair has: asks the driver again)
                    dense_step = false;
                    dense_off = true;
                    c->last_dense = 0;
                    rc = enqueue_row_op(c, p, n, bwX, alloc_upper, &ua);
                }
            } else if (c->comm) {
                rc = enqueue_row_op_split(c, p, n, bwX, halo_pending, alloc_upper, &ua);
            } else {
                rc = enqueue_row_op(c, p, n, bwX, alloc_upper, &ua);
            }
            if (rc) { status = rc; break; }
            halo_pending = false;
            if (c->sym_nomem) sym_off = true;  // U did not fit: whole rows from now on
            const bool upper = c->last_upper != 0;
            if (upper) {
                // U's status aside, then X_{n+1} row i = L_i || U_i with the step's status
                int32_t* aux = (int32_t*)c->symaux.p;
                CK(cudaMemcpyAsync(aux + 2, c->d_status, 2 * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->stream));
                if (c->comm) {
                    // every rank redoes an overflowed upper triangle together
                    NK(g_nccl.GroupStart());
                    NK(g_nccl.AllReduce(aux + 2, aux + 2, 1, ncclInt32, ncclSum, c->comm, c->stream));
                    NK(g_nccl.AllReduce(aux + 3, aux + 3, 1, ncclInt32, ncclMax, c->comm, c->stream));
                    NK(g_nccl.GroupEnd());
                    // L_i needs column i of the U rows j in [i - reach, i); U_j ends by j + 2 h_X
                    // (X_{n+1} lies within the band of X_n^2), so rank q reads the U rows
                    // [r0_q - 2 h_X, r0_q) of lower ranks: a second, one-sided halo
                    std::vector<int64_t> needU(2 * (size_t)c->nranks);
                    const int64_t per = r1 - r0;
                    for (int q = 0; q < c->nranks; ++q) {
                        needU[2 * q] = std::max<int64_t>(0, (int64_t)q * per - 2 * (int64_t)bwX[0]);
                        needU[2 * q + 1] = (int64_t)(q + 1) * per - 1;
                    }
                    if ((rc = halo_exec(c, &U.d, needU.data()))) { status = rc; break; }
                }
                CK(cudaMemcpyAsync(c->h->status_u, aux + 2, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
                CK(cudaMemsetAsync(c->d_status, 0, 2 * sizeof(int32_t), c->stream));
                CK(cudaMemsetAsync(aux + 1, 0, sizeof(int32_t), c->stream));
                CK(launch_upper_reach(kmat(&U.d), r0, r1, aux + 1, c->stream));
                if (c->comm) NK(g_nccl.AllReduce(aux + 1, aux + 1, 1, ncclInt32, ncclMax, c->comm, c->stream));
                CK(launch_sym_assemble(kmat(&U.d), kmat(&X.d), kout(&Y.d), r0, r1, aux + 1, p.diag_s, p.normsq,
                                       c->d_status, c->num_sms, c->stream));
                c->launches += 2;
            }
            if (c->comm)
                NK(g_nccl.AllReduce(c->d_keys + 4, c->d_keys + 4, 1, ncclUint64, ncclSum, c->comm, c->stream));
            CK(cudaMemcpyAsync(&c->h->keys[1], c->d_keys + 4, 8, cudaMemcpyDeviceToHost, c->stream));
            c->last_step_general = !p.fast;
            cudaEventRecord(c->ev[1], c->stream);
            if ((rc = reduce_status(c))) { status = rc; break; }
            if (closest) {
                // T2 of X_{n+1} (this rank's rows), summed with this step's traces
                CK(launch_sumsq_rows(kmat(&Y.d), r0, r1, (double*)c->rows[3].p, c->stream));
                c->launches++;
            }
            const double* arrs[4] = {p.diag_s, p.diag_c, p.normsq, (const double*)c->rows[3].p};
            const int narr = closest ? 4 : 3;
            if ((rc = enqueue_canonical(c, arrs, narr, n))) { status = rc; break; }
            // the probe of X_{n+1} for the next step (its own rows; reaches all-gathered)
            if ((rc = enqueue_next_probe(c, &Y.d))) { status = rc; break; }
            if (measure_work) {
                // the next step's dense work, exactly: occupancy bitsets of X_{n+1}, then the occupied
                // (tile, k block) pairs of the symmetric GEMM -- read back with this step's status
                const int64_t np = dense_np(n);
                const size_t fw = (size_t)(np / kDenseTile) * (size_t)((np / kDenseK + 63) / 64);
                RK(grow(c, c->docc, fw * 8));
                CK(cudaMemsetAsync(c->docc.p, 0, fw * 8, c->stream));
                CK(cudaMemsetAsync(c->d_keys + 5, 0, 8, c->stream));
                CK(launch_occupancy(kmat(&Y.d), n, (int)np, (unsigned long long*)c->docc.p, c->num_sms, c->stream));
                CK(launch_dense_work((const unsigned long long*)c->docc.p, (int)np, c->d_keys + 5, c->num_sms,
                                     c->stream));
                c->launches += 2;
                CK(cudaMemcpyAsync(&c->h->keys[2], c->d_keys + 5, 8, cudaMemcpyDeviceToHost, c->stream));
            }
            cudaEventRecord(c->ev[2], c->stream);
            if ((rc = fetch(c, narr, true))) { status = rc; break; }
            float ms1 = 0.f, ms2 = 0.f;
            cudaEventElapsedTime(&ms1, c->ev[0], c->ev[1]);
            cudaEventElapsedTime(&ms2, c->ev[1], c->ev[2]);
            t_x2 += ms1 * 1e-3;
            t_norm += ms2 * 1e-3;
            step_ms = ms1;
            if (upper && c->h->status_u[0] > 0) {
                // the upper triangle overflowed its buffer (so does X_{n+1}): the step's counts are
                // not exact -- grow the physical width (or, at the ceiling, take the full path) and
                // redo the step before any logical decision
                if (wcap >= maxw) {
                    sym_off = true;
                } else {
                    const int64_t want = round_up32((int64_t)c->h->status_u[1] * 4);
                    wcap = (int32_t)std::min<int64_t>(maxw, std::max<int64_t>(want, (int64_t)wcap * 2));
                    const int32_t need = std::min<int32_t>(maxw, std::max<int32_t>(Y.d.w + 32,
                                                                                   round_up32(c->h->status_u[1])));
                    if ((rc = dm_alloc_headroom(c, Y, n, wcap, need))) { status = rc; break; }
                }
                redo = true;
                continue;
            }
            kept_max = c->h->status[1];
            if (kept_max > wy) {
                // the logical width grows (the oracle's regrow)
                if (o.on_overflow == SP2_FAIL || kept_max > maxw) {
                    // rows over the LOGICAL width wy: the step's status counts rows over the
                    // physical width; when that is wider, Y's stored counts min(kept, physical)
                    // exceed wy exactly for the rows whose kept count does
                    int64_t ovf = c->h->status[0];
                    if (Y.d.w > wy && (rc = count_rows_over(c, &Y.d, wy, &ovf))) { status = rc; break; }
                    R.stop_reason = SP2_OVERFLOWED;
                    R.overflow_rows = ovf;
                    R.required_width = kept_max;
                    R.fail_iter = it;
                    c->last_ovf_rows = R.overflow_rows;
                    c->last_req = kept_max;
                    status = ELLPACK_ERR_OVERFLOW;
                    break;
                }
                wy = round_up32(kept_max) < maxw ? round_up32(kept_max) : maxw;
                R.regrows++;
            }
            if (c->h->status[0] > 0) {
                // the physical buffer overflowed: re-create it with headroom and redo step n
                // (deterministic: the same values)
                // headroom x4: the fill of gapless iterates grows 2.5-4x per early iteration
                const int64_t want = round_up32((int64_t)kept_max * 4);
                wcap = (int32_t)(want < maxw ? want : maxw);
                if (wcap < wy) wcap = wy;
                const int32_t need = std::max<int32_t>(wy, std::min<int32_t>(maxw, round_up32(kept_max)));
                if ((rc = dm_alloc_headroom(c, Y, n, wcap, need))) { status = rc; break; }
                redo = true;
            }
        } while (redo);
        if (status != ELLPACK_OK) break;
        const double trS = c->h->sums[0];
        const double trY = c->h->sums[1];
        const double fn = std::sqrt(c->h->sums[2]);
        const double e = trX - trS;
        if (iters) {
            iters[it].trX = trX;
            iters[it].trS = trS;
            iters[it].e = e;
            iters[it].fnorm = fn;
            iters[it].branch = branch;
            iters[it].width = wy;
            iters[it].required = kept_max;
            iters[it].regime = c->last_dense;
            iters[it].products = (int64_t)c->h->keys[0];  // landed with the status fetch
            iters[it].frob2 = t2;
            // products executed: the general kernel counts them; the ring path runs all of them
            iters[it].products_exec = c->last_step_general ? (int64_t)c->h->keys[1] : (int64_t)c->h->keys[0];
            iters[it].step_ms = step_ms;
        }
        if (closest) t2 = c->h->sums[3];
        p_prev2 = p_prev;
        p_prev = (double)c->h->keys[0];
        if (measure_work) w_next = (double)c->h->keys[2] * kDenseK * kDenseTile * kDenseTile;
        // the rates the next regime choice predicts with (device time of this step)
        // (only steps long enough for their rate to carry over: short sparse steps run far below the
        // rate of the long ones -- cfg4's iteration 1 at 1.4e11 products/s, iteration 5 at 7.8e11)
        // (a dense step that zeroed the whole N_p^2 array -- the first of a context -- and a run's first
        // step carry one-time costs; sparse steps grow more efficient with size: the best rate seen)
        // (with a communicator the rates stay the seeds: a rank's own step time must not steer a choice
        // every rank has to make alike)
        if (c->last_dense) {
            dense_tried = true;
            if (!c->comm && step_ms >= 1.0 && !c->dense_full_clear && w_dense > 0.0)
                rate_dense = w_dense / (step_ms * 1e-3);
        } else if (!c->comm && it >= 1 && step_ms >= 10.0 && p_prev >= 1e10) {
            rate_sparse_seen = std::max(rate_sparse_seen, p_prev / (step_ms * 1e-3));
            rate_sparse = rate_sparse_seen;
        }
        take_probe(c, bwX, needX);
        // the next step reads only the rows of X_{n+1} its rows reference (band-aware halo, f1),
        // planned from the reaches that arrived with this step's status
        if (c->comm) {
            if ((rc = start_halo(c, &Y.d, needX.data()))) { status = rc; break; }
            halo_pending = true;
        }
        std::swap(X, Y);
        wx = wy;
        trX = trY;
        if (std::fabs(e) <= tol) stop = SP2_CONVERGED;
        else if (it + 1 >= o.min_iter && e <= o.stag_gate && !std::isnan(e_hist[0]) && e >= e_hist[0])
            stop = SP2_STAGNATED;
        else if (it + 1 == o.max_iter) stop = SP2_MAXITER;
        e_hist[0] = e_hist[1];
        e_hist[1] = e;
        if (stop >= 0) { ++it; break; }
    }
    const double t_loop_end = now_s();
    phase.next("SP2 final iterate");
    if (halo_pending) CK(cudaStreamWaitEvent(c->stream, c->sev[1], 0));  // before D is assembled
    R.iterations = it;
    R.final_width = X.owned ? wx : 0;
    R.trD = trX;
    if (status == ELLPACK_OK) {
        R.stop_reason = stop;
        RK(allgather_desc(c, &X.d));  // D is replicated: every block of the final iterate
        CK(cudaMemsetAsync(c->d_status, 0, 8, c->stream));
        CK(launch_copy_rows(kmat(&X.d), kout(dout), 0, n, c->d_status, c->stream));
        c->launches++;
        RK(fetch(c, 0));
        if (c->h->status[0] > 0) {
            R.required_width = c->h->status[1];
            c->last_req = c->h->status[1];
            c->last_ovf_rows = c->h->status[0];
            status = ELLPACK_ERR_OVERFLOW;
        } else if (stop == SP2_MAXITER) {
            status = ELLPACK_ERR_NOCONV;
        }
    }
    cleanup();
    c->host_syncs++;
    cudaStreamSynchronize(c->stream);
    R.t_read_hamiltonian = t_read_end - t_start;
    R.t_init_misc = t_init_end - t_read_end;
    R.t_sp2_loop_x2 = t_x2;
    R.t_sp2_loop_norm = t_norm;
    R.t_sp2_loop_misc = (t_loop_end - t_init_end) - t_x2 - t_norm;
    if (rep) *rep = R;
    return status;
}

int ellpack_row_split(int64_t r0, int64_t r1, int64_t h, int64_t out[6]) {
    if (!out || r0 < 0 || r1 < r0 || h < 0) return ELLPACK_ERR_ARG;
    const int64_t i0 = std::min(r1, r0 + h), i1 = std::max(i0, r1 - h);
    out[0] = i0;  // interior [i0, i1): every column within [r0, r1)
    out[1] = i1;
    out[2] = r0;  // boundary [r0, i0) and [i1, r1)
    out[3] = i0;
    out[4] = i1;
    out[5] = r1;
    return ELLPACK_OK;
}

int ellpack_multiply_x2_halo(ellpack_ctx c, ellpack_desc* x, ellpack_desc* x2, double tau, double* trace_x,
                             double* trace_x2) {
    if (!c) return ELLPACK_ERR_ARG;
    RK(check_desc(x));
    RK(check_desc(x2));
    if (x->n != x2->n) return ELLPACK_ERR_DIM;
    RK(check_comm_n(c, x->n));
    if (!valid_tau(tau)) return ELLPACK_ERR_ARG;
    if (same(x, x2)) return ELLPACK_ERR_ARG;
    NvtxRange nv("ellpack_multiply_x2_halo (halo || interior rows, then boundary rows)");
    CK(cudaSetDevice(c->device));
    RK(validate_inputs(c, {x}));
    const int64_t n = x->n;
    int64_t r0, r1;
    rows_of(c, n, &r0, &r1);
    RK(grow(c, c->rows[0], sizeof(double) * n));
    RK(grow(c, c->rows[1], sizeof(double) * n));
    // 1. the probe of this rank's rows (maxima all-reduced, reaches all-gathered): one read-back
    RK(enqueue_next_probe(c, x));
    RK(fetch(c, 0, true));
    int32_t bwv[kProbe];
    std::vector<int64_t> need(2 * (size_t)c->nranks);
    take_probe(c, bwv, need);
    // 2. the band-aware halo on the side stream, beside the interior rows
    if (c->comm) RK(start_halo(c, x, need.data()));
    // 3-4. interior rows now, boundary rows once the halo is in
    RowOpParams p = base_params(c, n);
    p.A = kmat(x);
    p.B = kmat(x);
    p.C = kout(x2);
    p.alpha = 1.0;
    p.tau = tau;
    p.diag_a = (double*)c->rows[0].p;
    p.diag_s = (double*)c->rows[1].p;
    RK(enqueue_row_op_split(c, p, n, bwv, c->comm != nullptr));
    // 5. traces from this rank's rows (canonical partials all-gathered), status all-reduced
    const double* arrs[2] = {p.diag_a, p.diag_s};
    RK(enqueue_canonical(c, arrs, 2, n));
    RK(reduce_status(c));
    RK(fetch(c, 2));
    RK(finish_status(c));
    if (trace_x) *trace_x = c->h->sums[0];
    if (trace_x2) *trace_x2 = c->h->sums[1];
    return ELLPACK_OK;
}

int ellpack_multiply_x2_host(ellpack_ctx c, int64_t n, int32_t wx, const double* xv, const int32_t* xc,
                             const int32_t* xn, int32_t wx2, double* yv, int32_t* yc, int32_t* yn,
                             double tau, double* trace_x, double* trace_x2) {
    if (!c || n <= 0 || wx <= 0 || wx2 <= 0 || (wx & 1) || (wx2 & 1) || !xv || !xc || !xn || !yv || !yc || !yn)
        return ELLPACK_ERR_ARG;
    CK(cudaSetDevice(c->device));
    const size_t cx = (size_t)n * wx, cy = (size_t)n * wx2;
    RK(grow(c, c->hx_val, cx * 8));
    RK(grow(c, c->hx_col, cx * 4));
    RK(grow(c, c->hx_nnz, n * 4));
    RK(grow(c, c->hy_val, cy * 8));
    RK(grow(c, c->hy_col, cy * 4));
    RK(grow(c, c->hy_nnz, n * 4));
    ellpack_desc X{n, wx, 0, (double*)c->hx_val.p, (int32_t*)c->hx_col.p, (int32_t*)c->hx_nnz.p};
    ellpack_desc Y{n, wx2, 0, (double*)c->hy_val.p, (int32_t*)c->hy_col.p, (int32_t*)c->hy_nnz.p};
    CK(cudaMemcpyAsync(X.val, xv, cx * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(X.col, xc, cx * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(X.nnz, xn, n * 4, cudaMemcpyHostToDevice, c->stream));
    double tx = 0, tx2 = 0;
    int rc = ellpack_multiply_x2(c, &X, &Y, tau, &tx, &tx2);
    if (rc != ELLPACK_OK && rc != ELLPACK_ERR_OVERFLOW) return rc;
    // this rank's rows of X^2 (all rows on one rank) come back
    int64_t r0, r1;
    rows_of(c, n, &r0, &r1);
    const size_t o0 = (size_t)r0 * wx2, cr = (size_t)(r1 - r0) * wx2;
    CK(cudaMemcpyAsync(yv + o0, Y.val + o0, cr * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(yc + o0, Y.col + o0, cr * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(yn + r0, Y.nnz + r0, (size_t)(r1 - r0) * 4, cudaMemcpyDeviceToHost, c->stream));
    RK(host_sync(c));
    if (rc == ELLPACK_OK) {
        if (trace_x) *trace_x = tx;
        if (trace_x2) *trace_x2 = tx2;
    }
    return rc;
}

}  // extern "C"
