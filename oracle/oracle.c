/*
 * oracle/oracle.c — plain, slow, obviously-correct CPU oracle for the hot path
 * of arXiv 2102.08505 (BML ELLPACK multiply with drop threshold + SP2 loop).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library. The
 * product path (paper_2102_08505_b200/) never imports, links or calls it, and
 * this file shares no code, header or helper with it.
 *
 * Citations: P:Lnn = /root/reference/PAPER.md line nn, S:Lnn = SPEC.md line nn,
 * "§8c-cN" = SURVEY.md §8(c) oracle item cN (the readings listed in DESIGN.md).
 *
 *  - multiply  C <- drop_tau(alpha*A*B + beta*C)            §8c-c2,c3,c4
 *  - x2        X2 <- drop_tau(X*X), tr(X), tr(X^2) pre-drop  §8c-c5
 *  - add / add_identity / scale_add_identity                 §8c-c6
 *  - trace (canonical 256-row-block sum)                     §8c-c7
 *  - fnorm_diff                                              §8c-c11
 *  - gershgorin                                              §8c-c8
 *  - sp2 (init + loop + stop rule)                           §8c-c9,c10
 *  - sp2 trace-closest branch rule (option)                  §8f-f4 (i); P:L52 (Niklasson 2002)
 *
 * Floating point: IEEE binary64, round-to-nearest-even. Every product-sum is
 * the explicit C99 fma() of the definition; the file is compiled with
 * -ffp-contract=off and never with -ffast-math, so the compiler cannot fuse or
 * reorder anything (reading S12).
 *
 * Accumulator (S:L106 design decision): a dense scratch row of length n plus a
 * touched list, sorted at row end. Rows are independent ("row-parallel
 * execution over disjoint output rows"), so an OpenMP parallel-for over rows
 * gives the same bits for any thread count.
 *
 * Parity pins: see tests/test_oracle_*.py (dense brute force with exact
 * rational fma, numpy GEMM, closed forms, symmetry, eigh projector, dimer
 * closed form, hand vectors in tests/golden/; the c6 single rounding and the
 * c10 (vi) stop rule in tests/test_oracle_pins_c6_c10.py). tools/oracle_mutants.py
 * applies plausible mistakes to this file and checks that a pin fails for each.
 * Functions without an external pin are marked "parity unpinned" below;
 * currently none.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t n;
    int32_t w;
    double* val;
    int32_t* col;
    int32_t* nnz;
} omat;

enum { O_OK = 0, O_ARG = 1, O_DIM = 2, O_OVERFLOW = 3, O_BOUNDS = 4, O_NOCONV = 5, O_NOMEM = 6 };

/* ------------------------------------------------------------ canonical sum
 * §8c-c7: blocks of 256 consecutive rows, T_b = ((0 + d_256b) + d_256b+1) + ...
 * left to right; total = ((0 + T_0) + T_1) + ... left to right. */
double oracle_canonical_sum(const double* d, int64_t n) {
    double total = 0.0;
    for (int64_t b = 0; b * 256 < n; ++b) {
        double t = 0.0;
        int64_t e = (b + 1) * 256 < n ? (b + 1) * 256 : n;
        for (int64_t i = b * 256; i < e; ++i) t = t + d[i];
        total = total + t;
    }
    return total;
}

/* block partials only (for the multi-rank emulation: T_b of rows [r0,r1), r0 % 256 == 0) */
void oracle_block_partials(const double* d, int64_t n, double* out_blocks) {
    for (int64_t b = 0; b * 256 < n; ++b) {
        double t = 0.0;
        int64_t e = (b + 1) * 256 < n ? (b + 1) * 256 : n;
        for (int64_t i = b * 256; i < e; ++i) t = t + d[i];
        out_blocks[b] = t;
    }
}

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* stored value of (i, j) in row i of M, or +0.0 with *found = 0 */
static double lookup(const omat* M, int64_t i, int32_t j, int* found) {
    const int32_t* c = M->col + (size_t)i * M->w;
    const double* v = M->val + (size_t)i * M->w;
    for (int32_t q = 0; q < M->nnz[i]; ++q)
        if (c[q] == j) { *found = 1; return v[q]; }
    *found = 0;
    return 0.0;
}

/* Per-thread scratch for one output row: dense s[n], touched mark + list. */
typedef struct {
    double* s;
    unsigned char* mark;
    int32_t* touched;
    int32_t nt;
    int32_t* ucols;  /* union columns, ascending */
    double* uval;    /* result values for ucols */
} scratch;

static int scratch_init(scratch* S, int64_t n) {
    S->s = (double*)calloc((size_t)n, sizeof(double));
    S->mark = (unsigned char*)calloc((size_t)n, 1);
    S->touched = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    S->ucols = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    S->uval = (double*)malloc(sizeof(double) * (size_t)n);
    S->nt = 0;
    return (S->s && S->mark && S->touched && S->ucols && S->uval) ? 0 : -1;
}
static void scratch_free(scratch* S) {
    free(S->s); free(S->mark); free(S->touched); free(S->ucols); free(S->uval);
}
static void touch(scratch* S, int32_t j) {
    if (!S->mark[j]) { S->mark[j] = 1; S->touched[S->nt++] = j; }
}
static void scratch_reset(scratch* S) {
    for (int32_t t = 0; t < S->nt; ++t) { S->s[S->touched[t]] = 0.0; S->mark[S->touched[t]] = 0; }
    S->nt = 0;
}

/* §8c-c2 step 2: s[j] <- fma(a_ik, b_kj, s[j]) for k ascending (A's row order),
 * then q ascending within B row k. */
static void accumulate_row(scratch* S, const omat* A, const omat* B, int64_t i) {
    const int32_t* ca = A->col + (size_t)i * A->w;
    const double* va = A->val + (size_t)i * A->w;
    for (int32_t p = 0; p < A->nnz[i]; ++p) {
        int32_t k = ca[p];
        double a = va[p];
        const int32_t* cb = B->col + (size_t)k * B->w;
        const double* vb = B->val + (size_t)k * B->w;
        for (int32_t q = 0; q < B->nnz[k]; ++q) {
            int32_t j = cb[q];
            S->s[j] = fma(a, vb[q], S->s[j]);
            touch(S, j);
        }
    }
}

/*
 * §8c-c2..c4: C <- drop_tau(alpha*A*B + beta*C_old), C_old = C (in place).
 * Row i:  1. s <- +0, touched <- {}   2. if alpha != 0: accumulate (above)
 *         3. U <- touched u (beta != 0 ? cols(C_old_i) : {}), ascending
 *         4. t <- (beta != 0 and j in C_old_i) ? beta*c_old_j : +0;  c <- fma(alpha, s_j, t)
 *         5. keep iff |c| > tau (c3), emit ascending j.
 * Overflow (c4): kept_i > C.w for some i -> O_OVERFLOW, required_width = max kept,
 * overflow_rows = #{kept_i > C.w}; C contents then unspecified (rows truncated).
 * Optional per-row outputs: diag_s[i] = pre-combine s_ii (0 if untouched).
 */
int oracle_multiply_ex(const omat* A, const omat* B, omat* C, double alpha, double beta, double tau,
                       int64_t* overflow_rows, int32_t* required_width, double* diag_s) {
    if (!A || !B || !C) return O_ARG;
    if (A->n != B->n || A->n != C->n) return O_DIM;
    if (!(tau >= 0.0) || !isfinite(tau)) return O_ARG;
    if (C->val == A->val || C->val == B->val) return O_ARG;
    int64_t n = A->n;
    int64_t ovf = 0;
    int32_t req = 0;
    int err = 0;
#pragma omp parallel reduction(+ : ovf) reduction(max : req) reduction(| : err)
    {
        scratch S;
        if (scratch_init(&S, n)) err |= 1;
        else {
#pragma omp for schedule(dynamic, 64)
            for (int64_t i = 0; i < n; ++i) {
                if (alpha != 0.0) accumulate_row(&S, A, B, i);
                if (diag_s) diag_s[i] = S.s[i];
                /* step 3: union with C_old row (beta != 0 only; beta == 0 -> C_old never read) */
                int32_t cold_n = (beta != 0.0) ? C->nnz[i] : 0;
                const int32_t* cc = C->col + (size_t)i * C->w;
                const double* cv = C->val + (size_t)i * C->w;
                for (int32_t q = 0; q < cold_n; ++q) touch(&S, cc[q]);
                qsort(S.touched, (size_t)S.nt, sizeof(int32_t), cmp_i32);
                /* step 4-5 (C_old row is sorted: walk it alongside the ascending union) */
                int32_t kept = 0, po = 0;
                for (int32_t t = 0; t < S.nt; ++t) {
                    int32_t j = S.touched[t];
                    double tt = 0.0;
                    while (po < cold_n && cc[po] < j) ++po;
                    if (po < cold_n && cc[po] == j) tt = beta * cv[po];
                    double c = fma(alpha, S.s[j], tt);
                    if (fabs(c) > tau) { S.ucols[kept] = j; S.uval[kept] = c; ++kept; }
                }
                scratch_reset(&S);
                if (kept > req) req = kept;
                if (kept > C->w) ++ovf;
                int32_t wr = kept < C->w ? kept : C->w;
                int32_t* oc = C->col + (size_t)i * C->w;
                double* ov = C->val + (size_t)i * C->w;
                for (int32_t q = 0; q < wr; ++q) { oc[q] = S.ucols[q]; ov[q] = S.uval[q]; }
                C->nnz[i] = wr;
            }
            scratch_free(&S);
        }
    }
    if (err) return O_NOMEM;
    if (overflow_rows) *overflow_rows = ovf;
    if (required_width) *required_width = req;
    return ovf ? O_OVERFLOW : O_OK;
}

int oracle_multiply(const omat* A, const omat* B, omat* C, double alpha, double beta, double tau,
                    int64_t* overflow_rows, int32_t* required_width) {
    return oracle_multiply_ex(A, B, C, alpha, beta, tau, overflow_rows, required_width, NULL);
}

/* stored diagonal of M as a dense per-row vector (0 if absent) */
static void stored_diag(const omat* M, double* d) {
    for (int64_t i = 0; i < M->n; ++i) {
        int found;
        d[i] = lookup(M, i, (int32_t)i, &found);
    }
}

/* §8c-c5: X2 <- drop_tau(X*X) (c2 with A = B = X, alpha = 1, beta = 0);
 * tr(X) = canonical sum of stored x_ii; tr(X^2) = canonical sum of pre-drop s_ii. */
int oracle_x2(const omat* X, omat* X2, double tau, double* trace_x, double* trace_x2,
              int64_t* overflow_rows, int32_t* required_width) {
    if (!X || !X2) return O_ARG;
    if (X->n != X2->n) return O_DIM;
    int64_t n = X->n;
    double* d = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* ds = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!d || !ds) { free(d); free(ds); return O_NOMEM; }
    stored_diag(X, d);
    double tx = oracle_canonical_sum(d, n);
    int rc = oracle_multiply_ex(X, X, X2, 1.0, 0.0, tau, overflow_rows, required_width, ds);
    double tx2 = oracle_canonical_sum(ds, n);
    free(d); free(ds);
    if (rc == O_OK) {
        if (trace_x) *trace_x = tx;
        if (trace_x2) *trace_x2 = tx2;
    }
    return rc;
}

/*
 * §8c-c6 add: A <- drop_tau(alpha*A + beta*B). U = cols(A_i) u cols(B_i) ascending;
 * v = fma(alpha, a_j (or 0), beta * b_j (or 0)); keep |v| > tau. B may be A itself.
 */
int oracle_add(omat* A, const omat* B, double alpha, double beta, double tau,
               int64_t* overflow_rows, int32_t* required_width) {
    if (!A || !B) return O_ARG;
    if (A->n != B->n) return O_DIM;
    if (!(tau >= 0.0) || !isfinite(tau)) return O_ARG;
    int64_t n = A->n, ovf = 0;
    int32_t req = 0;
    int32_t* uc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(A->w + B->w + 1));
    double* uv = (double*)malloc(sizeof(double) * (size_t)(A->w + B->w + 1));
    if (!uc || !uv) { free(uc); free(uv); return O_NOMEM; }
    for (int64_t i = 0; i < n; ++i) {
        const int32_t* ca = A->col + (size_t)i * A->w;
        const double* va = A->val + (size_t)i * A->w;
        const int32_t* cb = B->col + (size_t)i * B->w;
        const double* vb = B->val + (size_t)i * B->w;
        int32_t na = A->nnz[i], nb = B->nnz[i], p = 0, q = 0, kept = 0;
        while (p < na || q < nb) {
            int32_t j;
            double a = 0.0, b = 0.0;
            if (q >= nb || (p < na && ca[p] < cb[q])) { j = ca[p]; a = va[p]; ++p; }
            else if (p >= na || cb[q] < ca[p]) { j = cb[q]; b = vb[q]; ++q; }
            else { j = ca[p]; a = va[p]; b = vb[q]; ++p; ++q; }
            double v = fma(alpha, a, beta * b);
            if (fabs(v) > tau) { uc[kept] = j; uv[kept] = v; ++kept; }
        }
        if (kept > req) req = kept;
        if (kept > A->w) ++ovf;
        int32_t wr = kept < A->w ? kept : A->w;
        int32_t* oc = A->col + (size_t)i * A->w;
        double* ov = A->val + (size_t)i * A->w;
        for (int32_t t = 0; t < wr; ++t) { oc[t] = uc[t]; ov[t] = uv[t]; }
        A->nnz[i] = wr;
    }
    free(uc); free(uv);
    if (overflow_rows) *overflow_rows = ovf;
    if (required_width) *required_width = req;
    return ovf ? O_OVERFLOW : O_OK;
}

/*
 * §8c-c6 scale_add_identity: A <- drop_tau(alpha*A + beta*I): off-diagonal alpha*a_ij,
 * diagonal fma(alpha, a_ii (or 0), beta); inserts the diagonal if absent.
 * add_identity(A, beta) is scale_add_identity with alpha = 1 (fma(1,a,beta) = a+beta).
 */
int oracle_scale_add_identity(omat* A, double alpha, double beta, double tau,
                              int64_t* overflow_rows, int32_t* required_width) {
    if (!A) return O_ARG;
    if (!(tau >= 0.0) || !isfinite(tau)) return O_ARG;
    int64_t n = A->n, ovf = 0;
    int32_t req = 0;
    int32_t* uc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(A->w + 1));
    double* uv = (double*)malloc(sizeof(double) * (size_t)(A->w + 1));
    if (!uc || !uv) { free(uc); free(uv); return O_NOMEM; }
    for (int64_t i = 0; i < n; ++i) {
        const int32_t* ca = A->col + (size_t)i * A->w;
        const double* va = A->val + (size_t)i * A->w;
        int32_t na = A->nnz[i], kept = 0, diag_done = 0;
        for (int32_t p = 0; p <= na; ++p) {
            if (!diag_done && (p == na || ca[p] >= (int32_t)i)) {
                double a = (p < na && ca[p] == (int32_t)i) ? va[p] : 0.0;
                double v = fma(alpha, a, beta);
                if (fabs(v) > tau) { uc[kept] = (int32_t)i; uv[kept] = v; ++kept; }
                diag_done = 1;
                if (p < na && ca[p] == (int32_t)i) continue;
            }
            if (p == na) break;
            double v = alpha * va[p];
            if (fabs(v) > tau) { uc[kept] = ca[p]; uv[kept] = v; ++kept; }
        }
        if (kept > req) req = kept;
        if (kept > A->w) ++ovf;
        int32_t wr = kept < A->w ? kept : A->w;
        int32_t* oc = A->col + (size_t)i * A->w;
        double* ov = A->val + (size_t)i * A->w;
        for (int32_t t = 0; t < wr; ++t) { oc[t] = uc[t]; ov[t] = uv[t]; }
        A->nnz[i] = wr;
    }
    free(uc); free(uv);
    if (overflow_rows) *overflow_rows = ovf;
    if (required_width) *required_width = req;
    return ovf ? O_OVERFLOW : O_OK;
}

int oracle_add_identity(omat* A, double beta, double tau, int64_t* overflow_rows, int32_t* required_width) {
    return oracle_scale_add_identity(A, 1.0, beta, tau, overflow_rows, required_width);
}

/* §8c-c7 trace: canonical sum of the stored diagonal */
int oracle_trace(const omat* A, double* out) {
    if (!A || !out) return O_ARG;
    double* d = (double*)malloc(sizeof(double) * (size_t)(A->n > 0 ? A->n : 1));
    if (!d) return O_NOMEM;
    stored_diag(A, d);
    *out = oracle_canonical_sum(d, A->n);
    free(d);
    return O_OK;
}

/* §8c-c11 fnorm_diff: ||A - B||_F over the union pattern. Order:
 * row by row, merged ascending columns; rows summed with the canonical sum. */
int oracle_fnorm_diff(const omat* A, const omat* B, double* out) {
    if (!A || !B || !out) return O_ARG;
    if (A->n != B->n) return O_DIM;
    int64_t n = A->n;
    double* r = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!r) return O_NOMEM;
    for (int64_t i = 0; i < n; ++i) {
        const int32_t* ca = A->col + (size_t)i * A->w;
        const double* va = A->val + (size_t)i * A->w;
        const int32_t* cb = B->col + (size_t)i * B->w;
        const double* vb = B->val + (size_t)i * B->w;
        int32_t na = A->nnz[i], nb = B->nnz[i], p = 0, q = 0;
        double s = 0.0;
        while (p < na || q < nb) {
            double a = 0.0, b = 0.0;
            if (q >= nb || (p < na && ca[p] < cb[q])) { a = va[p]; ++p; }
            else if (p >= na || cb[q] < ca[p]) { b = vb[q]; ++q; }
            else { a = va[p]; b = vb[q]; ++p; ++q; }
            double d = a - b;
            s = s + d * d;
        }
        r[i] = s;
    }
    *out = sqrt(oracle_canonical_sum(r, n));
    free(r);
    return O_OK;
}

/* §8c-c8 Gershgorin: r_i = ((0 + |v_1|) + |v_2|) + ... over off-diagonal slots in
 * slot order; lo_i = h_ii - r_i, hi_i = h_ii + r_i; eps_min = min lo_i, eps_max = max hi_i.
 * (S:L358-363). An empty row contributes (0, 0). */
int oracle_gershgorin(const omat* H, double* emin, double* emax) {
    if (!H || !emin || !emax || H->n <= 0) return O_ARG;
    double lo_min = INFINITY, hi_max = -INFINITY;
    for (int64_t i = 0; i < H->n; ++i) {
        const int32_t* c = H->col + (size_t)i * H->w;
        const double* v = H->val + (size_t)i * H->w;
        double r = 0.0, d = 0.0;
        for (int32_t q = 0; q < H->nnz[i]; ++q) {
            if (c[q] == (int32_t)i) d = v[q];
            else r = r + fabs(v[q]);
        }
        double lo = d - r, hi = d + r;
        if (lo < lo_min) lo_min = lo;
        if (hi > hi_max) hi_max = hi;
    }
    *emin = lo_min;
    *emax = hi_max;
    return O_OK;
}

/* ------------------------------------------------------------------ SP2 */

typedef struct {
    double threshold;   /* tau (0) */
    int32_t max_iter;   /* 100 */
    int32_t min_iter;   /* 20 */
    double stag_gate;   /* 1e-3 */
    double emin, emax;  /* NaN -> Gershgorin */
    int32_t on_overflow;/* 0 FAIL, 1 GROW */
    int32_t max_width;  /* <= 0 -> n */
    int32_t initial_width; /* <= 0 -> H.w */
    int32_t branch_rule;   /* 0 trace sign (default), 1 trace-closest (§8f-f4 i) */
} osp2_opts;

typedef struct {
    double trX, trS, e, fnorm;
    int32_t branch;   /* 0 SQUARE, 1 EXPAND */
    int32_t width;    /* width of X_{n+1} storage after this step */
    int32_t required; /* max kept count of X_{n+1} */
    int32_t pad;
    int64_t products;
    double frob2;     /* branch_rule 1: T2_n (see sp2_frob2), else 0 */
} osp2_iter;

typedef struct {
    int32_t iterations, stop_reason; /* 0 CONVERGED, 1 STAGNATED, 2 NOCONV, 3 OVERFLOW */
    int32_t final_width, regrows;
    double emin, emax, trD;
    int64_t overflow_rows;           /* on OVERFLOW stop */
    int32_t required_width, fail_iter;
} osp2_report;

static int32_t round_up32(int32_t x) { return (x + 31) & ~31; }

/*
 * One SP2 step (§8c-c10 (ii)-(iii)) on rows of X (all rows):
 *   S = X*X pre-drop (c2 accumulate), trS partials = s_ii,
 *   X1 = drop_tau(S) if SQUARE else drop_tau(fma(2, x_ij (or 0), -s_ij)) over the union,
 *   ||S - X||_F^2 over the union, per-row.
 * Rows are written into Y (width Y->w); kept counts returned via req/ovf.
 */
static int sp2_step(const omat* X, omat* Y, int branch, double tau, double* ds, double* dy,
                    double* nrm, int64_t* ovf_out, int32_t* req_out, int64_t* prod_out) {
    int64_t n = X->n, ovf = 0, prod = 0;
    int32_t req = 0;
    int err = 0;
#pragma omp parallel reduction(+ : ovf, prod) reduction(max : req) reduction(| : err)
    {
        scratch S;
        if (scratch_init(&S, n)) err |= 1;
        else {
#pragma omp for schedule(dynamic, 64)
            for (int64_t i = 0; i < n; ++i) {
                accumulate_row(&S, X, X, i);
                for (int32_t p = 0; p < X->nnz[i]; ++p) prod += X->nnz[X->col[(size_t)i * X->w + p]];
                ds[i] = S.s[i];
                const int32_t* cx = X->col + (size_t)i * X->w;
                const double* vx = X->val + (size_t)i * X->w;
                for (int32_t q = 0; q < X->nnz[i]; ++q) touch(&S, cx[q]);
                qsort(S.touched, (size_t)S.nt, sizeof(int32_t), cmp_i32);
                int32_t kept = 0, px = 0, nx = X->nnz[i];
                double nr = 0.0, diag = 0.0;
                for (int32_t t = 0; t < S.nt; ++t) {
                    int32_t j = S.touched[t];
                    double x = 0.0;
                    while (px < nx && cx[px] < j) ++px;
                    if (px < nx && cx[px] == j) x = vx[px];
                    double s = S.s[j];
                    double dd = s - x;
                    nr = nr + dd * dd;
                    double c = (branch == 0) ? s : fma(2.0, x, -s);
                    if (fabs(c) > tau) {
                        S.ucols[kept] = j; S.uval[kept] = c; ++kept;
                        if (j == (int32_t)i) diag = c;
                    }
                }
                scratch_reset(&S);
                nrm[i] = nr;
                dy[i] = diag;
                if (kept > req) req = kept;
                if (kept > Y->w) ++ovf;
                int32_t wr = kept < Y->w ? kept : Y->w;
                int32_t* oc = Y->col + (size_t)i * Y->w;
                double* ov = Y->val + (size_t)i * Y->w;
                for (int32_t q = 0; q < wr; ++q) { oc[q] = S.ucols[q]; ov[q] = S.uval[q]; }
                Y->nnz[i] = wr;
            }
            scratch_free(&S);
        }
    }
    if (err) return O_NOMEM;
    *ovf_out = ovf;
    *req_out = req;
    *prod_out = prod;
    return O_OK;
}

/*
 * Trace-closest branch rule (§8f-f4 (i), Niklasson 2002 SP2; reading R19):
 * SQUARE iff tr(X_n^2) is closer to nocc than tr(2X_n - X_n^2) = 2 tr(X_n) - tr(X_n^2).
 * tr(X^2) must be known BEFORE the fused step, so it is taken from X_n itself:
 * for symmetric X (every SP2 iterate of a symmetric H, P4) tr(X^2) = sum_ij x_ij x_ji
 * = sum_ij x_ij^2. T2 = canonical sum (c7) of q_i, q_i = fma chain over the stored
 * slots of row i in ascending order, q <- fma(x, x, q) from +0.
 * Decision: |T2 - nocc| < |(2 trX - T2) - nocc| -> SQUARE, else EXPAND (tie -> EXPAND).
 */
static double sp2_frob2(const omat* X, double* q) {
    for (int64_t i = 0; i < X->n; ++i) {
        const double* v = X->val + (size_t)i * X->w;
        double s = 0.0;
        for (int32_t p = 0; p < X->nnz[i]; ++p) s = fma(v[p], v[p], s);
        q[i] = s;
    }
    return oracle_canonical_sum(q, X->n);
}

static int mat_alloc(omat* M, int64_t n, int32_t w) {
    M->n = n; M->w = w;
    M->val = (double*)calloc((size_t)n * (size_t)w, sizeof(double));
    M->col = (int32_t*)calloc((size_t)n * (size_t)w, sizeof(int32_t));
    M->nnz = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    return (M->val && M->col && M->nnz) ? 0 : -1;
}
static void mat_free(omat* M) { free(M->val); free(M->col); free(M->nnz); M->val = 0; M->col = 0; M->nnz = 0; }

/*
 * SP2-Basic (§8c-c9, c10):
 *  init : (emin, emax) <- Gershgorin (or opts); D = emax - emin; D <= 0 or non-finite -> BOUNDS;
 *         alpha = -1/D, beta = emax/D; X0 = scale_add_identity(H, alpha, beta, tau); trX0 canonical.
 *  loop n = 0, 1, ...:
 *    (i)   b_n = SQUARE if trX_n > nocc else EXPAND (tie -> EXPAND); with branch_rule 1 the
 *          trace-closest rule of sp2_frob2 instead
 *    (ii)  S_n = X_n X_n (pre-drop); trS_n canonical
 *    (iii) X_{n+1} = drop(S_n) | drop(fma(2, x, -s)) over the union
 *    (iv)  overflow -> FAIL: return OVERFLOW(n) | GROW: width <- round_up32(required) (<= max_width)
 *    (v)   e_n = trX_n - trS_n; trX_{n+1} canonical over X_{n+1}'s stored diagonal
 *    (vi)  CONVERGED if |e_n| <= tol; STAGNATED if n+1 >= min_iter and e_n <= stag_gate and
 *          e_n >= e_{n-2}; NOCONV if n+1 == max_iter. D = X_{n+1}, iterations = n+1.
 * iters (nullable, >= max_iter entries) receives the per-iteration record.
 * D receives the result at width D->w (OVERFLOW if too narrow).
 */
int oracle_sp2(const omat* H, int64_t nocc, double tol, const osp2_opts* o, omat* D,
               osp2_report* rep, osp2_iter* iters) {
    if (!H || !D || !o) return O_ARG;
    int64_t n = H->n;
    if (nocc < 0 || nocc > n || !(tol >= 0.0) || D->n != n) return O_ARG;
    double tau = o->threshold;
    double emin = o->emin, emax = o->emax;
    if (isnan(emin) || isnan(emax)) oracle_gershgorin(H, &emin, &emax);
    double Dl = emax - emin;
    osp2_report R;
    memset(&R, 0, sizeof R);
    R.emin = emin; R.emax = emax;
    if (!(Dl > 0.0) || !isfinite(Dl)) { if (rep) *rep = R; return O_BOUNDS; }
    double alpha = -1.0 / Dl, beta = emax / Dl;
    /* widths are even (reading R20: the ABI's ELLPACK widths are even, 16-byte slot pairs) */
    int32_t maxw = ((o->max_width > 0 ? o->max_width : (int32_t)n) + 1) & ~1;
    int32_t w = ((o->initial_width > 0 ? o->initial_width : H->w) + 1) & ~1;
    /* X0 = drop(alpha*H + beta*I) computed at width H.w + 1 (always enough: a row of H
     * plus its diagonal); its max kept count decides FAIL / GROW against the width w. */
    omat T, X, Y;
    if (mat_alloc(&T, n, H->w + 1)) return O_NOMEM;
    for (int64_t i = 0; i < n; ++i) {
        int32_t k = H->nnz[i];
        memcpy(T.col + (size_t)i * T.w, H->col + (size_t)i * H->w, sizeof(int32_t) * (size_t)k);
        memcpy(T.val + (size_t)i * T.w, H->val + (size_t)i * H->w, sizeof(double) * (size_t)k);
        T.nnz[i] = k;
    }
    int64_t ovf = 0;
    int32_t req = 0;
    oracle_scale_add_identity(&T, alpha, beta, tau, &ovf, &req);
    if (req > w) {
        if (o->on_overflow == 0 || req > maxw) {
            /* c4: overflow_rows = #{i : kept_i > W} with W the width X0 was asked to fit */
            int64_t over = 0;
            for (int64_t i = 0; i < n; ++i) over += T.nnz[i] > w;
            R.stop_reason = 3; R.overflow_rows = over; R.required_width = req; R.fail_iter = -1;
            mat_free(&T); if (rep) *rep = R; return O_OVERFLOW;
        }
        w = round_up32(req) < maxw ? round_up32(req) : maxw;
        R.regrows++;
    }
    if (mat_alloc(&X, n, w)) { mat_free(&T); return O_NOMEM; }
    for (int64_t i = 0; i < n; ++i) {
        int32_t k = T.nnz[i];
        memcpy(X.col + (size_t)i * w, T.col + (size_t)i * T.w, sizeof(int32_t) * (size_t)k);
        memcpy(X.val + (size_t)i * w, T.val + (size_t)i * T.w, sizeof(double) * (size_t)k);
        X.nnz[i] = k;
    }
    mat_free(&T);
    double trX;
    oracle_trace(&X, &trX);
    double* ds = (double*)malloc(sizeof(double) * (size_t)n);
    double* dy = (double*)malloc(sizeof(double) * (size_t)n);
    double* nr = (double*)malloc(sizeof(double) * (size_t)n);
    double e_hist[2] = {NAN, NAN}; /* e_{n-2}, e_{n-1} */
    int32_t wy = w;
    int stop = -1, status = O_OK;
    int32_t it;
    for (it = 0; it < o->max_iter; ++it) {
        int branch = (trX > (double)nocc) ? 0 : 1;
        double t2 = 0.0;
        if (o->branch_rule == 1) {
            t2 = sp2_frob2(&X, nr);
            branch = (fabs(t2 - (double)nocc) < fabs((2.0 * trX - t2) - (double)nocc)) ? 0 : 1;
        }
        if (mat_alloc(&Y, n, wy)) { status = O_NOMEM; break; }
        int64_t prod = 0;
        sp2_step(&X, &Y, branch, tau, ds, dy, nr, &ovf, &req, &prod);
        if (ovf) {
            if (o->on_overflow == 0 || req > maxw) {
                R.stop_reason = 3; R.overflow_rows = ovf; R.required_width = req; R.fail_iter = it;
                mat_free(&Y); status = O_OVERFLOW; break;
            }
            /* GROW: recompute step n at the required width (deterministic; same values) */
            mat_free(&Y);
            wy = round_up32(req) < maxw ? round_up32(req) : maxw;
            if (mat_alloc(&Y, n, wy)) { status = O_NOMEM; break; }
            sp2_step(&X, &Y, branch, tau, ds, dy, nr, &ovf, &req, &prod);
            R.regrows++;
        }
        double trS = oracle_canonical_sum(ds, n);
        double trY = oracle_canonical_sum(dy, n);
        double fn = sqrt(oracle_canonical_sum(nr, n));
        double e = trX - trS;
        if (iters) {
            iters[it].trX = trX; iters[it].trS = trS; iters[it].e = e; iters[it].fnorm = fn;
            iters[it].branch = branch; iters[it].width = wy; iters[it].required = req;
            iters[it].products = prod;
            iters[it].frob2 = t2;
        }
        mat_free(&X);
        X = Y;
        trX = trY;
        if (fabs(e) <= tol) stop = 0;
        else if (it + 1 >= o->min_iter && e <= o->stag_gate && !isnan(e_hist[0]) && e >= e_hist[0]) stop = 1;
        else if (it + 1 == o->max_iter) stop = 2;
        e_hist[0] = e_hist[1];
        e_hist[1] = e;
        if (stop >= 0) { ++it; break; }
    }
    free(ds); free(dy); free(nr);
    R.iterations = it;
    R.final_width = X.w;
    R.trD = trX;
    if (status == O_OK) {
        R.stop_reason = stop;
        /* copy X into D */
        int32_t mx = 0;
        for (int64_t i = 0; i < n; ++i) if (X.nnz[i] > mx) mx = X.nnz[i];
        if (mx > D->w) {
            R.required_width = mx; status = O_OVERFLOW;
        } else {
            for (int64_t i = 0; i < n; ++i) {
                int32_t k = X.nnz[i];
                memcpy(D->col + (size_t)i * D->w, X.col + (size_t)i * X.w, sizeof(int32_t) * (size_t)k);
                memcpy(D->val + (size_t)i * D->w, X.val + (size_t)i * X.w, sizeof(double) * (size_t)k);
                for (int32_t q = k; q < D->w; ++q) { D->col[(size_t)i * D->w + q] = 0; D->val[(size_t)i * D->w + q] = 0.0; }
                D->nnz[i] = k;
            }
            if (stop == 2) status = O_NOCONV;
        }
    }
    mat_free(&X);
    if (rep) *rep = R;
    return status;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}
