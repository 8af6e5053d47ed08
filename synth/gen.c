/*
 * synth/gen.c — seeded synthetic ELLPACK inputs for BASELINE.json configs 1..5.
 *
 * This module is INPUT SYNTHESIS ONLY. It holds none of the method's
 * arithmetic (no products, sums, thresholds or traces): it draws random
 * patterns and values and writes them in canonical ELLPACK storage
 * (row-major val[N][W] f64, col[N][W] i32, nnz[N] i32; each row's columns
 * strictly ascending). Both the CPU oracle (oracle/) and the CUDA path
 * (paper_2102_08505_b200/) consume exactly these bytes, so parity never
 * depends on this file; reproducibility across runs does.
 *
 * RNG (SURVEY.md §8d / reading S14):
 *   splitmix64, one stream per config, seeded with the config's seed;
 *   uniform  u = (x >> 11) * 2^-53 in [0,1);   U(a,b) = a + (b-a)*u
 *   normal   z = sqrt(-2 ln(1-u1)) * cos(2*pi*u2)  (two uniforms per normal)
 *   sign     s = (x >> 63) ? -1 : +1
 *   "k distinct partners in band b" = repeated uniform draws from
 *   [max(0,i-b), min(N-1,i+b)] \ {i}, rejecting repeats, kept in draw order.
 *
 * Build: gcc -O2 -fPIC -shared (see __graft_entry__.build()).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef struct { uint64_t s; } rng_t;

static uint64_t sm64(rng_t* r) {
    uint64_t z = (r->s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static double unif(rng_t* r) { return (double)(sm64(r) >> 11) * 0x1.0p-53; }
static double unif_ab(rng_t* r, double a, double b) { return a + (b - a) * unif(r); }
static double normal(rng_t* r) {
    double u1 = unif(r), u2 = unif(r);
    return sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586476925286766559 * u2);
}
static double rsign(rng_t* r) { return (sm64(r) >> 63) ? -1.0 : 1.0; }

/* uniform draw of a partner j in band b of row i, j != i; requires cnt >= 1 */
static int64_t draw_partner(rng_t* r, int64_t n, int64_t i, int64_t b) {
    int64_t lo = i - b < 0 ? 0 : i - b;
    int64_t hi = i + b > n - 1 ? n - 1 : i + b;
    int64_t cnt = hi - lo; /* (hi-lo+1) candidates minus i itself */
    int64_t idx = (int64_t)(unif(r) * (double)cnt);
    if (idx >= cnt) idx = cnt - 1;
    int64_t j = lo + idx;
    if (j >= i) j += 1;
    return j;
}

static int row_has(const int32_t* col, int32_t cnt, int32_t j) {
    for (int32_t q = 0; q < cnt; ++q) if (col[q] == j) return 1;
    return 0;
}

/* sort each row's (col,val) ascending by col: insertion sort for short rows,
 * heap-free merge via qsort on an index for long rows. */
typedef struct { int32_t c; double v; } cv_t;
static int cmp_cv(const void* a, const void* b) {
    int32_t x = ((const cv_t*)a)->c, y = ((const cv_t*)b)->c;
    return (x > y) - (x < y);
}
static void sort_rows(int64_t n, int32_t w, double* val, int32_t* col, const int32_t* nnz) {
    cv_t* tmp = (cv_t*)malloc(sizeof(cv_t) * (size_t)(w > 0 ? w : 1));
    for (int64_t i = 0; i < n; ++i) {
        double* v = val + (size_t)i * w;
        int32_t* c = col + (size_t)i * w;
        int32_t k = nnz[i];
        for (int32_t q = 0; q < k; ++q) { tmp[q].c = c[q]; tmp[q].v = v[q]; }
        qsort(tmp, (size_t)k, sizeof(cv_t), cmp_cv);
        for (int32_t q = 0; q < k; ++q) { c[q] = tmp[q].c; v[q] = tmp[q].v; }
        for (int32_t q = k; q < w; ++q) { c[q] = 0; v[q] = 0.0; }
    }
    free(tmp);
}

/*
 * Symmetric banded matrix with the "cap at W" rule:
 *  (1) diagonal for i = 0..n-1 in order: diag_kind 1 -> U(dlo,dhi); 2 -> N(0,1)
 *  (2) for i = 0..n-1: draw `partners` distinct partners j in band `band`;
 *      for each in draw order: skip if (i,j) already stored, skip if row i or
 *      row j already holds w entries; else draw the value and store it at
 *      (i,j) and (j,i).
 *      off_kind 0: v = z * exp(-|i-j|/decay), z ~ N(0,1)
 *      off_kind 1: v = amp * exp(-|i-j|/decay) * s,  s = random sign
 *  Rows are then sorted ascending by column.
 */
int synth_sym_banded(int64_t n, int32_t w, int32_t partners, int64_t band,
                     int diag_kind, double dlo, double dhi,
                     int off_kind, double decay, double amp, uint64_t seed,
                     double* val, int32_t* col, int32_t* nnz) {
    if (n <= 0 || w <= 0 || partners < 0 || band < 1) return -1;
    rng_t r = {seed};
    memset(nnz, 0, sizeof(int32_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        double d = diag_kind == 1 ? unif_ab(&r, dlo, dhi) : normal(&r);
        size_t o = (size_t)i * w;
        col[o] = (int32_t)i; val[o] = d; nnz[i] = 1;
    }
    int64_t maxcand = 2 * band;
    int64_t* drawn = (int64_t*)malloc(sizeof(int64_t) * (size_t)(partners > 0 ? partners : 1));
    for (int64_t i = 0; i < n; ++i) {
        int64_t cand = (i + band > n - 1 ? n - 1 : i + band) - (i - band < 0 ? 0 : i - band);
        int32_t want = partners;
        if (want > cand) want = (int32_t)cand;
        (void)maxcand;
        int32_t nd = 0;
        while (nd < want) {
            int64_t j = draw_partner(&r, n, i, band);
            int dup = 0;
            for (int32_t t = 0; t < nd; ++t) if (drawn[t] == j) { dup = 1; break; }
            if (!dup) drawn[nd++] = j;
        }
        for (int32_t t = 0; t < nd; ++t) {
            int64_t j = drawn[t];
            int32_t* ci = col + (size_t)i * w;
            if (row_has(ci, nnz[i], (int32_t)j)) continue;
            if (nnz[i] >= w || nnz[j] >= w) continue;
            double dist = (double)(i > j ? i - j : j - i);
            double v;
            if (off_kind == 0) v = normal(&r) * exp(-dist / decay);
            else v = amp * exp(-dist / decay) * rsign(&r);
            size_t oi = (size_t)i * w + nnz[i], oj = (size_t)j * w + nnz[j];
            col[oi] = (int32_t)j; val[oi] = v; nnz[i]++;
            col[oj] = (int32_t)i; val[oj] = v; nnz[j]++;
        }
    }
    free(drawn);
    sort_rows(n, w, val, col, nnz);
    return 0;
}

/*
 * Non-symmetric banded matrix: for each row i in order:
 * draw `partners` distinct off-diagonal partners in band, then the diagonal
 * value z ~ N(0,1) (e^0 = 1), then one z per partner in draw order:
 * v = z * exp(-|i-j|/decay). Exactly partners+1 entries per row (when the band
 * holds enough candidates). Requires w >= partners + 1.
 */
static int synth_nonsym_banded(int64_t n, int32_t w, int32_t partners, int64_t band,
                        double decay, rng_t* r,
                        double* val, int32_t* col, int32_t* nnz) {
    if (n <= 0 || w < partners + 1) return -1;
    int64_t* drawn = (int64_t*)malloc(sizeof(int64_t) * (size_t)(partners > 0 ? partners : 1));
    for (int64_t i = 0; i < n; ++i) {
        int64_t cand = (i + band > n - 1 ? n - 1 : i + band) - (i - band < 0 ? 0 : i - band);
        int32_t want = partners;
        if (want > cand) want = (int32_t)cand;
        int32_t nd = 0;
        while (nd < want) {
            int64_t j = draw_partner(r, n, i, band);
            int dup = 0;
            for (int32_t t = 0; t < nd; ++t) if (drawn[t] == j) { dup = 1; break; }
            if (!dup) drawn[nd++] = j;
        }
        size_t o = (size_t)i * w;
        col[o] = (int32_t)i; val[o] = normal(r);
        for (int32_t t = 0; t < nd; ++t) {
            double dist = (double)(i > drawn[t] ? i - drawn[t] : drawn[t] - i);
            col[o + 1 + t] = (int32_t)drawn[t];
            val[o + 1 + t] = normal(r) * exp(-dist / decay);
        }
        nnz[i] = nd + 1;
    }
    free(drawn);
    sort_rows(n, w, val, col, nnz);
    return 0;
}

/* cfg2: A, then B, then C_old from ONE stream seeded `seed`. Each of the three
 * output triples is n x w. */
int synth_cfg2(int64_t n, int32_t w, int32_t partners, int64_t band, double decay, uint64_t seed,
               double* va, int32_t* ca, int32_t* na,
               double* vb, int32_t* cb, int32_t* nb,
               double* vc, int32_t* cc, int32_t* nc) {
    rng_t r = {seed};
    int e = synth_nonsym_banded(n, w, partners, band, decay, &r, va, ca, na);
    if (e) return e;
    e = synth_nonsym_banded(n, w, partners, band, decay, &r, vb, cb, nb);
    if (e) return e;
    return synth_nonsym_banded(n, w, partners, band, decay, &r, vc, cc, nc);
}

/*
 * cfg4: 3D cubic lattice L^3 sites, 2 orbitals per site, open boundaries.
 * site s = x + L*y + L*L*z; row = 2*s + o.
 *  (1) on-site energies eps ~ U(-0.5, 0.5) for rows 0..N-1 in order;
 *  (2) for s ascending, for each neighbour offset in the fixed list below
 *      (6 nearest + 12 face-diagonal next-nearest) with t = s+offset inside the
 *      lattice and t > s, for o in {0,1}, for o' in {0,1}:
 *      h ~ U(-1, -0.5) stored at (2s+o, 2t+o') and mirrored.
 * No on-site inter-orbital term. Interior rows hold 1 + 18*2 = 37 entries.
 */
int synth_lattice(int32_t L, int32_t w, uint64_t seed, double* val, int32_t* col, int32_t* nnz) {
    static const int off[18][3] = {
        {1,0,0},{-1,0,0},{0,1,0},{0,-1,0},{0,0,1},{0,0,-1},
        {1,1,0},{1,-1,0},{-1,1,0},{-1,-1,0},
        {1,0,1},{1,0,-1},{-1,0,1},{-1,0,-1},
        {0,1,1},{0,1,-1},{0,-1,1},{0,-1,-1}};
    int64_t S = (int64_t)L * L * L, n = 2 * S;
    if (w < 37) return -1;
    rng_t r = {seed};
    for (int64_t i = 0; i < n; ++i) {
        size_t o = (size_t)i * w;
        col[o] = (int32_t)i; val[o] = unif_ab(&r, -0.5, 0.5); nnz[i] = 1;
    }
    for (int64_t s = 0; s < S; ++s) {
        int x = (int)(s % L), y = (int)((s / L) % L), z = (int)(s / ((int64_t)L * L));
        for (int b = 0; b < 18; ++b) {
            int x2 = x + off[b][0], y2 = y + off[b][1], z2 = z + off[b][2];
            if (x2 < 0 || y2 < 0 || z2 < 0 || x2 >= L || y2 >= L || z2 >= L) continue;
            int64_t t = x2 + (int64_t)L * y2 + (int64_t)L * L * z2;
            if (t <= s) continue;
            for (int o = 0; o < 2; ++o)
                for (int o2 = 0; o2 < 2; ++o2) {
                    double h = unif_ab(&r, -1.0, -0.5);
                    int64_t i = 2 * s + o, j = 2 * t + o2;
                    size_t oi = (size_t)i * w + nnz[i], oj = (size_t)j * w + nnz[j];
                    col[oi] = (int32_t)j; val[oi] = h; nnz[i]++;
                    col[oj] = (int32_t)i; val[oj] = h; nnz[j]++;
                }
        }
    }
    sort_rows(n, w, val, col, nnz);
    return 0;
}

/*
 * Generic seeded sparse test matrix (for parity edge cases): each row i gets
 * k_i ~ U{kmin..kmax} distinct columns drawn from [max(0,i-band), min(n-1,i+band)]
 * (diagonal allowed), values U(-1,1) (or N(0,1) scaled by `scale`);
 * a fraction `p_empty` of rows is left empty. Not symmetric.
 */
int synth_random(int64_t n, int32_t w, int32_t kmin, int32_t kmax, int64_t band,
                 double p_empty, double scale, uint64_t seed,
                 double* val, int32_t* col, int32_t* nnz) {
    if (n <= 0 || w <= 0 || kmin < 0 || kmax < kmin || kmax > w) return -1;
    rng_t r = {seed};
    for (int64_t i = 0; i < n; ++i) {
        size_t o = (size_t)i * w;
        int64_t lo = i - band < 0 ? 0 : i - band;
        int64_t hi = i + band > n - 1 ? n - 1 : i + band;
        int64_t cand = hi - lo + 1;
        int32_t k = kmin + (int32_t)(unif(&r) * (double)(kmax - kmin + 1));
        if (k > kmax) k = kmax;
        if (unif(&r) < p_empty) k = 0;
        if (k > cand) k = (int32_t)cand;
        int32_t c = 0;
        while (c < k) {
            int64_t j = lo + (int64_t)(unif(&r) * (double)cand);
            if (j > hi) j = hi;
            if (row_has(col + o, c, (int32_t)j)) continue;
            col[o + c] = (int32_t)j;
            val[o + c] = scale * unif_ab(&r, -1.0, 1.0);
            ++c;
        }
        nnz[i] = c;
    }
    sort_rows(n, w, val, col, nnz);
    return 0;
}

/* products count P = sum_i sum_{k in A_i} nnz_B(k) (pattern-only; used by the
 * harness to report GFLOP/s). */
int64_t synth_products(int64_t n, int32_t wa, const int32_t* ca, const int32_t* na,
                       const int32_t* nb) {
    int64_t p = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int32_t q = 0; q < na[i]; ++q) p += nb[ca[(size_t)i * wa + q]];
    return p;
}

/* ------------------------------------------------------------------ model Hamiltonian
 * The paper's two-level-system model Hamiltonian:
 * n/2 dimers, orbitals interleaved [A0, B0, A1, B1, ...] (orbital o = 2 d + t, t = 0 A, 1 B).
 *   diagonal            eps_t * (1 + r * RAND)
 *   same dimer, A-B     dAB_intra * (1 + r * RAND)                       (distance 0)
 *   dimers d1 != d2     delta(t1, t2) * exp(k * |d2 - d1|) * (1 + r * RAND)
 *                       delta = dAA (A-A), dBB (B-B), dAB_cross (A-B, B-A)
 * RAND in [-1, 1] is ONE draw per unordered pair (and per diagonal), from a counter-based
 * hash of (seed, min(o1, o2), max(o1, o2)), so the matrix is exactly symmetric and independent
 * of the enumeration order. An entry is stored iff |value| > tau_store; pairs whose largest
 * possible magnitude |delta| (1 + r) exp(k d) is <= tau_store are never enumerated (the SPEC's
 * cutoff, exact for the stored pattern). Input synthesis only. Returns the max row count when
 * val == NULL (sizing pass), else 0; -1 on bad arguments or a row wider than w. */
static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static double pair_rand(uint64_t seed, int64_t a, int64_t b) { /* uniform in [-1, 1) */
    uint64_t h = mix64(seed ^ mix64(((uint64_t)a << 32) ^ (uint64_t)b ^ 0x9E3779B97F4A7C15ULL));
    return 2.0 * ((double)(h >> 11) * 0x1.0p-53) - 1.0;
}

int64_t synth_model(int64_t n, int32_t w, double eps_a, double eps_b, double d_aa, double d_bb,
                    double d_ab_intra, double d_ab_cross, double k, double r, double tau_store, uint64_t seed,
                    double* val, int32_t* col, int32_t* nnz) {
    if (n < 2 || (n & 1) || k > 0.0 || r < 0.0 || tau_store < 0.0) return -1;
    const int64_t nd = n / 2;
    double dmaxc = fabs(d_aa);
    if (fabs(d_bb) > dmaxc) dmaxc = fabs(d_bb);
    if (fabs(d_ab_cross) > dmaxc) dmaxc = fabs(d_ab_cross);
    int64_t dcut = nd; /* largest dimer distance with |delta| (1 + r) e^{k d} > tau_store */
    if (k < 0.0 && dmaxc > 0.0 && tau_store > 0.0) {
        double dd = log(tau_store / (dmaxc * (1.0 + r))) / k;
        dcut = dd < 0.0 ? 0 : (int64_t)dd + 1;
        if (dcut > nd) dcut = nd;
    } else if (dmaxc == 0.0) {
        dcut = 0;
    }
    int64_t maxrow = 0;
    for (int64_t o = 0; o < n; ++o) {
        const int64_t d = o >> 1;
        const int t = (int)(o & 1);
        int32_t cnt = 0;
        const int64_t dlo = d - dcut < 0 ? 0 : d - dcut, dhi = d + dcut > nd - 1 ? nd - 1 : d + dcut;
        for (int64_t d2 = dlo; d2 <= dhi; ++d2) {
            for (int t2 = 0; t2 < 2; ++t2) {
                const int64_t o2 = 2 * d2 + t2;
                double base;
                if (o2 == o) base = t ? eps_b : eps_a;
                else if (d2 == d) base = d_ab_intra;
                else base = (t == 0 && t2 == 0) ? d_aa : (t == 1 && t2 == 1) ? d_bb : d_ab_cross;
                if (base == 0.0) continue;
                const int64_t lo = o < o2 ? o : o2, hi = o < o2 ? o2 : o;
                const int64_t dist = d2 > d ? d2 - d : d - d2;
                const double v = base * exp(k * (double)dist) * (1.0 + r * pair_rand(seed, lo, hi));
                if (!(fabs(v) > tau_store)) continue;
                if (val) {
                    if (cnt >= w) return -1;
                    val[(size_t)o * w + cnt] = v;
                    col[(size_t)o * w + cnt] = (int32_t)o2;
                }
                ++cnt;
            }
        }
        if (val) nnz[o] = cnt;
        if (cnt > maxrow) maxrow = cnt;
    }
    return val ? 0 : maxrow;
}
