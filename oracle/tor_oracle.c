/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference Torontonian engine
 * (torfp, /root/reference/proj) in plain C.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline/reference legs load it (as the checker); the product
 * library never links it.
 *
 * Parity PINNED: tests/test_oracle.py checks every raw fixed-point limb this file
 * produces against the golden values written by the unmodified reference
 * (tests/golden/reference_values.json via oracle/_ref) -- limb-exact.
 *
 * Restated algorithms (each function cites the reference lines it follows):
 *   fixed-point Wide<W>: fixed_point.hpp:49-185, fixed_point.cpp:52-162
 *   hermitian_det_fixed / hermitian_det_float: linalg.cpp:7-88
 *   extract_i_minus_az / i_minus_az_float / selected_modes: torontonian.cpp:14-65
 *   torontonian_partial / run_engine / torontonian_reference: torontonian.cpp:72-200
 *   binom / get_kth_mask / get_next_mask / partition: subsets.cpp:13-88
 *   select_precision / force_width and bound estimators: precision.cpp:16-148
 */
#define _POSIX_C_SOURCE 200809L
#include "tor_oracle.h"

#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef unsigned __int128 u128;
typedef uint64_t u64;

#define MAXW 4

/* ------------------------------------------------------------ errors ---- */
static void seterr(or_err* e, int status, const char* code, const char* msg, int64_t row, uint64_t mask) {
    if (!e) return;
    e->status = status;
    strncpy(e->code, code, sizeof(e->code) - 1);
    e->code[sizeof(e->code) - 1] = 0;
    strncpy(e->message, msg, sizeof(e->message) - 1);
    e->message[sizeof(e->message) - 1] = 0;
    e->row = row;
    e->mask = mask;
}

/* ------------------------------------------------- fixed point (W limbs) --- */
typedef struct {
    u64 w[MAXW];
} wide;

static int is_neg(const wide* a, int W) { return (int)(a->w[W - 1] >> 63); }
static int is_zero(const wide* a, int W) {
    u64 acc = 0;
    for (int i = 0; i < W; ++i) acc |= a->w[i];
    return acc == 0;
}
static wide w_add(wide a, wide b, int W) { /* fixed_point.hpp:49-63 */
    wide r = {{0}};
    u128 c = 0;
    for (int i = 0; i < W; ++i) {
        c += a.w[i];
        c += b.w[i];
        r.w[i] = (u64)c;
        c >>= 64;
    }
    return r;
}
static wide w_sub(wide a, wide b, int W) { /* fixed_point.hpp:65-79 */
    wide r = {{0}};
    u64 br = 0;
    for (int i = 0; i < W; ++i) {
        const u128 cur = (u128)a.w[i] - b.w[i] - br;
        r.w[i] = (u64)cur;
        br = (u64)((cur >> 64) & 1);
    }
    return r;
}
static wide w_neg(wide a, int W) {
    wide z = {{0}};
    return w_sub(z, a, W);
}
static wide w_one(unsigned f) { /* fixed_point.hpp:163-168 */
    wide r = {{0}};
    r.w[f >> 6] = (u64)1 << (f & 63);
    return r;
}

/* floor(a*b / 2^f) mod 2^(64W): unsigned product, two's-complement sign fix of the
 * high half, arithmetic shift (fixed_point.hpp:97-160). */
static wide w_mul(wide a, wide b, unsigned f, int W) {
    u64 p[2 * MAXW] = {0};
    for (int i = 0; i < W; ++i) {
        u64 carry = 0;
        for (int j = 0; j < W; ++j) {
            const u128 cur = (u128)a.w[i] * b.w[j] + p[i + j] + carry;
            p[i + j] = (u64)cur;
            carry = (u64)(cur >> 64);
        }
        p[i + W] = carry;
    }
    const u64 ma = 0 - (a.w[W - 1] >> 63), mb = 0 - (b.w[W - 1] >> 63);
    u64 br1 = 0, br2 = 0;
    for (int i = 0; i < W; ++i) {
        u128 cur = (u128)p[W + i] - (b.w[i] & ma) - br1;
        p[W + i] = (u64)cur;
        br1 = (u64)((cur >> 64) & 1);
        cur = (u128)p[W + i] - (a.w[i] & mb) - br2;
        p[W + i] = (u64)cur;
        br2 = (u64)((cur >> 64) & 1);
    }
    const unsigned ws = f >> 6, bs = f & 63;
    wide r = {{0}};
    for (int i = 0; i < W; ++i) {
        const u64 lo = p[i + ws], hi = p[i + ws + 1];
        r.w[i] = (lo >> bs) | ((hi << (63 - bs)) << 1);
    }
    return r;
}

/* L-limb helpers for division / square root */
static void shl1(u64* v, int L, u64 in) {
    u64 carry = in;
    for (int i = 0; i < L; ++i) {
        const u64 nx = v[i] >> 63;
        v[i] = (v[i] << 1) | carry;
        carry = nx;
    }
}
static int ucmp(const u64* a, int La, const u64* b, int Lb) {
    const int L = La > Lb ? La : Lb;
    for (int i = L - 1; i >= 0; --i) {
        const u64 x = i < La ? a[i] : 0, y = i < Lb ? b[i] : 0;
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}
static void usub(u64* a, int La, const u64* b, int Lb) {
    u64 br = 0;
    for (int i = 0; i < La; ++i) {
        const u128 cur = (u128)a[i] - (i < Lb ? b[i] : 0) - br;
        a[i] = (u64)cur;
        br = (u64)((cur >> 64) & 1);
    }
}

/* floor(2^num_pow / d), quotient bits >= limit -> overflow (fixed_point.cpp:52-72). */
static int div_pow2(const u64* d, int W, unsigned num_pow, unsigned limit, u64* q, int QW) {
    u64 rem[MAXW] = {0};
    memset(q, 0, sizeof(u64) * QW);
    for (int i = (int)num_pow; i >= 0; --i) {
        shl1(rem, W, i == (int)num_pow ? 1 : 0);
        if (ucmp(rem, W, d, W) >= 0) {
            usub(rem, W, d, W);
            if ((unsigned)i >= limit) return -1;
            q[i >> 6] |= (u64)1 << (i & 63);
        }
    }
    return 0;
}

/* integer square root of a 2W-limb value, digit by digit (fixed_point.cpp:74-96) */
static void isqrt(const u64* x, int W, u64* out) {
    u64 rem[2 * MAXW + 1] = {0}, root[MAXW + 1] = {0}, trial[MAXW + 1];
    for (int k = 64 * W - 1; k >= 0; --k) {
        const unsigned b1 = 2 * k + 1, b0 = 2 * k;
        shl1(rem, 2 * W + 1, (x[b1 >> 6] >> (b1 & 63)) & 1);
        shl1(rem, 2 * W + 1, (x[b0 >> 6] >> (b0 & 63)) & 1);
        memcpy(trial, root, sizeof(trial));
        shl1(trial, W + 1, 0);
        shl1(trial, W + 1, 1);
        shl1(root, W + 1, 0);
        if (ucmp(rem, 2 * W + 1, trial, W + 1) >= 0) {
            usub(rem, 2 * W + 1, trial, W + 1);
            root[0] |= 1;
        }
    }
    for (int i = 0; i < W; ++i) out[i] = root[i];
}

static int w_recip(wide a, unsigned f, int W, wide* r) { /* fixed_point.cpp:100-108 */
    if (is_neg(&a, W) || is_zero(&a, W)) return -2;
    wide q = {{0}};
    if (div_pow2(a.w, W, 2 * f, 64u * W - 1, q.w, W)) return -1;
    *r = q;
    return 0;
}
static int w_rsqrt(wide a, unsigned f, int W, wide* r) { /* fixed_point.cpp:110-121 */
    if (is_neg(&a, W) || is_zero(&a, W)) return -2;
    u64 x[2 * MAXW] = {0};
    if (div_pow2(a.w, W, 3 * f, 2u * 64u * W - 2, x, 2 * W)) return -1;
    wide out = {{0}};
    isqrt(x, W, out.w);
    *r = out;
    return 0;
}
static wide w_from_real(double x, unsigned f, int W) { /* fixed_point.cpp:123-150 */
    wide r = {{0}};
    if (x == 0.0) return r;
    int e = 0;
    const double fr = frexp(fabs(x), &e);
    const u64 m = (u64)ldexp(fr, 53);
    const int s = e - 53 + (int)f;
    if (s >= 0) {
        const unsigned limb = (unsigned)s >> 6, bits = (unsigned)s & 63;
        r.w[limb] = m << bits;
        if (bits != 0 && limb + 1 < (unsigned)W) r.w[limb + 1] = m >> (64 - bits);
    } else {
        const unsigned sh = (unsigned)(-s);
        if (sh <= 53) r.w[0] = (m >> sh) + ((m >> (sh - 1)) & 1);
    }
    return x < 0 ? w_neg(r, W) : r;
}
static double w_to_real(wide a, unsigned f, int W) { /* fixed_point.cpp:152-162 */
    const int neg = is_neg(&a, W);
    const wide mag = neg ? w_neg(a, W) : a;
    long double acc = 0.0L;
    for (int i = W - 1; i >= 0; --i) acc = ldexpl(acc, 64) + (long double)mag.w[i];
    const double out = (double)ldexpl(acc, -(int)f);
    return neg ? -out : out;
}

/* ------------------------------------------------------------- input ---- */
typedef struct {
    int n;
    const double* a00; /* interleaved triangle */
    const double* a01;
} inp;

static size_t tri(int n, int i, int j) { return (size_t)i * n - (size_t)i * (i + 1) / 2 + (size_t)j; }
static double complex a00_at(const inp* a, int i, int j) { /* matrix_io.cpp:80-83 */
    if (i <= j) {
        const size_t k = tri(a->n, i, j);
        return a->a00[2 * k] + I * a->a00[2 * k + 1];
    }
    const size_t k = tri(a->n, j, i);
    return a->a00[2 * k] - I * a->a00[2 * k + 1];
}
static double complex a01_at(const inp* a, int i, int j) { /* matrix_io.cpp:85-88 */
    const size_t k = i <= j ? tri(a->n, i, j) : tri(a->n, j, i);
    return a->a01[2 * k] + I * a->a01[2 * k + 1];
}

/* ----------------------------------------------------------- subsets ---- */
static u64 PASCAL[63][63];
static pthread_once_t pascal_once = PTHREAD_ONCE_INIT;
static void pascal_init(void) { /* subsets.cpp:13-24 */
    for (int n = 0; n <= 62; ++n) {
        PASCAL[n][0] = 1;
        for (int k = 1; k <= n; ++k) PASCAL[n][k] = PASCAL[n - 1][k - 1] + (k <= n - 1 ? PASCAL[n - 1][k] : 0);
    }
}
uint64_t or_binom(int n, int k) {
    pthread_once(&pascal_once, pascal_init);
    if (n < 0 || k < 0 || k > n || n > 62) return 0;
    return PASCAL[n][k];
}
uint64_t or_get_kth_mask(int N, int z, uint64_t k) { /* subsets.cpp:36-54 */
    u64 m = 0;
    int rem = z;
    for (int p = N - 1; p >= 0 && rem > 0; --p) {
        const u64 cnt = or_binom(p, rem - 1);
        if (k < cnt) {
            m |= (u64)1 << p;
            --rem;
        } else {
            k -= cnt;
        }
    }
    return m;
}
uint64_t or_get_next_mask(uint64_t mask) { /* subsets.cpp:56-64 */
    int t = 0;
    while ((mask >> t) & 1) ++t;
    const u64 x = mask - (((u64)1 << t) - 1);
    if (x == 0) return 0;
    const int p = __builtin_ctzll(x);
    return x - ((u64)1 << (p - t - 1));
}

/* -------------------------------------------------------- elimination ---- */
typedef struct {
    wide re, im;
} cw;

/* I - A_Z in (modes, modes+N) block order at scaling f (torontonian.cpp:44-65) */
static void extract(const inp* a, u64 mask, unsigned f, int W, cw* out, int* dim) {
    int sel[64], z = 0;
    for (int j = 0; j < a->n; ++j)
        if ((mask >> (a->n - 1 - j)) & 1) sel[z++] = j;
    const int d = 2 * z;
    *dim = d;
    for (int p = 0; p < d; ++p)
        for (int q = p; q < d; ++q) {
            double complex v;
            if (q < z) v = a00_at(a, sel[p], sel[q]);
            else if (p < z) v = a01_at(a, sel[p], sel[q - z]);
            else v = conj(a00_at(a, sel[p - z], sel[q - z]));
            cw* e = &out[tri(d, p, q)];
            if (p == q) {
                e->re = w_from_real(1.0 - creal(v), f, W);
                memset(&e->im, 0, sizeof(wide));
            } else {
                e->re = w_from_real(-creal(v), f, W);
                e->im = w_from_real(-cimag(v), f, W);
            }
        }
}

/* hermitian_det_fixed (linalg.cpp:7-61); returns 0, or -1 with *bad_row on breakdown */
static int herm_det_fixed(cw* m, int n, unsigned f, int W, wide* det_out, int* bad_row) {
    wide det = w_one(f), zero = {{0}};
    for (int k = 0; k < n; ++k) {
        const wide pivot = m[tri(n, k, k)].re;
        if (is_neg(&pivot, W) || is_zero(&pivot, W)) {
            *bad_row = k;
            return -1;
        }
        det = w_mul(det, pivot, f, W);
        if (k == n - 1) break;
        wide pinv;
        if (w_recip(pivot, f, W, &pinv)) {
            *bad_row = k;
            return -1;
        }
        for (int i = k + 1; i < n; ++i) {
            const cw aki = m[tri(n, k, i)];
            const wide nim = w_neg(aki.im, W);
            cw s;
            s.re = w_sub(w_mul(aki.re, pinv, f, W), w_mul(nim, zero, f, W), W);
            s.im = w_add(w_mul(aki.re, zero, f, W), w_mul(nim, pinv, f, W), W);
            wide* dii = &m[tri(n, i, i)].re;
            const wide pr = w_sub(w_mul(s.re, aki.re, f, W), w_mul(s.im, aki.im, f, W), W);
            *dii = w_sub(*dii, pr, W);
            for (int j = i + 1; j < n; ++j) {
                const cw akj = m[tri(n, k, j)];
                cw* aij = &m[tri(n, i, j)];
                const wide p_re = w_sub(w_mul(s.re, akj.re, f, W), w_mul(s.im, akj.im, f, W), W);
                const wide p_im = w_add(w_mul(s.re, akj.im, f, W), w_mul(s.im, akj.re, f, W), W);
                aij->re = w_sub(aij->re, p_re, W);
                aij->im = w_sub(aij->im, p_im, W);
            }
        }
    }
    *det_out = det;
    return 0;
}

/* hermitian_det_float (linalg.cpp:66-88) */
static double herm_det_float(double complex* m, int n, int* nonfinite) {
    double det = 1.0;
    for (int k = 0; k < n; ++k) {
        const double pivot = creal(m[tri(n, k, k)]);
        det *= pivot;
        if (k == n - 1) break;
        const double pinv = 1.0 / pivot;
        for (int i = k + 1; i < n; ++i) {
            const double complex s = conj(m[tri(n, k, i)]) * pinv;
            m[tri(n, i, i)] -= creal(s * m[tri(n, k, i)]);
            for (int j = i + 1; j < n; ++j) m[tri(n, i, j)] -= s * m[tri(n, k, j)];
        }
    }
    *nonfinite = !isfinite(det);
    return det;
}

/* one mask's root 1/sqrt(det(I - A_Z)) in fixed point (torontonian.cpp:83-96) */
static int mask_root(const inp* a, u64 mask, unsigned f, int W, cw* scratch, wide* root, int* bad_row) {
    int d;
    extract(a, mask, f, W, scratch, &d);
    wide det;
    if (herm_det_fixed(scratch, d, f, W, &det, bad_row)) return -1;
    if (w_rsqrt(det, f, W, root)) {
        *bad_row = -1;
        return -1;
    }
    return 0;
}

/* ----------------------------------------------------- partial engines ---- */
typedef struct {
    const inp* a;
    int W;
    unsigned f;
    int k;          /* class bits (slice mode) or -1 (partition mode) */
    u64 cls_lo, cls_hi;
    int nproc, rank_lo, nranks;
    volatile u64 next;
    pthread_mutex_t mu;
    /* outputs */
    wide* class_sums;
    double* class_abs;
    u64 done;
    int err;
    u64 err_mask;
    int err_row;
} job_t;

static u64 take(job_t* j) {
    pthread_mutex_lock(&j->mu);
    const u64 v = j->next++;
    pthread_mutex_unlock(&j->mu);
    return v;
}

static void record_err(job_t* j, u64 mask, int row) {
    pthread_mutex_lock(&j->mu);
    if (!j->err || mask < j->err_mask) {
        j->err = 1;
        j->err_mask = mask;
        j->err_row = row;
    }
    pthread_mutex_unlock(&j->mu);
}

static void* slice_worker(void* p) {
    job_t* j = (job_t*)p;
    const int N = j->a->n, r = N - j->k;
    cw* scratch = malloc(sizeof(cw) * tri(2 * N, 2 * N - 1, 2 * N - 1) + sizeof(cw) * 2);
    for (;;) {
        const u64 i = take(j);
        if (i >= j->cls_hi - j->cls_lo) break;
        const u64 base = (j->cls_lo + i) << r;
        wide acc = {{0}};
        double sabs = 0.0;
        for (u64 low = 0; low < ((u64)1 << r); ++low) {
            const u64 mask = base | low;
            const int z = __builtin_popcountll(mask);
            if (z == 0) { /* empty set, rank-0 term (torontonian.cpp:98-101) */
                const wide one = w_one(j->f);
                acc = (N & 1) ? w_sub(acc, one, j->W) : w_add(acc, one, j->W);
                sabs += 1.0;
                continue;
            }
            wide root;
            int row;
            if (mask_root(j->a, mask, j->f, j->W, scratch, &root, &row)) {
                record_err(j, mask, row);
                break;
            }
            sabs += fabs(w_to_real(root, j->f, j->W));
            acc = ((N - z) & 1) ? w_sub(acc, root, j->W) : w_add(acc, root, j->W);
        }
        j->class_sums[i] = acc;
        j->class_abs[i] = sabs;
    }
    free(scratch);
    return NULL;
}

/* torontonian_partial over partition(N, rank, nproc) (torontonian.cpp:72-103) */
static void* partition_worker(void* p) {
    job_t* j = (job_t*)p;
    const int N = j->a->n;
    cw* scratch = malloc(sizeof(cw) * tri(2 * N, 2 * N - 1, 2 * N - 1) + sizeof(cw) * 2);
    u64 done = 0;
    for (;;) {
        const u64 i = take(j);
        if (i >= (u64)j->nranks) break;
        const int rank = j->rank_lo + (int)i;
        wide acc = {{0}};
        for (int z = 1; z <= N; ++z) {
            const u64 total = or_binom(N, z);
            const u64 lo = (u64)((u128)total * rank / j->nproc);
            const u64 hi = (u64)((u128)total * (rank + 1) / j->nproc);
            if (hi == lo) continue;
            u64 mask = or_get_kth_mask(N, z, lo);
            for (u64 t = 0; t < hi - lo; ++t, mask = or_get_next_mask(mask)) {
                wide root;
                int row;
                if (mask_root(j->a, mask, j->f, j->W, scratch, &root, &row)) {
                    record_err(j, mask, row);
                    goto out;
                }
                acc = ((N - z) & 1) ? w_sub(acc, root, j->W) : w_add(acc, root, j->W);
                ++done;
            }
        }
        if (rank == 0) {
            const wide one = w_one(j->f);
            acc = (N & 1) ? w_sub(acc, one, j->W) : w_add(acc, one, j->W);
        }
        j->class_sums[i] = acc;
    }
out:
    pthread_mutex_lock(&j->mu);
    j->done += done;
    pthread_mutex_unlock(&j->mu);
    free(scratch);
    return NULL;
}

static void run_threads(void* (*fn)(void*), job_t* j, int threads) {
    if (threads < 1) threads = 1;
    pthread_t* th = malloc(sizeof(pthread_t) * threads);
    for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, fn, j);
    fn(j);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
}

static void limbs_out(wide a, int W, uint64_t* out4) {
    for (int i = 0; i < 4; ++i) out4[i] = i < W ? a.w[i] : 0;
}

/* ------------------------------------------------------------ precision ---- */
static double det_i_minus_a(const inp* a, int* nonfinite) { /* precision.cpp:16-36 */
    const int n = a->n, d = 2 * n;
    double complex* m = malloc(sizeof(double complex) * (size_t)d * (d + 1) / 2);
    for (int i = 0; i < d; ++i)
        for (int j = i; j < d; ++j) {
            double complex v;
            if (j < n) v = a00_at(a, i, j);
            else if (i < n) v = a01_at(a, i, j - n);
            else v = conj(a00_at(a, i - n, j - n));
            m[tri(d, i, j)] = (i == j) ? 1.0 - v : -v;
        }
    const double det = herm_det_float(m, d, nonfinite);
    free(m);
    return det;
}

static int upper_bits(const inp* a, or_err* e) { /* precision.cpp:73-78 */
    int nf;
    const double det = det_i_minus_a(a, &nf);
    if (nf) {
        seterr(e, 3, "linalg/nonfinite", "non-finite determinant in float elimination", -1, 0);
        return -1;
    }
    if (!(det > 0.0)) {
        seterr(e, 3, "precision/det-nonpositive", "det(I-A) must be positive", -1, 0);
        return -1;
    }
    const int b = (int)ceil(-log2(det));
    return b > 1 ? b : 1;
}

static int lower_bits(int N, double a_repr, double k, int* out, or_err* e) { /* precision.cpp:52-71 */
    if (a_repr <= 0.0) {
        *out = 0;
        return 0;
    }
    if (!(a_repr < 1.0)) {
        seterr(e, 3, "precision/model-range", "representative diagonal must be < 1", -1, 0);
        return -1;
    }
    const double oma = 1.0 - a_repr;
    if (!(k * N / oma < oma)) {
        seterr(e, 3, "precision/model-range", "correction term leaves the model's validity domain", -1, 0);
        return -1;
    }
    const double base = (a_repr / oma) * pow(1.0 - k * N / (oma * oma), 2);
    const double bits = -(double)N * log2(base);
    const int b = (int)ceil(bits);
    *out = b > 0 ? b : 0;
    return 0;
}

int or_select_precision(int n, const double* a00, const double* a01, int N, int sig, double alpha, or_cfg* c,
                        or_err* e) { /* precision.cpp:80-121 */
    const inp a = {n, a00, a01};
    memset(c, 0, sizeof(*c));
    if (N < 1 || sig < 1 || !(alpha > 0.0)) {
        seterr(e, 1, "precision/range", "bad argument", -1, 0);
        return 1;
    }
    c->alpha = alpha;
    c->b_sgn = (int)ceil(sig * log2(10.0));
    c->b_accum = (int)ceil(log2(alpha) + N + 2.0 * log2(N));
    c->b_upper = upper_bits(&a, e);
    if (c->b_upper < 0) return 3;
    double diag = 0.0;
    for (int i = 0; i < n; ++i) diag += creal(a00_at(&a, i, i));
    c->a_repr = diag / n;
    int nf;
    const double det = det_i_minus_a(&a, &nf);
    double kf = 0.0035;
    if (c->a_repr > 0.0 && c->a_repr < 1.0) {
        const double oma = 1.0 - c->a_repr;
        const double fitted = (oma * oma - pow(det, 1.0 / N)) / N;
        if (isfinite(fitted)) kf = fitted;
    }
    c->k_corr = kf < 0.0009 ? 0.0009 : (kf > 0.0035 ? 0.0035 : kf);
    if (lower_bits(N, c->a_repr, c->k_corr, &c->b_lower, e)) return 3;
    const int B = c->b_lower + c->b_upper + c->b_sgn + c->b_accum;
    if (B <= 128) c->width_bits = 128;
    else if (B <= 256) c->width_bits = 256;
    else {
        seterr(e, 3, "precision/unsupported", "required bit budget exceeds 256 bits", -1, 0);
        return 3;
    }
    c->frac_bits = c->width_bits - 1 - c->b_upper;
    return 0;
}

int or_force_width(int n, const double* a00, const double* a01, int width, or_cfg* c, or_err* e) {
    /* precision.cpp:123-148 */
    const inp a = {n, a00, a01};
    memset(c, 0, sizeof(*c));
    if (width != 128 && width != 256) {
        seterr(e, 1, "precision/range", "width must be 128 or 256", -1, 0);
        return 1;
    }
    c->width_bits = width;
    c->alpha = 0.5;
    c->b_sgn = (int)ceil(3 * log2(10.0));
    c->b_upper = upper_bits(&a, e);
    if (c->b_upper < 0) return 3;
    c->b_accum = (int)ceil(log2(0.5) + n + 2.0 * log2(n));
    double diag = 0.0;
    for (int i = 0; i < n; ++i) diag += creal(a00_at(&a, i, i));
    c->a_repr = diag / n;
    c->k_corr = 0.0035;
    const int f = width - 1 - c->b_upper;
    if (f < 1) {
        seterr(e, 3, "precision/scaling", "upper bound leaves no room for fraction bits at this width", -1, 0);
        return 3;
    }
    c->frac_bits = f;
    or_err ignore;
    if (lower_bits(n, c->a_repr, c->k_corr, &c->b_lower, &ignore)) c->b_lower = 0;
    return 0;
}

/* ---------------------------------------------------------------- API ---- */
int or_slice(int n, const double* a00, const double* a01, int width, int frac_bits, int k, uint64_t lo,
             uint64_t hi, int threads, uint64_t* class_limbs, double* class_abs, uint64_t* total_limbs,
             or_err* e) {
    const inp a = {n, a00, a01};
    const int W = width / 64;
    if ((W != 2 && W != 4) || k < 0 || k > n || hi <= lo || frac_bits < 1 || frac_bits > 64 * W - 2) {
        seterr(e, 1, "oracle/range", "bad slice", -1, 0);
        return 1;
    }
    job_t j;
    memset(&j, 0, sizeof(j));
    j.a = &a;
    j.W = W;
    j.f = (unsigned)frac_bits;
    j.k = k;
    j.cls_lo = lo;
    j.cls_hi = hi;
    pthread_mutex_init(&j.mu, NULL);
    j.class_sums = calloc(hi - lo, sizeof(wide));
    j.class_abs = calloc(hi - lo, sizeof(double));
    run_threads(slice_worker, &j, threads);
    pthread_mutex_destroy(&j.mu);
    int st = 0;
    if (j.err) {
        seterr(e, 2, "linalg/breakdown", "non-positive pivot in elimination", j.err_row, j.err_mask);
        st = 2;
    } else {
        wide tot = {{0}};
        for (u64 i = 0; i < hi - lo; ++i) {
            tot = w_add(tot, j.class_sums[i], W);
            if (class_limbs) limbs_out(j.class_sums[i], W, class_limbs + 4 * i);
            if (class_abs) class_abs[i] = j.class_abs[i];
        }
        if (total_limbs) limbs_out(tot, W, total_limbs);
    }
    free(j.class_sums);
    free(j.class_abs);
    return st;
}

int or_torontonian(int n, const double* a00, const double* a01, int precision, int threads, double* value,
                   uint64_t* limbs4, or_cfg* cfg, or_err* e) { /* torontonian.cpp:151-177 */
    if (n < 1 || n > 40) {
        seterr(e, 1, "torontonian/range", "engine supports 1 <= N <= 40", -1, 0);
        return 1;
    }
    int st = precision == 0 ? or_select_precision(n, a00, a01, n, 3, 0.5, cfg, e)
                            : or_force_width(n, a00, a01, precision == 1 ? 128 : 256, cfg, e);
    if (st) return st;
    const int W = cfg->width_bits / 64;
    uint64_t tot[4];
    const int k = n < 8 ? n : 8;
    st = or_slice(n, a00, a01, cfg->width_bits, (int)cfg->frac_bits, k, 0, (uint64_t)1 << k, threads, NULL, NULL,
                  tot, e);
    if (st) return st;
    wide acc = {{0}};
    for (int i = 0; i < W; ++i) acc.w[i] = tot[i];
    *value = w_to_real(acc, cfg->frac_bits, W);
    for (int i = 0; i < 4; ++i) limbs4[i] = tot[i];
    return 0;
}

int or_torontonian_reference(int n, const double* a00, const double* a01, double* value, or_err* e) {
    /* torontonian.cpp:179-200 */
    if (n < 1 || n > 20) {
        seterr(e, 1, "torontonian/range", "reference path supports 1 <= N <= 20", -1, 0);
        return 1;
    }
    const inp a = {n, a00, a01};
    double acc = (n & 1) ? -1.0 : 1.0;
    double complex* m = malloc(sizeof(double complex) * (size_t)(2 * n) * (2 * n + 1) / 2);
    for (int z = 1; z <= n; ++z) {
        const u64 total = or_binom(n, z);
        u64 mask = or_get_kth_mask(n, z, 0);
        for (u64 t = 0; t < total; ++t, mask = or_get_next_mask(mask)) {
            int sel[64], zz = 0;
            for (int j = 0; j < n; ++j)
                if ((mask >> (n - 1 - j)) & 1) sel[zz++] = j;
            const int d = 2 * zz;
            for (int p = 0; p < d; ++p)
                for (int q = p; q < d; ++q) {
                    double complex v;
                    if (q < zz) v = a00_at(&a, sel[p], sel[q]);
                    else if (p < zz) v = a01_at(&a, sel[p], sel[q - zz]);
                    else v = conj(a00_at(&a, sel[p - zz], sel[q - zz]));
                    m[tri(d, p, q)] = (p == q) ? (double complex)(1.0 - creal(v)) : -v;
                }
            int nf;
            const double det = herm_det_float(m, d, &nf);
            const double term = 1.0 / sqrt(det);
            if (nf || !isfinite(term)) {
                free(m);
                seterr(e, 3, nf ? "linalg/nonfinite" : "torontonian/nonfinite", "non-finite term", -1, mask);
                return 3;
            }
            acc += ((n - z) & 1) ? -term : term;
        }
    }
    free(m);
    *value = acc;
    return 0;
}

int or_partial_sample(int n, const double* a00, const double* a01, int width, int nproc, int rank_lo,
                      int nranks, int threads, uint64_t* done, double* seconds, or_err* e) {
    const inp a = {n, a00, a01};
    or_cfg c;
    const int st = or_force_width(n, a00, a01, width, &c, e);
    if (st) return st;
    job_t j;
    memset(&j, 0, sizeof(j));
    j.a = &a;
    j.W = width / 64;
    j.f = c.frac_bits;
    j.nproc = nproc;
    j.rank_lo = rank_lo;
    j.nranks = nranks;
    pthread_mutex_init(&j.mu, NULL);
    j.class_sums = calloc((size_t)nranks, sizeof(wide));
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    run_threads(partition_worker, &j, threads);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    pthread_mutex_destroy(&j.mu);
    free(j.class_sums);
    *done = j.done;
    *seconds = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);
    if (j.err) {
        seterr(e, 2, "linalg/breakdown", "non-positive pivot in elimination", j.err_row, j.err_mask);
        return 2;
    }
    return 0;
}

int or_wide_mul(const uint64_t* a, const uint64_t* b, int width, unsigned f, uint64_t* out) {
    wide x = {{0}}, y = {{0}};
    const int W = width / 64;
    for (int i = 0; i < W; ++i) {
        x.w[i] = a[i];
        y.w[i] = b[i];
    }
    limbs_out(w_mul(x, y, f, W), W, out);
    return 0;
}

int or_wide_rsqrt(const uint64_t* a, int width, unsigned f, uint64_t* out) {
    wide x = {{0}}, r;
    const int W = width / 64;
    for (int i = 0; i < W; ++i) x.w[i] = a[i];
    const int st = w_rsqrt(x, f, W, &r);
    if (st) return st;
    limbs_out(r, W, out);
    return 0;
}
