/* TEST INFRASTRUCTURE ONLY: C restatement of the reference engine (see tor_oracle.c). */
#ifndef TOR_ORACLE_H
#define TOR_ORACLE_H
#include <stdint.h>

typedef struct {
    int status; /* 1 InvalidArgument, 2 Breakdown, 3 Precision */
    char code[48];
    char message[160];
    int64_t row;
    uint64_t mask;
} or_err;

typedef struct {
    int width_bits;
    unsigned frac_bits;
    int b_lower, b_upper, b_sgn, b_accum;
    double a_repr, k_corr, alpha;
} or_cfg;

uint64_t or_binom(int n, int k);
uint64_t or_get_kth_mask(int N, int z, uint64_t k);
uint64_t or_get_next_mask(uint64_t mask);
int or_select_precision(int n, const double* a00, const double* a01, int N, int sig, double alpha, or_cfg* c,
                        or_err* e);
int or_force_width(int n, const double* a00, const double* a01, int width, or_cfg* c, or_err* e);
int or_torontonian(int n, const double* a00, const double* a01, int precision, int threads, double* value,
                   uint64_t* limbs4, or_cfg* cfg, or_err* e);
int or_torontonian_reference(int n, const double* a00, const double* a01, double* value, or_err* e);
int or_slice(int n, const double* a00, const double* a01, int width, int frac_bits, int k, uint64_t lo,
             uint64_t hi, int threads, uint64_t* class_limbs, double* class_abs, uint64_t* total_limbs, or_err* e);
int or_partial_sample(int n, const double* a00, const double* a01, int width, int nproc, int rank_lo, int nranks,
                      int threads, uint64_t* done, double* seconds, or_err* e);
int or_wide_mul(const uint64_t* a, const uint64_t* b, int width, unsigned f, uint64_t* out);
int or_wide_rsqrt(const uint64_t* a, int width, unsigned f, uint64_t* out);
#endif
