/*
 * tor_capi.h -- C ABI of the B200 Torontonian engine (libtor_b200.so).
 *
 * Drop-in boundary for the reference's hot path (torfp, /root/reference/proj):
 *
 *   reference C++ entry point                                      replaced by
 *   ---------------------------------------------------------------------------------
 *   TorontonianResult torontonian(const InputMatrix&,              tor_torontonian
 *       PrecisionChoice = Auto, int workers = 0)
 *       (include/torfp/torontonian.hpp:50-51, src/torontonian.cpp:151-177)
 *   double torontonian_reference(const InputMatrix&)               tor_torontonian_reference
 *       (torontonian.hpp:55, torontonian.cpp:179-200)
 *   PrecisionConfig select_precision(const InputMatrix&, int N,    tor_select_precision
 *       int sig = 3, double alpha = 0.5)
 *       (precision.hpp:66-67, precision.cpp:80-121)
 *   PrecisionConfig force_width(const InputMatrix&, int width)     tor_force_width
 *       (precision.hpp:71, precision.cpp:123-148)
 *   Wide<W> torontonian_partial<W>(a, WorkAssignment, cfg, ops)    tor_torontonian_slice
 *       (torontonian.hpp:43-45, torontonian.cpp:72-103)             (prefix-class shards)
 *   double det_i_minus_a_float(const InputMatrix&)                 tor_det_i_minus_a
 *       (precision.hpp:61, precision.cpp:34-36)
 *   SymmetryReport check_symmetries(dense, 2N)                     tor_check_symmetries
 *       (matrix_io.hpp:64, matrix_io.cpp:285-305)
 *   double probability(a_full, ClickPattern, workers)              tor_probability
 *       (torontonian.hpp:60, torontonian.cpp:202-209)
 *   (new) many-instance throughput path, BASELINE config 3         tor_torontonian_batch
 *   (new) fixed-order fold of shard partials (multi-GPU)           tor_fold_partials
 *
 * Conventions
 *   - Input: InputMatrix (matrix_io.hpp:18-26): two upper triangles of n(n+1)/2
 *     complex entries, row-major, index i*n - i(i+1)/2 + j, interleaved (re, im)
 *     doubles.  Caller-owned, read-only for the call.
 *   - Subset masks follow the reference (subsets.hpp:11-13): bit N-1-j = mode j.
 *     Prefix classes are the top `class_bits` bits of that mask.
 *   - No exceptions cross the ABI.  Every entry point returns a status (TOR_OK or
 *     one of TOR_E_*), mapped 1:1 onto the reference's error classes
 *     (errors.hpp:13-78), and fills *err (may be NULL) with the same stable
 *     "module/kind" code strings the reference throws.
 *   - Reentrant.  No hidden global state besides a per-device context cache
 *     guarded by a mutex.  `devices` replaces the reference's `workers`.
 */
#ifndef TOR_CAPI_H
#define TOR_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TOR_ABI_VERSION 1

/* status codes (errors.hpp class -> code) */
#define TOR_OK 0
#define TOR_E_INVALID 1   /* InvalidArgument */
#define TOR_E_BREAKDOWN 2 /* BreakdownError (non-positive pivot) */
#define TOR_E_PRECISION 3 /* PrecisionError */
#define TOR_E_PARSE 4     /* ParseError */
#define TOR_E_RESOURCE 5  /* ResourceError */
#define TOR_E_DEVICE 6    /* CUDA / NCCL failure (no reference counterpart) */
#define TOR_E_ERROR 7     /* plain Error, e.g. "torontonian/symmetry" */

/* precision selector: PrecisionChoice {Auto, Bits128, Bits256} (torontonian.hpp:31)
 * plus the fp64 oracle path.  128-bit -> double-double, 256-bit -> quad-double. */
typedef enum {
    TOR_PREC_AUTO = 0,
    TOR_PREC_W128_DD = 1,
    TOR_PREC_W256_QD = 2,
    TOR_PREC_FP64 = 3,
    /* exact fixed-point validation modes (n <= 24): the reference's own per-subset
     * algorithm on the GPU integer pipes; raw_limbs identical to the reference */
    TOR_PREC_FIXED128 = 4,
    TOR_PREC_FIXED256 = 5
} tor_precision;

typedef struct {
    int n;                   /* modes N (InputMatrix::n_modes) */
    const double* a00_upper; /* n(n+1)/2 complex, interleaved (re, im): A00, Hermitian */
    const double* a01_upper; /* n(n+1)/2 complex, interleaved (re, im): A01, symmetric */
} tor_input;

/* PrecisionConfig (precision.hpp:17-29) */
typedef struct {
    int width_bits;
    unsigned frac_bits;
    int b_lower;
    int b_upper;
    int b_sgn;
    int b_accum;
    double a_repr;
    double k_corr;
    double alpha;
} tor_precision_config;

typedef struct {
    char code[48];      /* "module/kind", as the reference's Error::code() */
    char message[200];
    int64_t pivot_row;  /* BreakdownError::pivot_row (pair order 2k: x_k, 2k+1: p_k), -1 n/a */
    uint64_t subset_mask; /* BreakdownError::subset_mask (reference convention), 0 n/a.  The engine
                             checks both pivots of every eliminated mode (leaf modes included) and
                             reports the numerically smallest failing mask, independent of the
                             schedule, the device count and the shard layout */
} tor_error;

/* TorontonianResult (torontonian.hpp:21-29) extended with the multi-word value and
 * the posterior cancellation check of the adaptive driver. */
typedef struct {
    double value;             /* nearest double of the multi-word sum */
    int mode;                 /* tor_precision actually used (never AUTO) */
    int width_bits;           /* 64 (fp64), 128 (DD) or 256 (QD) */
    int nwords;               /* significant words in `words` (1, 2 or 4) */
    double words[4];          /* unevaluated-sum value, leading word first */
    tor_precision_config config; /* select_precision / force_width outcome */
    uint64_t term_count;      /* 2^N (or the slice's share) */
    /* OpCounters (linalg.hpp:44-57) as closed-form equivalents of the reference's
     * per-subset elimination: mults + adds = Eq. 8, recips = sum C(n,z)(2z-1),
     * rsqrts = 2^n - 1 */
    uint64_t mults, adds, recips, rsqrts;
    double wall_seconds;      /* host-to-result wall time of the call */
    double device_ms;         /* device time of the engine pipeline (CUDA events) */
    double kernel_ms;         /* device time of the subtree kernel */
    int devices;              /* GPUs used */
    int escalated;            /* 1 when the adaptive driver re-ran DD as QD */
    double sum_abs_terms;     /* sum over subsets of |term| (fp64) */
    double cancellation_bits; /* log2(sum|t| / |Tor|) */
    double bits_left;         /* mantissa - cancellation - growth allowance */
    uint64_t kernel_launches; /* device kernels launched by the call */
    uint64_t h2d_bytes;       /* host->device bytes copied by the call */
    uint64_t d2h_bytes;       /* device->host bytes copied by the call */
    uint64_t raw_limbs[4];    /* FixedValue limbs (torontonian.hpp:14-29), low limb first:
                                 FIXED modes: the exact accumulator (identical to the
                                 reference's); DD/QD: round(sum(words) * 2^config.frac_bits)
                                 (ties toward +inf, exact) as width_bits two's complement;
                                 fp64: 0 */
} tor_result;

/* Shard partial for multi-GPU / multi-process folds: a contiguous, power-of-two
 * aligned range of prefix classes reduced along the engine's fixed binary tree. */
typedef struct {
    int mode;
    int class_bits;
    uint64_t class_lo, class_hi;
    double words[4];
    double sum_abs;
    uint64_t term_count;
} tor_partial;

/* ------------------------------------------------------------------ API -- */
int tor_abi_version(void);

/* check_symmetries with the reference's 1e-12 gate; devs = {hermitian, a01_sym,
 * block_conj}. */
int tor_check_symmetries(const tor_input* in, double devs[3], int* pass, tor_error* err);

/* Same gate on a dense 2N x 2N complex matrix (interleaved), as from_dense. */
int tor_check_dense(int two_n, const double* dense, double devs[3], int* pass, tor_error* err);

/* det(I - A) in floating point, reference elimination order (precision.cpp:34). */
int tor_det_i_minus_a(const tor_input* in, double* det, tor_error* err);

int tor_select_precision(const tor_input* in, int N, int sig_decimal_digits, double alpha,
                         tor_precision_config* out, tor_error* err);
int tor_force_width(const tor_input* in, int width_bits, tor_precision_config* out, tor_error* err);

/* Full evaluation (validation N in [1,40], symmetry gate, precision selection,
 * adaptive escalation, device evaluation).  devices == NULL / ndev <= 0: device 0.  With
 * ndev > 1 the 64 top-level prefix classes split into ndev contiguous ranges (any device
 * count <= 64; sizes differ by at most one class), one host thread per listed device, and
 * the per-class partials fold along the fixed tree: bit-identical to one device;
 * out->devices = the devices used (the reference's `workers` fan-out).  Instances with
 * fewer than 6 prefix levels (N < 15 in DD, 16 in fp64, 14 in QD) run on the first device.
 * AUTO: the width select_precision picks (128 -> DD, 256 -> QD), then the posterior check:
 * if fewer than b_sgn bits survive the cancellation (bits_left < b_sgn; a sum that cancels
 * to exactly 0 counts as no bits left unless the input is exactly zero), DD re-runs in QD
 * (escalated = 1), and a QD result that still fails raises PrecisionError
 * "precision/insufficient". */
int tor_torontonian(const tor_input* in, tor_precision prec, const int* devices, int ndev,
                    tor_result* out, tor_error* err);

/* fp64 oracle semantics (N <= 20, PrecisionError "torontonian/nonfinite"), computed
 * on the device by the same engine in fp64.  Like the reference there is no pivot check:
 * a non-positive pivot makes the sum non-finite ("torontonian/nonfinite").  Difference: on
 * an input whose I - A_Z has a negative-definite 2x2 mode block (det > 0) the reference's
 * LU-style elimination returns a finite number, this Cholesky-based path "nonfinite"; such
 * inputs are not physical states (I - A must be positive definite). */
int tor_torontonian_reference(const tor_input* in, double* value, tor_error* err);

/* `count` instances of equal N in one device pass (BASELINE config 3); prec AUTO, 128, 256 or
 * fp64.  AUTO selects the width per instance exactly as tor_torontonian (DD and QD
 * sub-batches) including the posterior check: failing DD instances re-run in QD, and a QD
 * instance that fails it raises "precision/insufficient" naming the instance; validation
 * errors report the first bad instance in index order. */
int tor_torontonian_batch(const tor_input* ins, int count, tor_precision prec, int device,
                          tor_result* outs, tor_error* err);

/* Partial sum over prefix classes [class_lo, class_hi) of the top class_bits mask
 * bits on one device (the subset of torontonian_partial's masks with those
 * prefixes).  prec: 128, 256 or fp64.  N in [1, 50] (beyond the reference's 40: the
 * paper's n = 50 case as checkpointable class ranges); slices, shards and plans only. */
int tor_torontonian_slice(const tor_input* in, tor_precision prec, int class_bits, uint64_t class_lo,
                          uint64_t class_hi, int device, tor_partial* out, tor_error* err);

/* Schedule hints for tor_torontonian_classes (0 = the default schedule).  prefix_jobs sets
 * the prefix depth c (the smallest c with 2^c >= prefix_jobs, capped by the problem), and so
 * the depth of the producer DFS below it; blocks_per_sm overrides the subtree kernel's CTAs
 * per SM.  Results stay within the mode's tolerance; they are bit-identical only between
 * runs with the same prefix_jobs.  Replaces round-1's TOR_WANT_JOBS / TOR_BLOCKS_PER_SM
 * environment knobs (the library reads no environment variable that changes results;
 * TOR_DEBUG_TIMING=1 only prints host/device timings to stderr). */
typedef struct {
    uint64_t prefix_jobs;
    int blocks_per_sm;
    int reserved;
} tor_schedule;

/* One partial per prefix class of [class_lo, class_hi) (class_hi - class_lo <= 2^24 entries in
 * outs, in class order) from ONE device pass.  Each class partial is an aligned subtree of
 * the engine's fixed fold tree, so any assignment of classes to devices or processes folds
 * bit-identically with tor_fold_partials (this is how N devices that are not a power of two
 * split a Torontonian).  sched may be NULL. */
int tor_torontonian_classes(const tor_input* in, tor_precision prec, int class_bits, uint64_t class_lo,
                            uint64_t class_hi, int device, const tor_schedule* sched, tor_partial* outs,
                            tor_error* err);

/* Rank `rank` of `world` (power of two) evaluates its aligned share of the 2^k
 * top-level classes. */
int tor_torontonian_shard(const tor_input* in, tor_precision prec, int rank, int world, int device,
                          tor_partial* out, tor_error* err);

/* Fold shard partials along the engine's fixed tree; bit-identical to a single-device run.
 * The partials must share mode and class_bits, be sorted and contiguous, cover every class
 * [0, 2^class_bits), each span an aligned power-of-two class range (lo % width == 0), and
 * their term counts must add up to 2^N; otherwise TOR_E_INVALID "torontonian/shard"
 * (e.g. a rank missing from an all-gather). */
int tor_fold_partials(const tor_partial* parts, int count, const tor_input* in, tor_result* out,
                      tor_error* err);

/* p(S) = Tor(A_S) sqrt(det(I - A)) (torontonian.cpp:202-209); pattern bit k = mode k. */
int tor_probability(const tor_input* full, uint64_t pattern_bits, tor_precision prec, int device,
                    double* p, tor_error* err);
/* The same with the click pattern as an ascending list of mode indices: no 64-mode limit on
 * the full state (the reference's ClickPattern is one u64, matrix_io.hpp:29-34). */
int tor_probability_modes(const tor_input* full, const int* modes, int nmodes, tor_precision prec, int device,
                          double* p, tor_error* err);

/* Prepared evaluation with device-resident inputs (the exact R is uploaded once):
 * create -> execute (repeatable; runs the whole device pipeline and reads back the
 * result words) -> destroy.  The range is [class_lo, class_hi) of the top class_bits
 * mask bits ([0,1) of 0 bits = the whole Torontonian).  prec: 128, 256 or fp64. */
typedef struct tor_plan tor_plan;
int tor_plan_create(const tor_input* in, tor_precision prec, int class_bits, uint64_t class_lo,
                    uint64_t class_hi, int device, tor_plan** out, tor_error* err);
int tor_plan_execute(tor_plan* plan, tor_result* out, tor_error* err);
void tor_plan_destroy(tor_plan* plan);

/* GBSA instance files (load_matrix_file / save_matrix, matrix_io.cpp:109-263; SURVEY 8(f)
 * rank 3).  Binary: "GBSA", u16 version 1, u32 N, u8 bits (16/32), then the A00 and A01 upper
 * triangles as (re, im) signed little-endian integers x 2^-(bits-1).  Text: "GBSA text 1",
 * "modes N", one "re im" line per entry.  tor_load_matrix sniffs the format from the magic
 * as the reference does; *n (and *quant_bits: 16/32 binary, 0 text) are always set, and the
 * triangles are written when both pointers are non-NULL (capacity >= N(N+1)/2 complex
 * entries; call once with NULL to size).  Parse errors: TOR_E_PARSE with the reference's
 * codes ("matrixio/magic|version|format|dim|truncated|entry|range") and the position (byte
 * offset / 1-based line) in err->pivot_row.  tor_save_matrix: format 0 text, 1 binary
 * (quant_bits 16/32, entries must satisfy |x| < 1); *len = the full size, min(len, capacity)
 * bytes are copied to buf (buf may be NULL). */
int tor_load_matrix(const void* bytes, size_t len, int* n, int* quant_bits, double* a00_upper, double* a01_upper,
                    size_t capacity, tor_error* err);
int tor_save_matrix(const tor_input* in, int format, int quant_bits, void* buf, size_t capacity, size_t* len,
                    tor_error* err);

/* Number of CUDA devices visible (0 without a GPU). */
int tor_device_count(void);

/* Frees the device memory the library keeps pooled between calls (plans reuse the
 * prefix pools / DFS scratch of finished calls; no reference counterpart). */
void tor_release_device_cache(void);

#ifdef __cplusplus
}
#endif

#endif /* TOR_CAPI_H */
