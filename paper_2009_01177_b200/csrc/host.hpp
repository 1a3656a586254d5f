// Host-side pieces of the engine (plain C++, no device code): the data model, the
// reference's validation and precision-selection logic restated for the C ABI, the
// exact R = T (I - O) T^H builder, and the closed-form operation counts.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace tor {

struct HostError : std::runtime_error {
    int status;
    std::string code;
    int64_t pivot_row = -1;
    uint64_t subset_mask = 0;
    HostError(int st, std::string c, const std::string& msg)
        : std::runtime_error(msg), status(st), code(std::move(c)) {}
};

// InputMatrix (matrix_io.hpp:18-26): two upper triangles, row-major.
struct Input {
    int n = 0;
    std::vector<std::complex<double>> a00, a01;
    std::complex<double> a00_at(int i, int j) const;  // matrix_io.cpp:80-83
    std::complex<double> a01_at(int i, int j) const;  // matrix_io.cpp:85-88
};

struct PrecCfg {
    int width_bits = 128;
    unsigned frac_bits = 0;
    int b_lower = 0, b_upper = 0, b_sgn = 0, b_accum = 0;
    double a_repr = 0.0, k_corr = 0.0, alpha = 0.5;
    int total_bits() const { return b_lower + b_upper + b_sgn + b_accum; }
};

struct SymReport {
    double hermitian_dev = 0, a01_sym_dev = 0, block_conj_dev = 0;
    bool pass = false;
};

Input make_input(int n, const double* a00, const double* a01);
std::vector<std::complex<double>> to_dense(const Input& a);
SymReport check_symmetries(const std::vector<std::complex<double>>& dense, int two_n);
// check_symmetries(to_dense(a), 2n) without the dense matrix (identical report)
SymReport check_symmetries_tri(const Input& a);
double det_i_minus_a_float(const Input& a);
PrecCfg select_precision(const Input& a, int N, int sig, double alpha);
PrecCfg force_width(const Input& a, int width_bits);

// Exact R in `words` doubles per entry (1: rounded fp64, 2: DD, 4: QD), packed upper
// triangle of the 2n x 2n matrix in pair order (x_0, p_0, x_1, p_1, ...).
std::vector<double> build_R(const Input& a, int words, bool grid = false, int* tscale_log2 = nullptr);
// the same into R (tri(2n) * words doubles)
void build_R_into(const Input& a, int words, bool grid, double* R, int* tscale_log2, bool stream = false);
// the same from interleaved (re, im) upper triangles (tor_input layout), no Input copy
void build_R_raw(int n, const double* a00, const double* a01, int words, bool grid, double* R, int* tscale_log2,
                 bool stream = false);
// stream = true writes R with non-temporal stores (pinned staging the GPU reads next: DMA reads
// of lines still dirty in the host caches are ~10x slower); build_R_fence() orders them before
// the copy is enqueued
void build_R_fence();

// Closed-form reference op counters (linalg.hpp:44-57, flops.cpp:9-31).
void op_counts(int n, uint64_t& mults, uint64_t& adds, uint64_t& recips, uint64_t& rsqrts);
unsigned __int128 total_op_count(int n);

Input extract_submatrix(const Input& full, uint64_t pattern_bits);
Input extract_modes(const Input& full, const std::vector<int>& ascending_modes);

// GBSA instance files (gbsa.cpp; matrix_io.cpp:92-263): format sniffed from the magic on
// load (*quant_bits = 16/32 for binary, 0 for text); save as text or binary (16/32 bits).
Input load_gbsa(const uint8_t* bytes, size_t len, int* quant_bits);
std::string save_gbsa(const Input& a, bool binary, int quant_bits);
int64_t quantize(double x, int bits);
double quant_unit(int bits);

}  // namespace tor
