// Host-side restatement of the reference's validation / precision logic for the C
// ABI.  The decisions (widths, bit budgets, fraction bits, k_corr) must be
// bit-identical to the reference's select_precision / force_width, so the
// floating-point expressions keep the reference's evaluation order; the cited
// lines are the behaviour each function reproduces.  Built with -O3 and
// -ffp-contract=off.
#include "host.hpp"

#if defined(__x86_64__)
#include <emmintrin.h>
#endif

#include <algorithm>
#include <cmath>
#include <cstring>

#include "../../include/tor_capi.h"
#include "arith.cuh"

namespace tor {

namespace {

constexpr double kTol = 1e-12;          // matrix_io.hpp:62
constexpr double kCorrMin = 0.0009;     // precision.cpp:11
constexpr double kCorrMax = 0.0035;     // precision.cpp:12

inline size_t tri(int n, int i, int j) {
    return static_cast<size_t>(i) * n - static_cast<size_t>(i) * (i + 1) / 2 + static_cast<size_t>(j);
}

// Packed complex upper triangle of dim d (HermitianFloat, linalg.hpp:27-30).
struct HermF {
    int d = 0;
    std::vector<std::complex<double>> u;
    std::complex<double>& at(int i, int j) { return u[tri(d, i, j)]; }
};

// hermitian_det_float (linalg.cpp:66-88): pivot product of the upper-triangle
// elimination in double; non-finite -> PrecisionError("linalg/nonfinite").
double herm_det(HermF m) {
    const int n = m.d;
    double det = 1.0;
    for (int k = 0; k < n; ++k) {
        const double pivot = m.at(k, k).real();
        det *= pivot;
        if (k == n - 1) break;
        const double pinv = 1.0 / pivot;
        for (int i = k + 1; i < n; ++i) {
            const std::complex<double> s = std::conj(m.at(k, i)) * pinv;
            m.at(i, i) -= std::complex<double>((s * m.at(k, i)).real(), 0.0);
            for (int j = i + 1; j < n; ++j) m.at(i, j) -= s * m.at(k, j);
        }
    }
    if (!std::isfinite(det))
        throw HostError(TOR_E_PRECISION, "linalg/nonfinite", "non-finite determinant in float elimination");
    return det;
}

int upper_bits(const Input& a) {  // precision.cpp:73-78
    const double det = det_i_minus_a_float(a);
    if (!(det > 0.0)) throw HostError(TOR_E_PRECISION, "precision/det-nonpositive", "det(I-A) must be positive");
    return std::max(1, static_cast<int>(std::ceil(-std::log2(det))));
}

int lower_bits(int N, double a_repr, double k_corr) {  // precision.cpp:52-71
    if (N < 1) throw HostError(TOR_E_INVALID, "precision/range", "N must be >= 1");
    if (a_repr <= 0.0) return 0;
    if (!(a_repr < 1.0))
        throw HostError(TOR_E_PRECISION, "precision/model-range", "representative diagonal must be < 1");
    const double one_minus_a = 1.0 - a_repr;
    if (!(k_corr * N / one_minus_a < one_minus_a))
        throw HostError(TOR_E_PRECISION, "precision/model-range",
                        "correction term leaves the model's validity domain");
    const double base = (a_repr / one_minus_a) * std::pow(1.0 - k_corr * N / (one_minus_a * one_minus_a), 2);
    const double bits = -static_cast<double>(N) * std::log2(base);
    return std::max(0, static_cast<int>(std::ceil(bits)));
}

}  // namespace

std::complex<double> Input::a00_at(int i, int j) const {
    if (i <= j) return a00[tri(n, i, j)];
    return std::conj(a00[tri(n, j, i)]);
}
std::complex<double> Input::a01_at(int i, int j) const {
    if (i <= j) return a01[tri(n, i, j)];
    return a01[tri(n, j, i)];
}

Input make_input(int n, const double* a00, const double* a01) {
    Input m;
    m.n = n;
    const size_t t = static_cast<size_t>(n) * (n + 1) / 2;
    m.a00.resize(t);
    m.a01.resize(t);
    for (size_t i = 0; i < t; ++i) {
        m.a00[i] = {a00[2 * i], a00[2 * i + 1]};
        m.a01[i] = {a01[2 * i], a01[2 * i + 1]};
    }
    return m;
}

std::vector<std::complex<double>> to_dense(const Input& a) {  // matrix_io.cpp:265-283
    const int n = a.n, d = 2 * n;
    std::vector<std::complex<double>> m(static_cast<size_t>(d) * d);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const auto v00 = a.a00_at(i, j);
            const auto v01 = a.a01_at(i, j);
            m[static_cast<size_t>(i) * d + j] = v00;
            m[static_cast<size_t>(i) * d + n + j] = v01;
            m[static_cast<size_t>(n + i) * d + j] = std::conj(v01);
            m[static_cast<size_t>(n + i) * d + n + j] = std::conj(v00);
        }
    return m;
}

SymReport check_symmetries(const std::vector<std::complex<double>>& dense, int two_n) {  // matrix_io.cpp:285-305
    if (two_n < 2 || two_n % 2 != 0 || dense.size() != static_cast<size_t>(two_n) * two_n)
        throw HostError(TOR_E_INVALID, "matrixio/dim", "dense matrix must be 2N x 2N");
    const int n = two_n / 2;
    auto at = [&](int i, int j) { return dense[static_cast<size_t>(i) * two_n + j]; };
    SymReport r;
    for (int i = 0; i < two_n; ++i)
        for (int j = 0; j < two_n; ++j) r.hermitian_dev = std::max(r.hermitian_dev, std::abs(at(i, j) - std::conj(at(j, i))));
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            r.a01_sym_dev = std::max(r.a01_sym_dev, std::abs(at(i, n + j) - at(j, n + i)));
            r.block_conj_dev = std::max(r.block_conj_dev, std::abs(at(i, j) - std::conj(at(n + i, n + j))));
        }
    r.pass = r.hermitian_dev <= kTol && r.a01_sym_dev <= kTol && r.block_conj_dev <= kTol;
    return r;
}

SymReport check_symmetries_tri(const Input& a) {
    // The dense matrix of a triangle-stored input (to_dense) mirrors every off-diagonal entry
    // exactly, so of check_symmetries' deviations only the A00 / conj(A00) diagonal can be
    // nonzero: |a_ii - conj(a_ii)|.  Same values, same gate, O(n) instead of O(n^2).
    SymReport r;
    for (int i = 0; i < a.n; ++i) {
        const std::complex<double> v = a.a00_at(i, i);
        r.hermitian_dev = std::max(r.hermitian_dev, std::abs(v - std::conj(v)));
    }
    r.pass = r.hermitian_dev <= kTol && r.a01_sym_dev <= kTol && r.block_conj_dev <= kTol;
    return r;
}

double det_i_minus_a_float(const Input& a) {  // precision.cpp:16-36
    const int n = a.n, d = 2 * n;
    HermF m;
    m.d = d;
    m.u.resize(static_cast<size_t>(d) * (d + 1) / 2);
    for (int i = 0; i < d; ++i)
        for (int j = i; j < d; ++j) {
            std::complex<double> v;
            if (j < n) v = a.a00_at(i, j);
            else if (i < n) v = a.a01_at(i, j - n);
            else v = std::conj(a.a00_at(i - n, j - n));
            m.at(i, j) = (i == j) ? 1.0 - v : -v;
        }
    return herm_det(m);
}

PrecCfg select_precision(const Input& a, int N, int sig, double alpha) {  // precision.cpp:80-121
    if (N < 1) throw HostError(TOR_E_INVALID, "precision/range", "N must be >= 1");
    if (sig < 1) throw HostError(TOR_E_INVALID, "precision/range", "need at least one significant digit");
    if (!(alpha > 0.0)) throw HostError(TOR_E_INVALID, "precision/range", "alpha must be positive");
    PrecCfg c;
    c.alpha = alpha;
    c.b_sgn = static_cast<int>(std::ceil(sig * std::log2(10.0)));
    c.b_accum = static_cast<int>(std::ceil(std::log2(alpha) + N + 2.0 * std::log2(N)));
    c.b_upper = upper_bits(a);
    double diag_sum = 0.0;
    for (int i = 0; i < a.n; ++i) diag_sum += a.a00_at(i, i).real();
    c.a_repr = diag_sum / a.n;
    const double det = det_i_minus_a_float(a);
    double k_fit = kCorrMax;
    if (c.a_repr > 0.0 && c.a_repr < 1.0) {
        const double one_minus_a = 1.0 - c.a_repr;
        const double fitted = (one_minus_a * one_minus_a - std::pow(det, 1.0 / N)) / N;
        if (std::isfinite(fitted)) k_fit = fitted;
    }
    c.k_corr = std::clamp(k_fit, kCorrMin, kCorrMax);
    c.b_lower = lower_bits(N, c.a_repr, c.k_corr);
    const int B = c.total_bits();
    if (B <= 128) c.width_bits = 128;
    else if (B <= 256) c.width_bits = 256;
    else
        throw HostError(TOR_E_PRECISION, "precision/unsupported",
                        "required bit budget exceeds 256 bits (B = " + std::to_string(B) + ")");
    c.frac_bits = static_cast<unsigned>(c.width_bits - 1 - c.b_upper);
    return c;
}

PrecCfg force_width(const Input& a, int width_bits) {  // precision.cpp:123-148
    if (width_bits != 128 && width_bits != 256)
        throw HostError(TOR_E_INVALID, "precision/range", "width must be 128 or 256");
    PrecCfg c;
    c.width_bits = width_bits;
    c.b_sgn = static_cast<int>(std::ceil(3 * std::log2(10.0)));
    c.b_upper = upper_bits(a);
    const int N = a.n;
    c.b_accum = static_cast<int>(std::ceil(std::log2(0.5) + N + 2.0 * std::log2(N)));
    double diag_sum = 0.0;
    for (int i = 0; i < N; ++i) diag_sum += a.a00_at(i, i).real();
    c.a_repr = diag_sum / N;
    c.k_corr = kCorrMax;
    const int f = width_bits - 1 - c.b_upper;
    if (f < 1)
        throw HostError(TOR_E_PRECISION, "precision/scaling",
                        "upper bound leaves no room for fraction bits at this width");
    c.frac_bits = static_cast<unsigned>(f);
    try {
        c.b_lower = lower_bits(N, c.a_repr, c.k_corr);
    } catch (const HostError&) {
        c.b_lower = 0;
    }
    return c;
}

// R = T (I - O) T^H, T = (1/sqrt2)[[I, I], [-iI, iI]] per mode, P = I - A00 (diagonal
// 1 - Re a_ii rounded to double exactly as extract_i_minus_az does,
// torontonian.cpp:58), Q = -A01:
//   R(x_i,x_j) = Re P + Re Q   R(x_i,p_j) = Im Q - Im P
//   R(p_i,x_j) = Im P + Im Q   R(p_i,p_j) = Re P - Re Q
// Each entry is the sum of two input doubles: exact as a DD (TwoSum), rounded once
// in fp64 mode.
std::vector<double> build_R(const Input& a, int words, bool grid, int* tscale_log2) {
    const int d = 2 * a.n;
    std::vector<double> R(static_cast<size_t>(d) * (d + 1) / 2 * words, 0.0);
    build_R_into(a, words, grid, R.data(), tscale_log2);
    return R;
}

void build_R_into(const Input& a, int words, bool grid, double* R, int* tscale_log2, bool stream) {
    // std::complex<double> arrays are layout-compatible with interleaved (re, im) doubles
    build_R_raw(a.n, reinterpret_cast<const double*>(a.a00.data()), reinterpret_cast<const double*>(a.a01.data()),
                words, grid, R, tscale_log2, stream);
}

namespace {
// Plain or non-temporal 8-byte store.  Pinned staging written with ordinary stores by many
// host threads stays dirty in their caches, and the GPU's DMA reads of it then run at ~5 GB/s
// instead of the link's ~50 GB/s (measured on the B200 boxes, tools/probes/h2d_probe.cu);
// streaming stores put the data in memory.  Callers fence (build_R_fence) before the copy.
template <bool kStream> inline void put_word(double* p, double v) {
#if defined(__x86_64__)
    if constexpr (kStream) {
        long long bits;
        std::memcpy(&bits, &v, sizeof(bits));
        _mm_stream_si64(reinterpret_cast<long long*>(p), bits);
        return;
    }
#endif
    *p = v;
}
template <bool kStream>
void build_R_impl(int n, const double* __restrict__ a00, const double* __restrict__ a01, int words, bool grid,
                  double* __restrict__ R, int* tscale_log2);
}  // namespace

void build_R_fence() {
#if defined(__x86_64__)
    _mm_sfence();
#endif
}

void build_R_raw(int n, const double* a00, const double* a01, int words, bool grid, double* R, int* tscale_log2,
                 bool stream) {
    if (stream) build_R_impl<true>(n, a00, a01, words, grid, R, tscale_log2);
    else build_R_impl<false>(n, a00, a01, words, grid, R, tscale_log2);
}

namespace {
template <bool kStream>
void build_R_impl(int n, const double* __restrict__ a00, const double* __restrict__ a01, int words, bool grid,
                  double* __restrict__ R, int* tscale_log2) {
    const int d = 2 * n;
    // entry (r, s), r <= s, of pair rows r = 2i + ri, s = 2j + sj: x + y with
    //   (x_i, x_j): Re P + Re Q   (x_i, p_j): Im Q - Im P   (p_i, x_j): Im P + Im Q   (p_i, p_j): Re P - Re Q
    // P = I - A00 (diagonal 1 - Re a_ii), Q = -A01, from the upper triangles (i <= j).
    // grid (fixed-exponent) DD states need max_k R_kk < 3.75 (arith.cuh); larger inputs are
    // scaled by an exact power of two, undone per term on the device (Acc::sc)
    int sc = 0;
    if (grid) {
        double dmax = 0.0;
        for (int i = 0; i < n; ++i) {
            const size_t t = static_cast<size_t>(i) * n - (static_cast<size_t>(i) * (i + 1)) / 2 + i;
            const double pre = 1.0 - a00[2 * t], qre = -a01[2 * t];
            dmax = std::max(dmax, std::max(std::fabs(pre + qre), std::fabs(pre + -qre)));
        }
        while (std::ldexp(dmax, -sc) >= 3.75) ++sc;
    }
    if (tscale_log2) *tscale_log2 = sc;
    const double f = std::ldexp(1.0, -sc);  // exact power of two
    auto put = [&](double* e, double x, double y) {
        if (grid) {
            const dd g = dd_to_grid(x * f, y * f);
            put_word<kStream>(e, g.hi);
            put_word<kStream>(e + 1, g.lo);
        } else {
            double hi, lo;
            two_sum(x, y, hi, lo);
            put_word<kStream>(e, hi);
            if (words >= 2) put_word<kStream>(e + 1, lo);
            for (int w = 2; w < words; ++w) put_word<kStream>(e + w, 0.0);
        }
    };
    // mode pair (i, j) fills two consecutive entries of pair rows 2i and 2i+1 (three entries for
    // i == j): both rows are written front to back
    size_t t = 0;  // packed index of (i, j) in the n x n upper triangles
    for (int i = 0; i < n; ++i) {
        const size_t r0 = 2 * static_cast<size_t>(i);
        double* row0 = R + static_cast<size_t>(words) * (r0 * d - (r0 * (r0 + 1)) / 2 + r0);
        double* row1 = row0 + static_cast<size_t>(words) * (d - r0);
        {
            const double pre = 1.0 - a00[2 * t], pim = 0.0;
            const double qre = -a01[2 * t], qim = -a01[2 * t + 1];
            put(row0, pre, qre);
            put(row0 + words, qim, -pim);
            put(row1, pre, -qre);
            row0 += 2 * words;
            row1 += words;
            ++t;
        }
        for (int j = i + 1; j < n; ++j, ++t, row0 += 2 * words, row1 += 2 * words) {
            const double pre = -a00[2 * t], pim = -a00[2 * t + 1];
            const double qre = -a01[2 * t], qim = -a01[2 * t + 1];
            put(row0, pre, qre);
            put(row0 + words, qim, -pim);
            put(row1, pim, qim);
            put(row1 + words, pre, -qre);
        }
    }
}

}  // namespace

unsigned __int128 total_op_count(int n) {  // flops.cpp:15-31 (Eq. 8)
    unsigned __int128 total = 0, binom = 1;
    for (int z = 1; z <= n; ++z) {
        binom = binom * (n - z + 1) / z;
        const unsigned __int128 dd_ = 2 * static_cast<unsigned __int128>(z);
        total += binom * ((4 * dd_ * dd_ * dd_ + 3 * dd_ * dd_ - 4 * dd_) / 3);
    }
    return total;
}

void op_counts(int n, uint64_t& mults, uint64_t& adds, uint64_t& recips, uint64_t& rsqrts) {
    // Per d x d elimination (linalg.cpp:7-61): for each pivot with r rows below it,
    // 1 det mult, r x (6 mults + 4 adds), and r(r-1)/2 x (4 mults + 4 adds).
    unsigned __int128 m = 0, ad = 0, rc = 0, binom = 1;
    for (int z = 1; z <= n; ++z) {
        binom = binom * (n - z + 1) / z;
        const int d = 2 * z;
        unsigned __int128 mz = 0, az = 0;
        for (int r = 0; r < d; ++r) {
            mz += 1 + 6 * static_cast<unsigned __int128>(r) + 2 * static_cast<unsigned __int128>(r) * (r > 0 ? r - 1 : 0);
            az += 4 * static_cast<unsigned __int128>(r) + 2 * static_cast<unsigned __int128>(r) * (r > 0 ? r - 1 : 0);
        }
        m += binom * mz;
        ad += binom * az;
        rc += binom * static_cast<unsigned __int128>(d - 1);
    }
    mults = static_cast<uint64_t>(m);
    adds = static_cast<uint64_t>(ad);
    recips = static_cast<uint64_t>(rc);
    rsqrts = (n >= 64) ? ~0ull : ((1ull << n) - 1);
}

Input extract_submatrix(const Input& full, uint64_t bits) {  // matrix_io.cpp:360-382
    std::vector<int> sel;
    for (int k = 0; k < full.n && k < 64; ++k)
        if (bits >> k & 1) sel.push_back(k);
    if (full.n < 64 && (bits >> full.n) != 0)
        throw HostError(TOR_E_INVALID, "matrixio/dim", "pattern mode count mismatch");
    return extract_modes(full, sel);
}

// Submatrix on an explicit ascending mode list: no 64-mode limit on the full state (the
// reference's ClickPattern is one u64, matrix_io.hpp:29-34).
Input extract_modes(const Input& full, const std::vector<int>& sel) {
    if (sel.empty()) throw HostError(TOR_E_INVALID, "matrixio/pattern", "empty click pattern");
    for (size_t k = 0; k < sel.size(); ++k)
        if (sel[k] < 0 || sel[k] >= full.n || (k > 0 && sel[k] <= sel[k - 1]))
            throw HostError(TOR_E_INVALID, "matrixio/pattern", "modes must be ascending and within the state");
    Input out;
    out.n = static_cast<int>(sel.size());
    const size_t t = static_cast<size_t>(out.n) * (out.n + 1) / 2;
    out.a00.resize(t);
    out.a01.resize(t);
    for (int i = 0; i < out.n; ++i)
        for (int j = i; j < out.n; ++j) {
            out.a00[tri(out.n, i, j)] = full.a00_at(sel[i], sel[j]);
            out.a01[tri(out.n, i, j)] = full.a01_at(sel[i], sel[j]);
        }
    return out;
}

}  // namespace tor
