// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI harness over the UNMODIFIED reference engine (torfp, C++20), compiled
// from the sources where they lie under /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libtorfp_ref.so.  Only tests/, bench.py's
// reference/cpu_baseline legs and the golden-fixture scripts load it.
//
// Every entry point forwards to a public reference symbol:
//   ref_torontonian            -> torfp::torontonian            (torontonian.cpp:151)
//   ref_torontonian_reference  -> torfp::torontonian_reference  (torontonian.cpp:179)
//   ref_select_precision       -> torfp::select_precision       (precision.cpp:80)
//   ref_force_width            -> torfp::force_width            (precision.cpp:123)
//   ref_det_i_minus_a_float    -> torfp::det_i_minus_a_float    (precision.cpp:34)
//   ref_check_symmetries       -> torfp::check_symmetries       (matrix_io.cpp:285)
//   ref_generate_instance      -> torfp::generate_instance      (matrix_io.cpp:307)
//   ref_slice                  -> per-mask templates extract_i_minus_az<W>,
//                                 hermitian_det_fixed<W>, fp_rsqrt<W>
//                                 (torontonian.hpp:36-38, linalg.hpp:67, fixed_point.hpp:178)
//                                 over the masks of prefix classes, i.e. exactly the
//                                 per-mask body of torontonian_partial (torontonian.cpp:83-96)
//   ref_save_matrix            -> torfp::save_matrix            (matrix_io.cpp:109)
//   ref_load_matrix            -> torfp::load_matrix_file       (matrix_io.cpp:253; the bytes
//                                 go through a temporary file so the reference's own format
//                                 sniffing is used)
//   ref_partial_sample         -> torfp::torontonian_partial<W> over partition(N, rank, P)
//                                 (torontonian.cpp:72, subsets.cpp:66), threaded; the
//                                 bounded CPU-baseline sample of bench.py
#include <atomic>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <string>
#include <unistd.h>
#include <thread>
#include <vector>

#include "torfp/flops.hpp"
#include "torfp/precision.hpp"
#include "torfp/subsets.hpp"
#include "torfp/torontonian.hpp"

using namespace torfp;

namespace {

struct ErrOut {
    char* code;
    int code_len;
    char* msg;
    int msg_len;
    std::uint64_t* mask;
    std::int64_t* row;
};

void put(char* dst, int len, const std::string& s) {
    if (!dst || len <= 0) return;
    std::strncpy(dst, s.c_str(), static_cast<std::size_t>(len - 1));
    dst[len - 1] = 0;
}

// 1 InvalidArgument, 2 Breakdown, 3 Precision, 4 Parse, 5 Resource, 7 other Error
int report(const ErrOut& e) {
    try {
        throw;
    } catch (const BreakdownError& x) {
        put(e.code, e.code_len, x.code());
        put(e.msg, e.msg_len, x.what());
        if (e.mask) *e.mask = x.subset_mask();
        if (e.row) *e.row = x.pivot_row() == SIZE_MAX ? -1 : static_cast<std::int64_t>(x.pivot_row());
        return 2;
    } catch (const InvalidArgument& x) {
        put(e.code, e.code_len, x.code());
        put(e.msg, e.msg_len, x.what());
        return 1;
    } catch (const PrecisionError& x) {
        put(e.code, e.code_len, x.code());
        put(e.msg, e.msg_len, x.what());
        return 3;
    } catch (const ParseError& x) {
        put(e.code, e.code_len, x.code());
        put(e.msg, e.msg_len, x.what());
        if (e.row) *e.row = static_cast<std::int64_t>(x.position());
        return 4;
    } catch (const ResourceError& x) {
        put(e.code, e.code_len, x.code());
        put(e.msg, e.msg_len, x.what());
        return 5;
    } catch (const Error& x) {
        put(e.code, e.code_len, x.code());
        put(e.msg, e.msg_len, x.what());
        return 7;
    } catch (const std::exception& x) {
        put(e.code, e.code_len, "harness/std");
        put(e.msg, e.msg_len, x.what());
        return 8;
    }
}

// a00/a01: n(n+1)/2 complex entries each, interleaved (re, im), row-major upper triangle.
InputMatrix make_input(int n, const double* a00, const double* a01) {
    InputMatrix m;
    m.n_modes = n;
    const std::size_t tri = static_cast<std::size_t>(n) * (n + 1) / 2;
    m.a00.resize(tri);
    m.a01.resize(tri);
    for (std::size_t i = 0; i < tri; ++i) {
        m.a00[i] = {a00[2 * i], a00[2 * i + 1]};
        m.a01[i] = {a01[2 * i], a01[2 * i + 1]};
    }
    return m;
}

void cfg_out(const PrecisionConfig& c, int* ints, double* dbls) {
    if (ints) {
        ints[0] = c.width_bits;
        ints[1] = static_cast<int>(c.frac_bits);
        ints[2] = c.b_lower;
        ints[3] = c.b_upper;
        ints[4] = c.b_sgn;
        ints[5] = c.b_accum;
    }
    if (dbls) {
        dbls[0] = c.a_repr;
        dbls[1] = c.k_corr;
        dbls[2] = c.alpha;
    }
}

template <int W> void limbs_out(const Wide<W>& a, std::uint64_t* limbs) {
    for (int i = 0; i < 4; ++i) limbs[i] = i < W ? a.w[static_cast<std::size_t>(i)] : 0;
}

// Per-mask body of torontonian_partial (torontonian.cpp:83-96) over all masks whose
// top `k` bits equal `cls` (bit N-1-j = mode j, subsets.hpp:11-13).  The empty set is
// included for class 0, as rank 0 does (torontonian.cpp:98-101).  Exact modular
// accumulation, so the limbs equal torontonian_partial over the same masks.
template <int W>
Wide<W> class_sum(const InputMatrix& a, unsigned f, int k, std::uint64_t cls, double* sum_abs) {
    const int N = a.n_modes;
    const int r = N - k;
    HermitianFixed<W> scratch;
    OpCounters ops;
    Wide<W> acc{};
    double sabs = 0.0;
    const std::uint64_t base = cls << r;
    const std::uint64_t count = std::uint64_t(1) << r;
    for (std::uint64_t low = 0; low < count; ++low) {
        const SubsetMask mask = base | low;
        const int z = std::popcount(mask);
        if (z == 0) {
            const Wide<W> one = fp_one<W>(f);
            acc = (N & 1) ? fp_sub(acc, one) : fp_add(acc, one);
            sabs += 1.0;
            continue;
        }
        extract_i_minus_az<W>(a, mask, f, scratch);
        Wide<W> root;
        try {
            const Wide<W> det = hermitian_det_fixed<W>(scratch, f, ops);
            root = fp_rsqrt<W>(det, f);
        } catch (BreakdownError& e) {
            e.set_subset_mask(mask);
            throw;
        }
        sabs += std::fabs(fp_to_real<W>(root, f));
        acc = ((N - z) & 1) ? fp_sub(acc, root) : fp_add(acc, root);
    }
    if (sum_abs) *sum_abs = sabs;
    return acc;
}

template <int W>
int slice_impl(const InputMatrix& a, unsigned f, int k, std::uint64_t lo, std::uint64_t hi,
               int threads, std::uint64_t* class_limbs, double* class_sum_abs,
               std::uint64_t* total_limbs, const ErrOut& e) {
    const std::uint64_t ncls = hi - lo;
    std::vector<Wide<W>> part(ncls);
    std::vector<double> sabs(ncls, 0.0);
    std::vector<std::exception_ptr> errs(static_cast<std::size_t>(threads));
    std::atomic<std::uint64_t> next{0};
    auto work = [&](int t) {
        try {
            for (;;) {
                const std::uint64_t i = next.fetch_add(1);
                if (i >= ncls) break;
                part[i] = class_sum<W>(a, f, k, lo + i, &sabs[i]);
            }
        } catch (...) {
            errs[static_cast<std::size_t>(t)] = std::current_exception();
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (auto& ep : errs)
        if (ep) {
            try {
                std::rethrow_exception(ep);
            } catch (...) {
                return report(e);
            }
        }
    Wide<W> tot{};
    for (std::uint64_t i = 0; i < ncls; ++i) {
        tot = fp_add(tot, part[i]);
        if (class_limbs) limbs_out<W>(part[i], class_limbs + 4 * i);
        if (class_sum_abs) class_sum_abs[i] = sabs[i];
    }
    if (total_limbs) limbs_out<W>(tot, total_limbs);
    return 0;
}

template <int W>
int sample_impl(const InputMatrix& a, const PrecisionConfig& cfg, int nproc, int rank_lo,
                int nranks, int threads, std::uint64_t* masks_done, double* seconds,
                const ErrOut& e) {
    std::vector<std::exception_ptr> errs(static_cast<std::size_t>(threads));
    std::vector<std::uint64_t> done(static_cast<std::size_t>(threads), 0);
    std::atomic<int> next{0};
    volatile std::uint64_t sink = 0;
    auto work = [&](int t) {
        try {
            for (;;) {
                const int i = next.fetch_add(1);
                if (i >= nranks) break;
                const WorkAssignment w = partition(a.n_modes, rank_lo + i, nproc);
                OpCounters ops;
                const Wide<W> v = torontonian_partial<W>(a, w, cfg, ops);
                sink = sink + v.w[0];
                done[static_cast<std::size_t>(t)] += ops.rsqrts;
            }
        } catch (...) {
            errs[static_cast<std::size_t>(t)] = std::current_exception();
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (auto& ep : errs)
        if (ep) {
            try {
                std::rethrow_exception(ep);
            } catch (...) {
                return report(e);
            }
        }
    std::uint64_t tot = 0;
    for (auto d : done) tot += d;
    *masks_done = tot;
    *seconds = dt;
    return 0;
}

} // namespace

#define ERR_ARGS char *code, int code_len, char *msg, int msg_len, std::uint64_t *err_mask, std::int64_t *err_row
#define ERR_INIT ErrOut e{code, code_len, msg, msg_len, err_mask, err_row}

extern "C" {

// precision: 0 Auto, 1 Bits128, 2 Bits256.  ints6/dbls3: config (see cfg_out).
// counters4: mults, adds, recips, rsqrts.
int ref_torontonian(int n, const double* a00, const double* a01, int precision, int workers,
                    double* value, std::uint64_t* limbs4, int* width_bits, int* cfg_ints6,
                    double* cfg_dbls3, std::uint64_t* counters4, std::uint64_t* term_count,
                    double* wall, int* workers_out, ERR_ARGS) {
    ERR_INIT;
    try {
        const InputMatrix m = make_input(n, a00, a01);
        const PrecisionChoice pc = precision == 1   ? PrecisionChoice::Bits128
                                   : precision == 2 ? PrecisionChoice::Bits256
                                                    : PrecisionChoice::Auto;
        const TorontonianResult r = torontonian(m, pc, workers);
        *value = r.value;
        for (int i = 0; i < 4; ++i) limbs4[i] = r.raw.limbs[static_cast<std::size_t>(i)];
        *width_bits = r.raw.width_bits;
        cfg_out(r.config, cfg_ints6, cfg_dbls3);
        counters4[0] = r.counters.mults;
        counters4[1] = r.counters.adds;
        counters4[2] = r.counters.recips;
        counters4[3] = r.counters.rsqrts;
        *term_count = r.term_count;
        *wall = r.wall_seconds;
        *workers_out = r.workers;
        return 0;
    } catch (...) {
        return report(e);
    }
}

int ref_torontonian_reference(int n, const double* a00, const double* a01, double* value,
                              ERR_ARGS) {
    ERR_INIT;
    try {
        *value = torontonian_reference(make_input(n, a00, a01));
        return 0;
    } catch (...) {
        return report(e);
    }
}

int ref_select_precision(int n, const double* a00, const double* a01, int N, int sig,
                         double alpha, int* ints6, double* dbls3, ERR_ARGS) {
    ERR_INIT;
    try {
        cfg_out(select_precision(make_input(n, a00, a01), N, sig, alpha), ints6, dbls3);
        return 0;
    } catch (...) {
        return report(e);
    }
}

int ref_force_width(int n, const double* a00, const double* a01, int width, int* ints6,
                    double* dbls3, ERR_ARGS) {
    ERR_INIT;
    try {
        cfg_out(force_width(make_input(n, a00, a01), width), ints6, dbls3);
        return 0;
    } catch (...) {
        return report(e);
    }
}

int ref_det_i_minus_a_float(int n, const double* a00, const double* a01, double* det,
                            ERR_ARGS) {
    ERR_INIT;
    try {
        *det = det_i_minus_a_float(make_input(n, a00, a01));
        return 0;
    } catch (...) {
        return report(e);
    }
}

// devs3: hermitian_dev, a01_sym_dev, block_conj_dev; returns pass in *pass.
int ref_check_symmetries(int n, const double* a00, const double* a01, double* devs3, int* pass,
                         ERR_ARGS) {
    ERR_INIT;
    try {
        const InputMatrix m = make_input(n, a00, a01);
        const auto r = check_symmetries(to_dense(m), 2 * n);
        devs3[0] = r.hermitian_dev;
        devs3[1] = r.a01_sym_dev;
        devs3[2] = r.block_conj_dev;
        *pass = r.pass ? 1 : 0;
        return 0;
    } catch (...) {
        return report(e);
    }
}

// Dense 2n x 2n complex (interleaved) -> symmetry check (bindings.cpp:26-47 from_dense gate).
int ref_check_dense(int two_n, const double* dense, double* devs3, int* pass, ERR_ARGS) {
    ERR_INIT;
    try {
        std::vector<std::complex<double>> d(static_cast<std::size_t>(two_n) * two_n);
        for (std::size_t i = 0; i < d.size(); ++i) d[i] = {dense[2 * i], dense[2 * i + 1]};
        const auto r = check_symmetries(d, two_n);
        devs3[0] = r.hermitian_dev;
        devs3[1] = r.a01_sym_dev;
        devs3[2] = r.block_conj_dev;
        *pass = r.pass ? 1 : 0;
        return 0;
    } catch (...) {
        return report(e);
    }
}

int ref_generate_instance(int n, double a_target, double spread, std::uint64_t seed,
                          double* a00_out, double* a01_out, ERR_ARGS) {
    ERR_INIT;
    try {
        const InputMatrix m = generate_instance(n, a_target, spread, seed);
        for (std::size_t i = 0; i < m.a00.size(); ++i) {
            a00_out[2 * i] = m.a00[i].real();
            a00_out[2 * i + 1] = m.a00[i].imag();
            a01_out[2 * i] = m.a01[i].real();
            a01_out[2 * i + 1] = m.a01[i].imag();
        }
        return 0;
    } catch (...) {
        return report(e);
    }
}

// Raw fixed-point sums over prefix classes [lo, hi) of the top k mask bits at width
// (128|256) and scaling frac_bits.  class_limbs: (hi-lo) x 4 u64 (may be null);
// class_sum_abs: (hi-lo) doubles of sum |term| (may be null); total_limbs: 4 u64.
int ref_slice(int n, const double* a00, const double* a01, int width, int frac_bits, int k,
              std::uint64_t lo, std::uint64_t hi, int threads, std::uint64_t* class_limbs,
              double* class_sum_abs, std::uint64_t* total_limbs, ERR_ARGS) {
    ERR_INIT;
    try {
        const InputMatrix m = make_input(n, a00, a01);
        if (k < 0 || k > n || hi < lo || hi > (std::uint64_t(1) << k))
            throw InvalidArgument("harness/range", "bad slice");
        if (threads < 1) threads = 1;
        if (width == 128)
            return slice_impl<2>(m, static_cast<unsigned>(frac_bits), k, lo, hi, threads,
                                 class_limbs, class_sum_abs, total_limbs, e);
        return slice_impl<4>(m, static_cast<unsigned>(frac_bits), k, lo, hi, threads,
                             class_limbs, class_sum_abs, total_limbs, e);
    } catch (...) {
        return report(e);
    }
}

// Timed bounded sample: torontonian_partial<W> for ranks [rank_lo, rank_lo+nranks) of
// partition(N, ., nproc) on `threads` threads.  precision: 1 Bits128, 2 Bits256 (force_width).
int ref_partial_sample(int n, const double* a00, const double* a01, int precision, int nproc,
                       int rank_lo, int nranks, int threads, std::uint64_t* masks_done,
                       double* seconds, ERR_ARGS) {
    ERR_INIT;
    try {
        const InputMatrix m = make_input(n, a00, a01);
        const PrecisionConfig cfg = force_width(m, precision == 2 ? 256 : 128);
        if (threads < 1) threads = 1;
        if (cfg.width_bits == 128)
            return sample_impl<2>(m, cfg, nproc, rank_lo, nranks, threads, masks_done, seconds, e);
        return sample_impl<4>(m, cfg, nproc, rank_lo, nranks, threads, masks_done, seconds, e);
    } catch (...) {
        return report(e);
    }
}

// Timed fp64 oracle (torontonian_reference, single thread by design).
int ref_reference_timed(int n, const double* a00, const double* a01, double* value,
                        double* seconds, ERR_ARGS) {
    ERR_INIT;
    try {
        const InputMatrix m = make_input(n, a00, a01);
        const auto t0 = std::chrono::steady_clock::now();
        *value = torontonian_reference(m);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return 0;
    } catch (...) {
        return report(e);
    }
}

int ref_total_op_count(int n, std::uint64_t* lo, std::uint64_t* hi, ERR_ARGS) {
    ERR_INIT;
    try {
        const unsigned __int128 v = total_op_count(n);
        *lo = static_cast<std::uint64_t>(v);
        *hi = static_cast<std::uint64_t>(v >> 64);
        return 0;
    } catch (...) {
        return report(e);
    }
}

// binary: 0 text, 1 binary (bits 16/32).  *len = full size; copies min(len, cap) bytes.
int ref_save_matrix(int n, const double* a00, const double* a01, int binary, int bits, unsigned char* buf,
                    std::size_t cap, std::size_t* len, ERR_ARGS) {
    ERR_INIT;
    try {
        const InputMatrix m = make_input(n, a00, a01);
        const auto b = save_matrix(m, binary ? MatrixFormat::Binary : MatrixFormat::Text, bits);
        *len = b.size();
        if (buf) std::memcpy(buf, b.data(), std::min(cap, b.size()));
        return 0;
    } catch (...) {
        return report(e);
    }
}

// bytes -> load_matrix_file (format sniffed by the reference); triangles copied when
// cap >= n(n+1)/2 entries.
int ref_load_matrix(const unsigned char* bytes, std::size_t len, int* n, int* bits, double* a00, double* a01,
                    std::size_t cap, ERR_ARGS) {
    ERR_INIT;
    char path[] = "/tmp/ref_gbsa_XXXXXX";
    const int fd = mkstemp(path);
    if (fd < 0) {
        put(code, code_len, "harness/tmp");
        return 8;
    }
    if (len && write(fd, bytes, len) != static_cast<ssize_t>(len)) {
        close(fd);
        unlink(path);
        put(code, code_len, "harness/tmp");
        return 8;
    }
    close(fd);
    try {
        const InputMatrix m = load_matrix_file(path);
        unlink(path);
        *n = m.n_modes;
        *bits = m.quant_bits;
        if (a00 && a01 && cap >= m.a00.size()) {
            for (std::size_t i = 0; i < m.a00.size(); ++i) {
                a00[2 * i] = m.a00[i].real();
                a00[2 * i + 1] = m.a00[i].imag();
                a01[2 * i] = m.a01[i].real();
                a01[2 * i + 1] = m.a01[i].imag();
            }
        }
        return 0;
    } catch (...) {
        unlink(path);
        return report(e);
    }
}

} // extern "C"
