// C ABI of the B200 Torontonian engine (include/tor_capi.h).  Validation, precision
// selection and the adaptive driver run on the host; every evaluation runs on the
// GPU through engine_run().  There is no CPU fallback: without a CUDA device the
// evaluation entry points fail with TOR_E_DEVICE.
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <algorithm>
#include <atomic>
#include <exception>
#include <thread>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/tor_capi.h"
#include "arith.cuh"
#include "engine.cuh"
#include "host.hpp"

using namespace tor;

namespace {

void set_err(tor_error* e, const char* code, const std::string& msg, int64_t row = -1, uint64_t mask = 0) {
    if (!e) return;
    std::memset(e, 0, sizeof(*e));
    std::strncpy(e->code, code, sizeof(e->code) - 1);
    std::strncpy(e->message, msg.c_str(), sizeof(e->message) - 1);
    e->pivot_row = row;
    e->subset_mask = mask;
}

int fail(tor_error* e, const HostError& h) {
    set_err(e, h.code.c_str(), h.what(), h.pivot_row, h.subset_mask);
    return h.status;
}

void clear_err(tor_error* e) {
    if (e) set_err(e, "", "");
}

// One host thread per index (a thread per device); the first failure in index order is
// rethrown.
template <class F>
void parallel_for_n(int n, F f) {
    std::vector<std::exception_ptr> errs(n);
    std::vector<std::thread> th;
    for (int t = 0; t < n; ++t)
        th.emplace_back([&, t] {
            try {
                f(t);
            } catch (...) {
                errs[t] = std::current_exception();
            }
        });
    for (auto& x : th) x.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

// Persistent host worker threads for the per-instance preparation of batches (spawning
// threads per call cost more than the work at config-3 sizes).
class HostPool {
  public:
    static HostPool& get() {
        static HostPool p;
        return p;
    }
    int size() const { return static_cast<int>(workers_.size()) + 1; }
    // runs job(t) for t in [0, nt) on the workers and the calling thread
    void run(int nt, const std::function<void(int)>& job) {
        std::unique_lock<std::mutex> call(call_mu_);  // one batch at a time
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &job;
            next_ = 1;
            total_ = nt;
            done_ = 0;
            ++gen_;
        }
        cv_.notify_all();
        job(0);
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {  // the caller helps with remaining tasks
            if (next_ < total_) {
                const int t = next_++;
                lk.unlock();
                job(t);
                lk.lock();
                ++done_;
                continue;
            }
            if (done_ == total_ - 1) break;
            done_cv_.wait(lk);
        }
        job_ = nullptr;
    }

  private:
    HostPool() {
        const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
        for (int i = 1; i < std::min(hw, 64); ++i) workers_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    void loop() {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {
            cv_.wait(lk, [&] { return stop_ || (gen_ != seen && job_ && next_ < total_); });
            if (stop_) return;
            seen = gen_;
            while (job_ && next_ < total_) {
                const int t = next_++;
                const auto* job = job_;
                lk.unlock();
                (*job)(t);
                lk.lock();
                if (++done_ == total_ - 1) done_cv_.notify_all();
            }
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* job_ = nullptr;
    int next_ = 0, total_ = 0, done_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// Host-side preparation of many instances (validation, precision bounds, exact R) in
// parallel chunks; the first failure in index order is rethrown (deterministic).
template <class F>
void parallel_for(int n, F f, int grain = 64) {
    HostPool& pool = HostPool::get();
    const int nt = std::min(pool.size(), std::max(1, n / grain));
    if (nt <= 1) {
        for (int i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::exception_ptr> errs(nt);
    pool.run(nt, [&](int t) {
        const int lo = static_cast<int>(static_cast<int64_t>(n) * t / nt);
        const int hi = static_cast<int>(static_cast<int64_t>(n) * (t + 1) / nt);
        try {
            for (int i = lo; i < hi; ++i) f(i);
        } catch (...) {
            errs[t] = std::current_exception();
        }
    });
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

// The reference's torontonian() takes N <= 40 (torontonian.cpp:153-154) and so does
// tor_torontonian; prefix-class slices / shards / plans go to N = 50 (the paper's 100x100
// case: checkpointable class ranges across devices and calls).
constexpr int kMaxSliceModes = 50;

// The reference's input validation (torontonian.cpp:151-157) on the raw tor_input: range,
// finite entries, then the symmetry gate (check_symmetries_tri: == the dense check).
void validate_raw(const tor_input* in, int nmax) {
    if (!in || in->n < 1 || in->n > nmax || !in->a00_upper || !in->a01_upper)
        throw HostError(TOR_E_INVALID, "torontonian/range",
                        nmax == 20   ? "reference path supports 1 <= N <= 20"
                        : nmax == 40 ? "engine supports 1 <= N <= 40"
                                     : "slices and shards support 1 <= N <= 50");
    const size_t t2 = static_cast<size_t>(in->n) * (in->n + 1);  // doubles per triangle
    for (const double* v : {in->a00_upper, in->a01_upper})
        for (size_t k = 0; k < t2; ++k)
            if (!std::isfinite(v[k])) throw HostError(TOR_E_INVALID, "torontonian/domain", "input entries must be finite");
    double hdev = 0.0;
    for (int i = 0; i < in->n; ++i) {
        const size_t t = static_cast<size_t>(i) * in->n - (static_cast<size_t>(i) * (i + 1)) / 2 + i;
        const std::complex<double> v{in->a00_upper[2 * t], in->a00_upper[2 * t + 1]};
        hdev = std::max(hdev, std::abs(v - std::conj(v)));
    }
    if (!(hdev <= 1e-12)) throw HostError(TOR_E_ERROR, "torontonian/symmetry", "input violates the block symmetries");
}

Input checked_input(const tor_input* in, int nmax) {
    validate_raw(in, nmax);
    return make_input(in->n, in->a00_upper, in->a01_upper);
}

void put_cfg(const PrecCfg& c, tor_precision_config* o) {
    o->width_bits = c.width_bits;
    o->frac_bits = c.frac_bits;
    o->b_lower = c.b_lower;
    o->b_upper = c.b_upper;
    o->b_sgn = c.b_sgn;
    o->b_accum = c.b_accum;
    o->a_repr = c.a_repr;
    o->k_corr = c.k_corr;
    o->alpha = c.alpha;
}

int mode_of(tor_precision p) {
    return p == TOR_PREC_FP64 ? MODE_FP64 : (p == TOR_PREC_W256_QD ? MODE_QD : MODE_DD);
}
int width_of(int mode) { return mode == MODE_FP64 ? 64 : (mode == MODE_DD ? 128 : 256); }
double mantissa_bits(int mode) { return mode == MODE_FP64 ? 52.0 : (mode == MODE_DD ? 104.0 : 208.0); }

double words_value(const double* w) { return ((w[3] + w[2]) + w[1]) + w[0]; }

// FixedValue limbs of a multi-word value: round(sum(words) * 2^frac_bits) (ties toward +inf)
// as width_bits two's complement, low limb first -- the reference's raw accumulator
// format (torontonian.hpp:14-29) at its own scaling.  Exact: the words are summed in a
// 2176-bit integer at scale 2^1100 (every finite double is an integer multiple of 2^-1074).
void requantise(const double* words, int nwords, int width_bits, unsigned frac_bits, uint64_t* limbs4) {
    for (int i = 0; i < 4; ++i) limbs4[i] = 0;
    if (width_bits != 128 && width_bits != 256) return;
    constexpr int kL = 34, kScale = 1100;
    uint64_t acc[kL] = {};
    auto add_shifted = [&](uint64_t m, int sh, bool neg) {  // acc += (neg ? -1 : 1) * m * 2^sh
        uint64_t t[kL] = {};
        const int li = sh / 64, bi = sh % 64;
        if (li < kL) t[li] = m << bi;
        if (bi && li + 1 < kL) t[li + 1] = m >> (64 - bi);
        if (neg) {  // two's complement of t
            uint64_t c = 1;
            for (int i = 0; i < kL; ++i) {
                const uint64_t v = ~t[i] + c;
                c = (c && v == 0) ? 1 : 0;
                t[i] = v;
            }
        }
        unsigned __int128 c = 0;
        for (int i = 0; i < kL; ++i) {
            c += static_cast<unsigned __int128>(acc[i]) + t[i];
            acc[i] = static_cast<uint64_t>(c);
            c >>= 64;
        }
    };
    for (int k = 0; k < nwords; ++k) {
        const double w = words[k];
        if (w == 0.0 || !std::isfinite(w)) continue;
        int e = 0;
        const double fr = std::frexp(std::fabs(w), &e);           // |w| = fr * 2^e, fr in [0.5, 1)
        const uint64_t m = static_cast<uint64_t>(std::ldexp(fr, 53));  // |w| = m * 2^(e-53), exact
        const int sh = e - 53 + kScale;
        if (sh < 0) continue;  // below 2^-1100: cannot occur for finite doubles
        add_shifted(m, sh, w < 0);
    }
    // + 2^(kScale - f - 1), then arithmetic shift right by kScale - f
    const int rs = kScale - static_cast<int>(frac_bits);
    if (rs <= 0 || rs > 64 * (kL - 4)) return;
    add_shifted(1, rs - 1, false);
    for (int i = 0; i < 4; ++i) {
        const int bit = rs + 64 * i, li = bit / 64, bi = bit % 64;
        uint64_t v = li < kL ? acc[li] >> bi : ~0ull;
        if (bi && li + 1 < kL) v |= acc[li + 1] << (64 - bi);
        limbs4[i] = i < width_bits / 64 ? v : 0;
    }
}

// Tor(0) = 0 exactly (every term is +-1): the only input whose zero sum is exempt from the
// posterior cancellation check.
bool zero_input(const Input& a) {
    for (const auto* v : {&a.a00, &a.a01})
        for (const auto& x : *v)
            if (x.real() != 0.0 || x.imag() != 0.0) return false;
    return true;
}

// AUTO's posterior check (precision.cpp:80-121 sizes the width a priori; the budget's
// lower bound is blind on pure states, a_repr = 0): at least b_sgn significant bits must
// survive the cancellation sum|t| / |Tor| after the growth allowance.
bool posterior_ok(const Input& a, const tor_result& r, const PrecCfg& cfg) {
    return zero_input(a) || r.bits_left >= cfg.b_sgn;
}

void device_check(int device) {
    int cnt = 0;
    const cudaError_t e = cudaGetDeviceCount(&cnt);
    if (e != cudaSuccess || cnt == 0)
        throw HostError(TOR_E_DEVICE, "device/unavailable",
                        std::string("no CUDA device: ") + (e == cudaSuccess ? "count 0" : cudaGetErrorString(e)));
    if (device < 0 || device >= cnt) throw HostError(TOR_E_INVALID, "device/range", "device index out of range");
}

// One asynchronous engine evaluation of `ins` over `range`: the constructor takes a cached
// plan for the shape (device buffers, stream, pinned staging), has the host threads build the
// exact R of every instance straight into the pinned staging block by block -- each block's
// host->device copy is enqueued as soon as it is built, overlapping the building -- and
// launches the device pipeline; wait() collects the results and maps failures onto the
// error taxonomy.  Host work placed between the two overlaps the device.
class DeviceRun {
  public:
    DeviceRun(int device, int mode, const std::vector<Input>& ins, const WorkRange& range)
        : DeviceRun(device, mode, ins[0].n, static_cast<int>(ins.size()), range,
                    [&](int i, double* R, int* tsc) { build_R_into(ins[i], mode_words(mode), mode == MODE_DD, R, tsc, true); }) {}

    // build(i, R, tsc) writes instance i's exact R (and may throw a validation error: the
    // first failing instance in index order is reported, before anything is launched)
    DeviceRun(int device, int mode, int n, int count, const WorkRange& range,
              const std::function<void(int, double*, int*)>& build) {
        const auto t0 = std::chrono::steady_clock::now();
        device_check(device);
        std::string err;
        if (staged_acquire(device, mode, n, count, range, &sp_, err) != 0)
            throw HostError(TOR_E_DEVICE, "device/cuda", err);
        const auto t_acq = std::chrono::steady_clock::now();
        std::vector<int> tsc(count, 0);
        // about two build blocks per host thread; their host->device copies go out in a few
        // large groups (a copy costs ~45 us before its first byte: 32 copies of 0.5 MB ran at
        // 14 GB/s, 4 copies of 4 MB at the link's ~48 GB/s), each enqueued by the worker that
        // completes the group's last block -- so copying still overlaps building
        const int kBlock = std::max(64, (count + 2 * HostPool::get().size() - 1) / (2 * HostPool::get().size()));
        const int nblocks = (count + kBlock - 1) / kBlock;
        const int ngroups = std::min(nblocks, 4);
        std::vector<int> gfirst(ngroups + 1);
        for (int g = 0; g <= ngroups; ++g) gfirst[g] = static_cast<int>(static_cast<int64_t>(nblocks) * g / ngroups);
        std::vector<std::atomic<int>> gleft(ngroups);
        for (int g = 0; g < ngroups; ++g) gleft[g].store(gfirst[g + 1] - gfirst[g]);
        std::vector<int> gst(ngroups, 0);
        std::vector<std::string> gerr(ngroups);
        std::vector<std::exception_ptr> bex(nblocks);
        parallel_for(
            nblocks,
            [&](int b) {
                const int lo = b * kBlock, hi = std::min(count, lo + kBlock);
                try {
                    for (int i = lo; i < hi; ++i) build(i, sp_->staging + i * sp_->stride, &tsc[i]);
                    build_R_fence();  // the builders' streaming stores before the group's copy
                } catch (...) {
                    bex[b] = std::current_exception();
                    return;  // the group's copy is never enqueued: the run fails below
                }
                const int g = static_cast<int>(std::upper_bound(gfirst.begin(), gfirst.end(), b) - gfirst.begin()) - 1;
                if (gleft[g].fetch_sub(1) == 1)
                    gst[g] = staged_upload_part(sp_, gfirst[g] * kBlock, std::min(count, gfirst[g + 1] * kBlock), gerr[g]);
            },
            1);
        const auto t_built = std::chrono::steady_clock::now();
        for (auto& e : bex)
            if (e) {
                staged_release(sp_);  // the pinned staging stays valid for copies in flight
                sp_ = nullptr;
                std::rethrow_exception(e);
            }
        int st = 0;
        for (int g = 0; g < ngroups && st == 0; ++g)
            if (gst[g]) {
                st = gst[g];
                err = gerr[g];
            }
        if (st == 0) st = staged_launch(sp_, *std::max_element(tsc.begin(), tsc.end()), err);
        if (st != 0) fail_and_release(err);
        launched_ = true;
        if (std::getenv("TOR_DEBUG_TIMING"))
            std::fprintf(stderr, "[tor] run: acquire %.2f ms, build+copies enqueued %.2f ms, prepare+launch %.2f ms\n",
                         std::chrono::duration<double, std::milli>(t_acq - t0).count(),
                         std::chrono::duration<double, std::milli>(t_built - t0).count(),
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    DeviceRun(const DeviceRun&) = delete;
    DeviceRun& operator=(const DeviceRun&) = delete;
    ~DeviceRun() {
        if (sp_) {  // never waited (an exception in between): finish the device work first
            std::vector<EngineOut> drop;
            std::string err;
            if (launched_) staged_collect(sp_, drop, nullptr, err);
            staged_release(sp_);
        }
    }

    std::vector<EngineOut> wait(EngineStats* stats, bool check_breakdown = true) {
        std::vector<EngineOut> out;
        std::string err;
        const int st = staged_collect(sp_, out, stats, err);
        staged_release(sp_);
        sp_ = nullptr;
        if (st != 0) throw HostError(TOR_E_DEVICE, "device/cuda", err);
        for (const auto& o : out)
            if (check_breakdown && o.breakdown) {
                HostError h(TOR_E_BREAKDOWN, "linalg/breakdown", "non-positive pivot in elimination");
                h.pivot_row = o.bad_row;
                h.subset_mask = o.bad_mask;
                throw h;
            }
        return out;
    }

  private:
    [[noreturn]] void fail_and_release(const std::string& err) {
        staged_release(sp_);
        sp_ = nullptr;
        throw HostError(TOR_E_DEVICE, "device/cuda", err);
    }
    StagedPlan* sp_ = nullptr;
    bool launched_ = false;
};

// Runs the engine synchronously.
std::vector<EngineOut> run(int device, int mode, const std::vector<Input>& ins, const WorkRange& range,
                           EngineStats* stats, bool check_breakdown = true) {
    DeviceRun r(device, mode, ins, range);
    return r.wait(stats, check_breakdown);
}

// op_counts depends on N only (closed forms with 128-bit binomials): computed once per N
void op_counts_cached(int n, uint64_t& mults, uint64_t& adds, uint64_t& recips, uint64_t& rsqrts) {
    struct Row {
        std::atomic<bool> ready{false};
        uint64_t v[4];
    };
    static Row rows[65];
    static std::mutex mu;
    if (n < 0 || n > 64) return op_counts(n, mults, adds, recips, rsqrts);
    Row& r = rows[n];
    if (!r.ready.load(std::memory_order_acquire)) {
        std::lock_guard<std::mutex> lk(mu);
        if (!r.ready.load(std::memory_order_relaxed)) {
            op_counts(n, r.v[0], r.v[1], r.v[2], r.v[3]);
            r.ready.store(true, std::memory_order_release);
        }
    }
    mults = r.v[0];
    adds = r.v[1];
    recips = r.v[2];
    rsqrts = r.v[3];
}

void fill_result(int n, int mode, const PrecCfg& cfg, const EngineOut& o, const EngineStats& st,
                 double wall, int ndev, tor_result* r) {
    std::memset(r, 0, sizeof(*r));
    r->mode = mode == MODE_FP64 ? TOR_PREC_FP64 : (mode == MODE_DD ? TOR_PREC_W128_DD : TOR_PREC_W256_QD);
    r->width_bits = width_of(mode);
    r->nwords = mode_words(mode);
    for (int i = 0; i < 4; ++i) r->words[i] = o.words[i];
    r->value = words_value(o.words);
    put_cfg(cfg, &r->config);
    r->term_count = o.terms;
    op_counts_cached(n, r->mults, r->adds, r->recips, r->rsqrts);
    r->wall_seconds = wall;
    r->device_ms = st.total_ms;
    r->kernel_ms = st.kernel_ms;
    r->devices = ndev;
    r->sum_abs_terms = o.sum_abs;
    const double av = std::fabs(r->value);
    r->cancellation_bits = av > 0 ? std::log2(o.sum_abs / av) : std::numeric_limits<double>::infinity();
    // error growth allowance: log2(n) + 4 bits over the working precision
    r->bits_left = mantissa_bits(mode) - r->cancellation_bits - (std::log2(static_cast<double>(n)) + 4.0);
    r->kernel_launches = st.launches;
    r->h2d_bytes = st.h2d_bytes;
    r->d2h_bytes = st.d2h_bytes;
    if (mode != MODE_FP64) requantise(o.words, mode_words(mode), r->width_bits, cfg.frac_bits, r->raw_limbs);
}

// One Torontonian on several devices of this process (the reference's `workers` fan-out,
// torontonian.cpp:112-147): the 2^kShardBits top-level prefix classes are split into P
// contiguous ranges (P = the device count, any P <= 2^kShardBits; ranges differ by at most
// one class), one host thread per device; each device returns one partial per class (an
// aligned subtree of the engine's fixed fold tree) and the host folds all classes along the
// same tree -- bit-identical to a single-device run.  Instances too small to have
// kShardBits prefix levels run on the first device.
constexpr int kShardBits = 6;
EngineOut run_devices(const std::vector<int>& devs, int mode, const Input& a, EngineStats* stats, int* used) {
    const int ncls = 1 << kShardBits;
    int P = std::min(static_cast<int>(devs.size()), ncls);
    if (a.n < engine_tree_min_n(mode) + kShardBits) P = 1;
    if (used) *used = P;
    if (P == 1) return run(devs[0], mode, {a}, WorkRange{}, stats)[0];
    std::vector<EngineOut> parts(P);
    std::vector<EngineStats> sts(P);
    parallel_for_n(P, [&](int r) {
        WorkRange wr;
        wr.class_bits = kShardBits;
        wr.class_lo = static_cast<uint64_t>(ncls) * r / P;
        wr.class_hi = static_cast<uint64_t>(ncls) * (r + 1) / P;
        wr.class_partials = true;
        parts[r] = run(devs[r], mode, {a}, wr, &sts[r])[0];
    });
    std::vector<double> buf;
    EngineOut o;
    for (int r = 0; r < P; ++r) {
        buf.insert(buf.end(), parts[r].class_parts.begin(), parts[r].class_parts.end());
        o.terms += parts[r].terms;
    }
    if (buf.size() != static_cast<size_t>(ncls) * 5) throw HostError(TOR_E_DEVICE, "device/cuda", "missing class partials");
    double w5[5];
    fold_words(mode, buf.data(), ncls, w5);
    for (int x = 0; x < 4; ++x) o.words[x] = w5[x];
    o.sum_abs = w5[4];
    if (stats) {
        *stats = EngineStats{};
        for (const auto& t : sts) {  // the slowest device bounds the call
            stats->kernel_ms = std::max(stats->kernel_ms, t.kernel_ms);
            stats->total_ms = std::max(stats->total_ms, t.total_ms);
            stats->launches += t.launches;
            stats->h2d_bytes += t.h2d_bytes;
            stats->d2h_bytes += t.d2h_bytes;
        }
    }
    return o;
}

// Exact fixed-point validation mode: the reference's algorithm on the GPU (fixed.cu).
void fixed_mode(const Input& a, int width, int dev, tor_result* r) {
    if (a.n > 24) throw HostError(TOR_E_INVALID, "torontonian/range", "fixed-point validation mode supports N <= 24");
    device_check(dev);
    const PrecCfg cfg = force_width(a, width);
    std::vector<double> w00(a.a00.size() * 2), w01(a.a01.size() * 2);
    for (size_t i = 0; i < a.a00.size(); ++i) {
        w00[2 * i] = a.a00[i].real();
        w00[2 * i + 1] = a.a00[i].imag();
        w01[2 * i] = a.a01[i].real();
        w01[2 * i + 1] = a.a01[i].imag();
    }
    uint64_t limbs[4] = {0, 0, 0, 0};
    FixedStats fs;
    std::string e;
    if (fixed_run(dev, width, a.n, w00.data(), w01.data(), cfg.frac_bits, limbs, &fs, e) != 0)
        throw HostError(TOR_E_DEVICE, "device/cuda", e);
    if (fs.breakdown) {
        HostError h(TOR_E_BREAKDOWN, "linalg/breakdown", "non-positive pivot in elimination");
        h.pivot_row = fs.bad_row == 0xff ? -1 : fs.bad_row;
        h.subset_mask = fs.bad_mask;
        throw h;
    }
    std::memset(r, 0, sizeof(*r));
    r->mode = width == 128 ? TOR_PREC_FIXED128 : TOR_PREC_FIXED256;
    r->width_bits = width;
    r->nwords = 1;
    // fp_to_real (fixed_point.cpp:152-162): long-double accumulation of the magnitude
    const int W = width / 64;
    const bool neg = (limbs[W - 1] >> 63) != 0;
    uint64_t mag[4] = {0, 0, 0, 0};
    if (neg) {
        uint64_t br = 0;
        for (int i = 0; i < W; ++i) {
            const uint64_t d = 0 - limbs[i];
            const uint64_t nb = limbs[i] != 0;
            mag[i] = d - br;
            br = nb | (d < br);
        }
    } else {
        for (int i = 0; i < W; ++i) mag[i] = limbs[i];
    }
    long double acc = 0.0L;
    for (int i = W - 1; i >= 0; --i) acc = std::ldexp(acc, 64) + static_cast<long double>(mag[i]);
    const double v = static_cast<double>(std::ldexp(acc, -static_cast<int>(cfg.frac_bits)));
    r->value = neg ? -v : v;
    r->words[0] = r->value;
    for (int i = 0; i < 4; ++i) r->raw_limbs[i] = limbs[i];
    put_cfg(cfg, &r->config);
    r->term_count = a.n >= 64 ? ~0ull : (1ull << a.n);
    op_counts(a.n, r->mults, r->adds, r->recips, r->rsqrts);
    r->device_ms = fs.device_ms;
    r->kernel_ms = fs.device_ms;
    r->devices = 1;
    r->kernel_launches = fs.launches;
    r->sum_abs_terms = std::nan("");
    r->cancellation_bits = std::nan("");
    r->bits_left = std::nan("");
    r->h2d_bytes = 2 * w00.size() * sizeof(double);
    r->d2h_bytes = W * 8 + 8;
}

}  // namespace

struct tor_plan {
    Input in;
    int mode = MODE_DD;
    PrecCfg cfg;
    Plan* plan = nullptr;
    ~tor_plan() { delete plan; }
};

extern "C" {

int tor_abi_version(void) { return TOR_ABI_VERSION; }

int tor_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}

void tor_release_device_cache(void) { release_device_cache(); }

int tor_check_symmetries(const tor_input* in, double devs[3], int* pass, tor_error* err) {
    try {
        clear_err(err);
        if (!in || in->n < 1) throw HostError(TOR_E_INVALID, "matrixio/dim", "matrix has no modes");
        const Input a = make_input(in->n, in->a00_upper, in->a01_upper);
        const SymReport s = check_symmetries(to_dense(a), 2 * a.n);
        devs[0] = s.hermitian_dev;
        devs[1] = s.a01_sym_dev;
        devs[2] = s.block_conj_dev;
        *pass = s.pass ? 1 : 0;
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_check_dense(int two_n, const double* dense, double devs[3], int* pass, tor_error* err) {
    try {
        clear_err(err);
        if (two_n < 2 || !dense) throw HostError(TOR_E_INVALID, "matrixio/dim", "dense matrix must be 2N x 2N");
        std::vector<std::complex<double>> d(static_cast<size_t>(two_n) * two_n);
        for (size_t i = 0; i < d.size(); ++i) d[i] = {dense[2 * i], dense[2 * i + 1]};
        const SymReport s = check_symmetries(d, two_n);
        devs[0] = s.hermitian_dev;
        devs[1] = s.a01_sym_dev;
        devs[2] = s.block_conj_dev;
        *pass = s.pass ? 1 : 0;
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_det_i_minus_a(const tor_input* in, double* det, tor_error* err) {
    try {
        clear_err(err);
        if (!in || in->n < 1) throw HostError(TOR_E_INVALID, "matrixio/dim", "matrix has no modes");
        *det = det_i_minus_a_float(make_input(in->n, in->a00_upper, in->a01_upper));
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_select_precision(const tor_input* in, int N, int sig, double alpha, tor_precision_config* out,
                         tor_error* err) {
    try {
        clear_err(err);
        if (!in || in->n < 1) throw HostError(TOR_E_INVALID, "precision/range", "N must be >= 1");
        put_cfg(select_precision(make_input(in->n, in->a00_upper, in->a01_upper), N, sig, alpha), out);
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_force_width(const tor_input* in, int width_bits, tor_precision_config* out, tor_error* err) {
    try {
        clear_err(err);
        if (!in || in->n < 1) throw HostError(TOR_E_INVALID, "precision/range", "N must be >= 1");
        put_cfg(force_width(make_input(in->n, in->a00_upper, in->a01_upper), width_bits), out);
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_torontonian(const tor_input* in, tor_precision prec, const int* devices, int ndev, tor_result* out,
                    tor_error* err) {
    try {
        clear_err(err);
        const auto t0 = std::chrono::steady_clock::now();
        const Input a = checked_input(in, 40);
        if (prec < TOR_PREC_AUTO || prec > TOR_PREC_FIXED256)
            throw HostError(TOR_E_INVALID, "precision/range", "unknown precision mode");
        std::vector<int> devs;
        if (devices && ndev > 0) devs.assign(devices, devices + ndev);
        else devs.push_back(0);
        const int dev = devs[0];
        if (prec == TOR_PREC_FIXED128 || prec == TOR_PREC_FIXED256) {
            fixed_mode(a, prec == TOR_PREC_FIXED128 ? 128 : 256, dev, out);
            out->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            return TOR_OK;
        }
        PrecCfg cfg;
        int mode;
        if (prec == TOR_PREC_AUTO) {
            cfg = select_precision(a, a.n, 3, 0.5);
            mode = cfg.width_bits == 128 ? MODE_DD : MODE_QD;
        } else if (prec == TOR_PREC_FP64) {
            cfg = force_width(a, 128);
            cfg.width_bits = 64;
            mode = MODE_FP64;
        } else {
            cfg = force_width(a, prec == TOR_PREC_W128_DD ? 128 : 256);
            mode = mode_of(prec);
        }
        EngineStats st;
        int used = 1;
        std::vector<EngineOut> res{run_devices(devs, mode, a, &st, &used)};
        int escalated = 0;
        if (prec == TOR_PREC_AUTO) {
            // posterior check: keep >= b_sgn significant bits after cancellation
            tor_result tmp;
            fill_result(a.n, mode, cfg, res[0], st, 0.0, 1, &tmp);
            if (!posterior_ok(a, tmp, cfg)) {
                if (mode == MODE_DD) {
                    mode = MODE_QD;
                    escalated = 1;
                    res = {run_devices(devs, mode, a, &st, &used)};
                    fill_result(a.n, mode, cfg, res[0], st, 0.0, 1, &tmp);
                }
                if (!posterior_ok(a, tmp, cfg))
                    throw HostError(TOR_E_PRECISION, "precision/insufficient",
                                    "cancellation leaves fewer than b_sgn significant bits");
            }
        }
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        fill_result(a.n, mode, cfg, res[0], st, wall, used, out);
        out->escalated = escalated;
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_torontonian_reference(const tor_input* in, double* value, tor_error* err) {
    try {
        clear_err(err);
        const Input a = checked_input(in, 20);
        EngineStats st;
        // torontonian_reference (torontonian.cpp:179-200) has no pivot check: a breakdown
        // surfaces as a non-finite sum (the Cholesky pivots of an indefinite block are NaN)
        const auto res = run(0, MODE_FP64, {a}, WorkRange{}, &st, /*check_breakdown=*/false);
        const double v = words_value(res[0].words);
        if (!std::isfinite(v))
            throw HostError(TOR_E_PRECISION, "torontonian/nonfinite", "non-finite term in reference summation");
        *value = v;
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_torontonian_batch(const tor_input* ins, int count, tor_precision prec, int device, tor_result* outs,
                          tor_error* err) {
    try {
        clear_err(err);
        if (count < 1 || !ins) throw HostError(TOR_E_INVALID, "torontonian/range", "empty batch");
        if (prec < TOR_PREC_AUTO || prec > TOR_PREC_FP64)
            throw HostError(TOR_E_INVALID, "precision/range", "batch supports auto, 128, 256 and fp64");
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<Input> as(count);
        const int mode = prec == TOR_PREC_AUTO ? MODE_DD : mode_of(prec);
        std::vector<PrecCfg> cfgs(count);
        // explicit widths: the per-instance force_width (a float determinant each) only feeds
        // the reported config, so it runs on the host threads while the device pipeline runs
        auto precision_of = [&](int i) {
            if (prec == TOR_PREC_AUTO) {
                cfgs[i] = select_precision(as[i], as[i].n, 3, 0.5);
            } else if (prec == TOR_PREC_FP64) {
                cfgs[i] = PrecCfg{};
                cfgs[i].width_bits = 64;
            } else {
                cfgs[i] = force_width(as[i], prec == TOR_PREC_W128_DD ? 128 : 256);
            }
        };
        auto shape_check = [&](int i) {
            validate_raw(&ins[i], 40);
            if (ins[i].n != ins[0].n) throw HostError(TOR_E_INVALID, "torontonian/range", "batch instances must share N");
        };
        // validation (the first bad instance in index order) before any device compute: AUTO in
        // a pass of its own (it also selects the widths); explicit widths inside the blocks that
        // build R (DeviceRun reports the first failing block's first failing instance and
        // launches nothing) -- unless there is no usable device, whose error must not hide a
        // validation error
        if (prec == TOR_PREC_AUTO) {
            parallel_for(count, [&](int i) {
                shape_check(i);
                as[i] = make_input(ins[i].n, ins[i].a00_upper, ins[i].a01_upper);
                precision_of(i);
            });
        } else {
            shape_check(0);
            try {
                device_check(device);
            } catch (const HostError&) {
                parallel_for(count, shape_check);
                throw;
            }
        }
        const auto t1 = std::chrono::steady_clock::now();
        EngineStats st;
        std::vector<int> modes(count, mode);
        std::vector<EngineOut> res(count);
        if (prec != TOR_PREC_AUTO) {
            // the exact R straight from the caller's arrays (no copies), validated block by block
            DeviceRun dr(device, mode, ins[0].n, count, WorkRange{}, [&](int i, double* R, int* tsc) {
                shape_check(i);
                build_R_raw(ins[i].n, ins[i].a00_upper, ins[i].a01_upper, mode_words(mode), mode == MODE_DD, R, tsc,
                            true);
            });
            if (prec != TOR_PREC_FP64)
                parallel_for(count, [&](int i) {
                    as[i] = make_input(ins[i].n, ins[i].a00_upper, ins[i].a01_upper);
                    precision_of(i);
                });
            else
                parallel_for(count, precision_of);
            res = dr.wait(&st);
        } else {
            // AUTO per instance, as tor_torontonian: the selected width picks DD or QD (one
            // sub-batch each), then the posterior check re-runs in QD every DD instance whose
            // cancellation leaves fewer than b_sgn bits
            auto run_group = [&](int md, const std::vector<int>& idx) {
                if (idx.empty()) return;
                std::vector<Input> sub;
                sub.reserve(idx.size());
                for (int i : idx) sub.push_back(as[i]);
                EngineStats gs;
                const auto r = run(device, md, sub, WorkRange{}, &gs);
                st.kernel_ms += gs.kernel_ms;
                st.total_ms += gs.total_ms;
                st.launches += gs.launches;
                st.h2d_bytes += gs.h2d_bytes;
                st.d2h_bytes += gs.d2h_bytes;
                for (size_t k = 0; k < idx.size(); ++k) {
                    res[idx[k]] = r[k];
                    modes[idx[k]] = md;
                }
            };
            std::vector<int> dd_idx, qd_idx;
            for (int i = 0; i < count; ++i) (cfgs[i].width_bits == 128 ? dd_idx : qd_idx).push_back(i);
            run_group(MODE_DD, dd_idx);
            run_group(MODE_QD, qd_idx);
            std::vector<int> esc;
            for (int i : dd_idx) {
                tor_result tmp;
                fill_result(as[i].n, MODE_DD, cfgs[i], res[i], st, 0.0, 1, &tmp);
                if (!posterior_ok(as[i], tmp, cfgs[i])) esc.push_back(i);
            }
            run_group(MODE_QD, esc);
            // every QD result (selected a priori or escalated) passes the same check as
            // tor_torontonian; the first failing instance in index order is reported
            std::vector<int> qd_all(qd_idx);
            qd_all.insert(qd_all.end(), esc.begin(), esc.end());
            std::sort(qd_all.begin(), qd_all.end());
            for (int i : qd_all) {
                tor_result tmp;
                fill_result(as[i].n, MODE_QD, cfgs[i], res[i], st, 0.0, 1, &tmp);
                if (!posterior_ok(as[i], tmp, cfgs[i]))
                    throw HostError(TOR_E_PRECISION, "precision/insufficient",
                                    "instance " + std::to_string(i) +
                                        ": cancellation leaves fewer than b_sgn significant bits");
            }
            for (int i : esc) modes[i] = -modes[i] - 1;  // mark escalated (decoded below)
        }
        const auto t2 = std::chrono::steady_clock::now();
        const double wall = std::chrono::duration<double>(t2 - t0).count();
        parallel_for(count, [&](int i) {
            const bool escalated = modes[i] < 0;
            const int md = escalated ? -modes[i] - 1 : modes[i];
            fill_result(ins[0].n, md, cfgs[i], res[i], st, wall, 1, &outs[i]);
            outs[i].escalated = escalated ? 1 : 0;
        });
        if (std::getenv("TOR_DEBUG_TIMING")) {
            auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            std::fprintf(stderr, "[tor] batch: validate+precision %.2f ms, run %.2f ms, results %.2f ms\n",
                         ms(t0, t1), ms(t1, t2), ms(t2, std::chrono::steady_clock::now()));
        }
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

namespace {
// explicit evaluation modes of slices, shards, class partials and plans
int explicit_mode(tor_precision prec, const char* what) {
    if (prec != TOR_PREC_W128_DD && prec != TOR_PREC_W256_QD && prec != TOR_PREC_FP64)
        throw HostError(TOR_E_INVALID, "precision/range", std::string(what) + " needs prec 128, 256 or fp64");
    return mode_of(prec);
}

WorkRange class_range(const Input& a, int class_bits, uint64_t class_lo, uint64_t class_hi) {
    if (class_bits < 0 || class_bits > a.n || class_bits > 62 || class_hi <= class_lo ||
        class_hi > (1ull << class_bits))
        throw HostError(TOR_E_INVALID, "torontonian/slice", "bad class range");
    WorkRange wr;
    wr.class_bits = class_bits;
    wr.class_lo = class_lo;
    wr.class_hi = class_hi;
    return wr;
}

void put_partial(tor_precision prec, const WorkRange& wr, const double* w5, uint64_t terms, tor_partial* out) {
    std::memset(out, 0, sizeof(*out));
    out->mode = prec;
    out->class_bits = wr.class_bits;
    out->class_lo = wr.class_lo;
    out->class_hi = wr.class_hi;
    for (int i = 0; i < 4; ++i) out->words[i] = w5[i];
    out->sum_abs = w5[4];
    out->term_count = terms;
}
}  // namespace

int tor_torontonian_slice(const tor_input* in, tor_precision prec, int class_bits, uint64_t class_lo,
                          uint64_t class_hi, int device, tor_partial* out, tor_error* err) {
    try {
        clear_err(err);
        const Input a = checked_input(in, kMaxSliceModes);
        const int mode = explicit_mode(prec, "slice");
        const WorkRange wr = class_range(a, class_bits, class_lo, class_hi);
        EngineStats st;
        const auto res = run(device, mode, {a}, wr, &st);
        double w5[5] = {res[0].words[0], res[0].words[1], res[0].words[2], res[0].words[3], res[0].sum_abs};
        put_partial(prec, wr, w5, res[0].terms, out);
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_torontonian_classes(const tor_input* in, tor_precision prec, int class_bits, uint64_t class_lo,
                            uint64_t class_hi, int device, const tor_schedule* sched, tor_partial* outs,
                            tor_error* err) {
    try {
        clear_err(err);
        const Input a = checked_input(in, kMaxSliceModes);
        const int mode = explicit_mode(prec, "class partials");
        WorkRange wr = class_range(a, class_bits, class_lo, class_hi);
        if (!outs) throw HostError(TOR_E_INVALID, "torontonian/slice", "null output array");
        if (class_hi - class_lo > (1ull << 24))
            throw HostError(TOR_E_INVALID, "torontonian/slice", "at most 2^24 class partials per call");
        wr.class_partials = true;
        if (sched) {
            wr.prefix_jobs = sched->prefix_jobs;
            wr.blocks_per_sm = sched->blocks_per_sm;
        }
        EngineStats st;
        const auto res = run(device, mode, {a}, wr, &st);
        const uint64_t ncls = class_hi - class_lo;
        if (res[0].class_parts.size() != ncls * 5) throw HostError(TOR_E_DEVICE, "device/cuda", "class partials lost");
        const uint64_t per = res[0].terms / ncls;
        for (uint64_t c = 0; c < ncls; ++c) {
            WorkRange one = wr;
            one.class_lo = class_lo + c;
            one.class_hi = class_lo + c + 1;
            put_partial(prec, one, &res[0].class_parts[5 * c], per, &outs[c]);
        }
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_torontonian_shard(const tor_input* in, tor_precision prec, int rank, int world, int device,
                          tor_partial* out, tor_error* err) {
    if (world < 1 || (world & (world - 1)) || rank < 0 || rank >= world) {
        set_err(err, "torontonian/shard", "world must be a power of two and 0 <= rank < world");
        return TOR_E_INVALID;
    }
    int k = 0;
    while ((1 << k) < world) ++k;
    if (prec == TOR_PREC_AUTO) {
        tor_precision_config c;
        const int st = tor_select_precision(in, in ? in->n : 0, 3, 0.5, &c, err);
        if (st) return st;
        prec = c.width_bits == 128 ? TOR_PREC_W128_DD : TOR_PREC_W256_QD;
    }
    return tor_torontonian_slice(in, prec, k, static_cast<uint64_t>(rank), static_cast<uint64_t>(rank) + 1, device,
                                 out, err);
}

int tor_fold_partials(const tor_partial* parts, int count, const tor_input* in, tor_result* out, tor_error* err) {
    try {
        clear_err(err);
        if (count < 1 || !parts) throw HostError(TOR_E_INVALID, "torontonian/shard", "no partials");
        const Input a = checked_input(in, kMaxSliceModes);
        const tor_precision prec = static_cast<tor_precision>(parts[0].mode);
        const int mode = explicit_mode(prec, "fold");
        const int k = parts[0].class_bits;
        if (k < 0 || k > a.n || k > 62) throw HostError(TOR_E_INVALID, "torontonian/shard", "bad class bits");
        std::vector<double> buf(static_cast<size_t>(count) * 5);
        std::vector<uint64_t> lo(count), wd(count);
        uint64_t terms = 0;
        for (int i = 0; i < count; ++i) {
            const tor_partial& p = parts[i];
            if (p.mode != parts[0].mode || p.class_bits != k)
                throw HostError(TOR_E_INVALID, "torontonian/shard", "partials of mixed modes or class bits");
            if (p.class_hi <= p.class_lo || (i > 0 && p.class_lo != parts[i - 1].class_hi))
                throw HostError(TOR_E_INVALID, "torontonian/shard", "partials must be contiguous and sorted");
            for (int x = 0; x < 4; ++x) buf[i * 5 + x] = p.words[x];
            buf[i * 5 + 4] = p.sum_abs;
            lo[i] = p.class_lo;
            wd[i] = p.class_hi - p.class_lo;
            terms += p.term_count;
        }
        if (parts[0].class_lo != 0 || parts[count - 1].class_hi != (1ull << k))
            throw HostError(TOR_E_INVALID, "torontonian/shard", "partials must cover every class (a missing rank?)");
        if (a.n < 64 && terms != (1ull << a.n))
            throw HostError(TOR_E_INVALID, "torontonian/shard", "partial term counts do not add up to 2^N");
        double w5[5];
        if (!fold_blocks(mode, buf.data(), lo.data(), wd.data(), count, k, w5))
            throw HostError(TOR_E_INVALID, "torontonian/shard",
                            "every partial must span an aligned power-of-two class range");
        EngineOut o;
        for (int x = 0; x < 4; ++x) o.words[x] = w5[x];
        o.sum_abs = w5[4];
        o.terms = terms;
        PrecCfg cfg = (mode == MODE_FP64) ? PrecCfg{} : force_width(a, mode == MODE_DD ? 128 : 256);
        if (mode == MODE_FP64) cfg.width_bits = 64;
        EngineStats st;
        fill_result(a.n, mode, cfg, o, st, 0.0, count, out);
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_plan_create(const tor_input* in, tor_precision prec, int class_bits, uint64_t class_lo, uint64_t class_hi,
                    int device, tor_plan** out, tor_error* err) {
    try {
        clear_err(err);
        *out = nullptr;
        const Input a = checked_input(in, kMaxSliceModes);
        const int mode = explicit_mode(prec, "plan");
        const WorkRange wr = class_range(a, class_bits, class_lo, class_hi);
        device_check(device);
        auto* p = new tor_plan();
        p->in = a;
        p->mode = mode;
        if (p->mode == MODE_FP64) p->cfg.width_bits = 64;
        else p->cfg = force_width(a, p->mode == MODE_DD ? 128 : 256);
        PreparedInput pi;
        pi.n = a.n;
        pi.R = build_R(a, mode_words(p->mode), p->mode == MODE_DD, &pi.tscale_log2);
        std::string e;
        if (plan_create(device, p->mode, {pi}, wr, &p->plan, e) != 0) {
            delete p;
            throw HostError(TOR_E_DEVICE, "device/cuda", e);
        }
        *out = p;
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_plan_execute(tor_plan* plan, tor_result* out, tor_error* err) {
    try {
        clear_err(err);
        if (!plan || !plan->plan) throw HostError(TOR_E_INVALID, "torontonian/plan", "null plan");
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<EngineOut> res;
        EngineStats st;
        std::string e;
        if (plan->plan->execute(res, &st, e) != 0) throw HostError(TOR_E_DEVICE, "device/cuda", e);
        if (res[0].breakdown) {
            HostError h(TOR_E_BREAKDOWN, "linalg/breakdown", "non-positive pivot in elimination");
            h.pivot_row = res[0].bad_row;
            h.subset_mask = res[0].bad_mask;
            throw h;
        }
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        st.h2d_bytes = 0;  // inputs are resident
        fill_result(plan->in.n, plan->mode, plan->cfg, res[0], st, wall, 1, out);
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

void tor_plan_destroy(tor_plan* plan) { delete plan; }

namespace {
int probability_of(const tor_input* full, const std::vector<int>* modes, uint64_t pattern_bits,
                   tor_precision prec, int device, double* p, tor_error* err) {
    if (!full || full->n < 1) throw HostError(TOR_E_INVALID, "matrixio/dim", "matrix has no modes");
    const Input a = make_input(full->n, full->a00_upper, full->a01_upper);
    const double det = det_i_minus_a_float(a);  // torontonian.cpp:203
    if (!(det > 0.0)) throw HostError(TOR_E_ERROR, "torontonian/invalid-state", "det(I - A) must be positive");
    if (modes ? modes->empty() : pattern_bits == 0) {
        *p = std::sqrt(det);
        return TOR_OK;
    }
    const Input sub = modes ? extract_modes(a, *modes) : extract_submatrix(a, pattern_bits);
    std::vector<double> w00(sub.a00.size() * 2), w01(sub.a01.size() * 2);
    for (size_t i = 0; i < sub.a00.size(); ++i) {
        w00[2 * i] = sub.a00[i].real();
        w00[2 * i + 1] = sub.a00[i].imag();
        w01[2 * i] = sub.a01[i].real();
        w01[2 * i + 1] = sub.a01[i].imag();
    }
    const tor_input si{sub.n, w00.data(), w01.data()};
    tor_result r;
    const int st = tor_torontonian(&si, prec, &device, 1, &r, err);
    if (st) return st;
    *p = r.value * std::sqrt(det);
    return TOR_OK;
}
}  // namespace

int tor_probability(const tor_input* full, uint64_t pattern_bits, tor_precision prec, int device, double* p,
                    tor_error* err) {
    try {
        clear_err(err);
        return probability_of(full, nullptr, pattern_bits, prec, device, p, err);
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_probability_modes(const tor_input* full, const int* modes, int nmodes, tor_precision prec, int device,
                          double* p, tor_error* err) {
    try {
        clear_err(err);
        if (nmodes < 0 || (nmodes > 0 && !modes)) throw HostError(TOR_E_INVALID, "matrixio/pattern", "bad mode list");
        const std::vector<int> sel(modes, modes + nmodes);
        return probability_of(full, &sel, 0, prec, device, p, err);
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_load_matrix(const void* bytes, size_t len, int* n, int* quant_bits, double* a00_upper, double* a01_upper,
                    size_t capacity, tor_error* err) {
    try {
        clear_err(err);
        if (!bytes && len) throw HostError(TOR_E_INVALID, "matrixio/io", "null buffer");
        if (!n) throw HostError(TOR_E_INVALID, "matrixio/io", "null output");
        int qb = 0;
        const Input a = load_gbsa(static_cast<const uint8_t*>(bytes), len, &qb);
        *n = a.n;
        if (quant_bits) *quant_bits = qb;
        if (a00_upper && a01_upper) {
            if (capacity < a.a00.size())
                throw HostError(TOR_E_INVALID, "matrixio/dim", "output triangles smaller than N(N+1)/2 entries");
            for (size_t i = 0; i < a.a00.size(); ++i) {
                a00_upper[2 * i] = a.a00[i].real();
                a00_upper[2 * i + 1] = a.a00[i].imag();
                a01_upper[2 * i] = a.a01[i].real();
                a01_upper[2 * i + 1] = a.a01[i].imag();
            }
        }
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

int tor_save_matrix(const tor_input* in, int format, int quant_bits, void* buf, size_t capacity, size_t* len,
                    tor_error* err) {
    try {
        clear_err(err);
        if (!in || in->n < 1 || !in->a00_upper || !in->a01_upper)
            throw HostError(TOR_E_INVALID, "matrixio/dim", "matrix has no modes");
        if (format != 0 && format != 1) throw HostError(TOR_E_INVALID, "matrixio/format", "format: 0 text, 1 binary");
        const std::string s = save_gbsa(make_input(in->n, in->a00_upper, in->a01_upper), format == 1, quant_bits);
        if (len) *len = s.size();
        if (buf) std::memcpy(buf, s.data(), std::min(capacity, s.size()));
        return TOR_OK;
    } catch (const HostError& h) {
        return fail(err, h);
    }
}

}  // extern "C"
