// Torontonian engine: internal host-side interface of the sm_100a kernels.
//
// Replaces the reference's per-subset O(z^3) evaluation loop
//   torontonian_partial<W> (torontonian.cpp:72-103) -> extract_i_minus_az (:44-65)
//   -> hermitian_det_fixed (linalg.cpp:7-61) -> fp_rsqrt (fixed_point.cpp:110)
// and its thread fan-out run_engine<W> (torontonian.cpp:112-147) with a
// prefix-tree Schur-complement recursion on the real symmetric matrix
// R = T (I - O) T^H (pair order x_j, p_j), amortised O(1) work per subset.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace tor {

enum Mode : int { MODE_FP64 = 0, MODE_DD = 1, MODE_QD = 2 };

inline int mode_words(int mode) { return mode == MODE_FP64 ? 1 : (mode == MODE_DD ? 2 : 4); }

// One problem instance after host preparation: the exact R matrix in the mode's
// word format (packed upper triangle of the 2n x 2n matrix, pair order, `words`
// doubles per entry).
struct PreparedInput {
    int n = 0;
    std::vector<double> R;  // tri(2n) * words
    int tscale_log2 = 0;    // R was scaled by 2^-s: every term is multiplied back by 2^(-s|Z|)
};

// Work selection: prefix classes of the top `class_bits` reference-mask bits
// (bit N-1-j = mode j, subsets.hpp:11-13), classes [class_lo, class_hi).
// class_bits = 0 and [0,1) means the whole Torontonian.
struct WorkRange {
    int class_bits = 0;
    uint64_t class_lo = 0;
    uint64_t class_hi = 1;
    // one partial per class of the range (EngineOut::class_parts) instead of one folded
    // partial: each class is an aligned subtree of the fixed fold tree, so any split of the
    // classes across devices folds bit-identically on the host (fold_blocks)
    bool class_partials = false;
    // schedule (0 = default): prefix jobs of the whole problem (sets the prefix depth c and
    // so the producer DFS depth n - c - Q0; results stay within the mode's tolerance but are
    // bit-identical only between runs of equal prefix_jobs), subtree-kernel CTAs per SM
    uint64_t prefix_jobs = 0;
    int blocks_per_sm = 0;
};

// Per-instance outcome.
struct EngineOut {
    double words[4] = {0, 0, 0, 0};  // signed sum, multi-word (1/2/4 significant words)
    double sum_abs = 0.0;            // sum |term| (fp64)
    uint64_t terms = 0;
    bool breakdown = false;
    uint64_t bad_mask = 0;           // reference mask convention
    int bad_row = -1;                // pair-order pivot row (2k: x_k, 2k+1: p_k)
    std::vector<double> class_parts; // WorkRange::class_partials: 5 doubles per class
};

struct EngineStats {
    double kernel_ms = 0.0;       // subtree kernel (device time, CUDA events)
    double total_ms = 0.0;        // whole device pipeline incl. prefix + reduction
    uint64_t launches = 0;        // kernels launched
    int prefix_depth = 0;
    uint64_t jobs = 0;
    uint64_t h2d_bytes = 0;       // inputs uploaded when the plan was created
    uint64_t d2h_bytes = 0;       // results read back per execute()
};

// Prepared evaluation with device-resident inputs (see PlanImpl in engine.cu).
class Plan {
  public:
    virtual ~Plan() = default;
    virtual int execute(std::vector<EngineOut>& out, EngineStats* stats, std::string& err) = 0;  // launch + collect
    virtual int launch(std::string& err) = 0;  // enqueue the pipeline (asynchronous)
    virtual int collect(std::vector<EngineOut>& out, EngineStats* stats, std::string& err) = 0;  // wait + decode
    // new inputs for the same geometry: R of every instance (count x tri(2n) entries of the
    // mode's words), copied asynchronously on the plan's stream
    virtual int upload(const double* R, int tscale_log2, std::string& err) = 0;
    // the same in parts: upload_part for instance ranges (asynchronous, any order), then
    // upload_finish once
    virtual int upload_part(const double* R, int lo, int hi, std::string& err) = 0;
    virtual int upload_finish(int tscale_log2, std::string& err) = 0;
};

// A plan whose inputs are written by the caller into pinned host staging (build_R_into,
// any host threads), then uploaded and executed: the repeated-call path of the C ABI.  Idle
// staged plans are cached per (device, mode, n, count, range) -- device buffers, stream,
// events and pinned memory are reused across calls (release_device_cache frees them).
struct StagedPlan {
    int device = 0, mode = 0, n = 0, count = 0;
    WorkRange range;
    Plan* plan = nullptr;
    double* staging = nullptr;  // count x stride doubles (pinned)
    size_t stride = 0;          // tri(2n) * words
    ~StagedPlan();
};
int staged_acquire(int device, int mode, int n, int count, const WorkRange& range, StagedPlan** out,
                   std::string& err);
int staged_execute(StagedPlan* sp, int tscale_log2, std::vector<EngineOut>& out, EngineStats* stats,
                   std::string& err);
// chunked form: staged_upload_part for instance ranges of sp->staging as they are built,
// then staged_execute_uploaded (upload_finish + execute)
int staged_upload_part(StagedPlan* sp, int lo, int hi, std::string& err);
int staged_execute_uploaded(StagedPlan* sp, int tscale_log2, std::vector<EngineOut>& out, EngineStats* stats,
                            std::string& err);
// the same split so host work can overlap the device pipeline
int staged_launch(StagedPlan* sp, int tscale_log2, std::string& err);
int staged_collect(StagedPlan* sp, std::vector<EngineOut>& out, EngineStats* stats, std::string& err);
void staged_release(StagedPlan* sp);  // back to the cache (or freed)

int plan_create(int device, int mode, const std::vector<PreparedInput>& inputs, const WorkRange& range, Plan** out,
                std::string& err);

// Runs the engine on `device` for all instances (same n) over `range`.
// Returns 0 or a CUDA error code; errors are described in `err`.
int engine_run(int device, int mode, const std::vector<PreparedInput>& inputs, const WorkRange& range,
               std::vector<EngineOut>& out, EngineStats* stats, std::string& err);

// Fixed-order binary fold of per-shard partials (power-of-two aligned shards),
// identical to the device reduction tree so results are bit-identical for any
// shard count.  `parts` are `count` x 5 doubles (4 words + sum_abs).
void fold_words(int mode, const double* parts, int count, double* out5);

// Fold of partials over aligned power-of-two class blocks that tile [0, 2^class_bits):
// block i covers classes [lo[i], lo[i] + width[i]) (sorted, width a power of two,
// lo % width == 0).  Each block's partial is the fixed tree's subtree over its classes, so
// folding the blocks along the same tree is bit-identical to a single-device run.
// Returns false if the blocks do not tile the range that way.
bool fold_blocks(int mode, const double* parts, const uint64_t* lo, const uint64_t* width, int count,
                 int class_bits, double* out5);

// Exact fixed-point validation mode (fixed.cu): the reference's per-subset algorithm on
// the GPU; limbs4 receives the raw accumulator (identical to the reference's).
struct FixedStats {
    double device_ms = 0.0;
    uint64_t launches = 0;
    bool breakdown = false;
    uint64_t bad_mask = 0;
    int bad_row = -1;
};
int fixed_run(int device, int width_bits, int n, const double* a00, const double* a01, unsigned frac_bits,
              uint64_t* limbs4, FixedStats* stats, std::string& err);

// Minimum instance size handled by the tree kernel; smaller n uses the direct path.
int engine_tree_min_n(int mode);
void release_device_cache();  // frees the pooled device allocations of finished plans

}  // namespace tor
