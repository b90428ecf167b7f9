// mlsk_internal.h -- host-side plumbing shared by the engines and the C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "mlsk_device.cuh"

namespace mlsk {

// Internal failures travel as exceptions and are mapped to the C-ABI status
// codes at the boundary (mlsk_api.cu).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void invalid(const std::string& m) { throw Error(MLSK_EINVAL, m); }

// Negative control of the parity harness (the reference's `oracle
// --inject-rescale-bug`, mlsketch_main.cpp:219-221, perturbs the rescale by
// 1 + 1e-6): a build with -DMLSK_INJECT_RESCALE_BUG=1 scales every level-sample
// rescale n / c by that factor, and the fp64 parity tests must then fail
// (tests/test_gpu_negative_control.py).  Never set in the product build.
#ifndef MLSK_INJECT_RESCALE_BUG
#define MLSK_INJECT_RESCALE_BUG 0
#endif
constexpr double kRescalePerturb = MLSK_INJECT_RESCALE_BUG ? 1.0 + 1e-6 : 1.0;

#define MLSK_CUDA(x)                                                                      \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess)                                                            \
            throw ::mlsk::Error(MLSK_ERUNTIME, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Kernel launches made by the calling thread (mlsk_kernel_launch_count).
extern thread_local int64_t g_launches;
// K-columns executed by the panel engines' GEMMs / sampled indices they stand
// for (mlsk_contraction_columns)
extern thread_local int64_t g_columns[2];
inline void launched(int n = 1) {
    g_launches += n;
    MLSK_CUDA(cudaGetLastError());
}

// Optional per-kernel timing with CUDA events on the launching stream
// (mlsk_profile_*); used by bench.py for the roofline's kernel duration.
struct Prof {
    const char* name;
    cudaStream_t stream;
    cudaEvent_t e0 = nullptr;
    Prof(const char* n, cudaStream_t s);
    ~Prof();
};

// Owning device allocation.  alloc_on() uses the stream-ordered allocator
// (pooled, no implicit device synchronisation on free) for per-call objects;
// alloc() is a plain cudaMalloc for long-lived workspaces.
void configure_mempool();  // retain pooled memory across calls (mlsk_model.cu)

template <class T>
struct DevArray {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    bool pooled = false;
    DevArray() = default;
    explicit DevArray(size_t count) { alloc(count); }
    DevArray(const DevArray&) = delete;
    DevArray& operator=(const DevArray&) = delete;
    DevArray(DevArray&& o) noexcept : p(o.p), n(o.n), s(o.s), pooled(o.pooled) { o.p = nullptr; o.n = 0; }
    DevArray& operator=(DevArray&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p; n = o.n; s = o.s; pooled = o.pooled;
            o.p = nullptr; o.n = 0;
        }
        return *this;
    }
    ~DevArray() { release(); }
    void alloc(size_t count) {
        release();
        if (count) MLSK_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
        pooled = false;
    }
    void alloc_on(size_t count, cudaStream_t st) {
        release();
        configure_mempool();
        if (count) MLSK_CUDA(cudaMallocAsync(&p, count * sizeof(T), st));
        n = count;
        s = st;
        pooled = true;
    }
    void ensure(size_t count) { if (count > n) alloc(count); }
    void release() {
        if (p) {
            if (pooled) cudaFreeAsync(p, s);
            else cudaFree(p);
        }
        p = nullptr;
        n = 0;
    }
    void zero(cudaStream_t st) { if (n) MLSK_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), st)); }
};

inline bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
inline int log2_exact(int64_t n) { int k = 0; while ((int64_t(1) << k) < n) ++k; return k; }
inline int64_t ipow(int64_t M, int64_t l) { int64_t r = 1; while (l-- > 0) r *= M; return r; }

// A model uploaded / generated on the device (models.cpp:12-97 as descriptors).
// Runs f once per (tag, current device): kernel attributes such as the dynamic
// shared-memory limit are set per device context; a process may drive several
// devices (mlsk_exec_opts.device).
template <class F>
void once_per_device(const void* tag, F&& f) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (done.count({tag, dev})) return;
    f();
    done.insert({tag, dev});
}

struct Model {
    uint64_t serial = 0;  // unique per built model (build_model): "same model as the last round"
    mlsk_model_desc desc{};
    DevModel dm{};
    bool vector = false;
    int64_t rows = 1, cols = 1;
    int64_t ref_u64 = 0;  // u64 the reference draw consumes before the indices
    DevArray<double> cum, mean_a, mean_b, mean_at, paper_b;
    DevArray<float> mean_a_f, mean_b_f, mean_at_f, rff_x, rff_xt, rff_w, rff_b;
};

// Validates the descriptor (the reference's constructor checks) and builds it.
void build_model(Model& M, const mlsk_model_desc* d, cudaStream_t st);
bool model_is_vector(const mlsk_model_desc* d);
Tables device_tables();
// index-samples / s of the config-1 per-index RNG work (mlsk_measure_index_rate)
double measure_index_rate(int device);

// A level of the MLMC hierarchy (estimators.cpp:120-122 with c_l = c0 M^l).
struct LevelSpec {
    uint64_t tag;  // l, or MLSK_TAG_MC for the single-level baseline
    int64_t c;     // fine sample size
    int64_t cc;    // coarse sample size (prefix), 0 at level 0 / MC
    bool full = false;  // the whole draw, columns 1..n in order, unweighted: the
                        // reference value (reference_inner/matmul, models.cpp:140-227)
};

// Per-level accumulator state on the device.
//  exact engine: `total` holds the chunk-order sum of closed 64-replication
//  chunks, `open` the partial sum of the chunk still being filled
//  (estimators.cpp:153-169); fused engine: everything lands in `total`.
struct LevelState {
    int64_t cells = 0;
    DevArray<double> buf;  // [total(cells) | total_sq | open(cells) | open_sq]
    int64_t count = 0;     // replications accumulated (this rank)
    int64_t open_count = 0;
    int64_t open_chunk = -1;
    double* total() const { return buf.p; }
    double* total_sq() const { return buf.p + cells; }
    double* open() const { return buf.p + cells + 1; }
    double* open_sq() const { return buf.p + 2 * cells + 1; }
    void init(int64_t cells_, cudaStream_t st) {
        cells = cells_;
        buf.alloc_on(2 * cells + 2, st);
        buf.zero(st);
        count = open_count = 0;
        open_chunk = -1;
    }
};

// A run of consecutive replications inside one 64-replication chunk.
struct Segment {
    int64_t chunk;   // global chunk index q (k / 64)
    int64_t k0;      // first replication
    int64_t count;   // replications in this segment
    bool resumes;    // continues the level's open chunk
    bool closes;     // completes its chunk
};

// Replications [k_begin, k_end) of a level owned by `rank` of `world`
// (chunk q belongs to rank q % world), as chunk segments.
std::vector<Segment> plan_segments(int64_t k_begin, int64_t k_end, int rank, int world,
                                   const LevelState& st);

// Pinned host staging (device->host reads of the level accumulators).
struct PinnedHost {
    double* p = nullptr;
    size_t cap = 0;
    PinnedHost() = default;
    PinnedHost(const PinnedHost&) = delete;
    PinnedHost& operator=(const PinnedHost&) = delete;
    ~PinnedHost() {
        if (p) cudaFreeHost(p);
    }
    double* ensure(size_t n) {
        if (n > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            MLSK_CUDA(cudaMallocHost(&p, n * sizeof(double)));
            cap = n;
        }
        return p;
    }
};

struct Workspace {
    std::shared_ptr<void> fused;  // engine-private pipeline state (mlsk_fused.cu)
    PinnedHost host;              // staging for level reads
    DevArray<uint64_t> stream;
    DevArray<int64_t> ks;
    DevArray<uint32_t> idx;
    DevArray<double> a_cols, b_rows, v, seg_part;
    DevArray<int64_t> seg_desc;
    DevArray<double> panel_a, panel_b, partial;
    DevArray<float> ypart;     // partial Y of a sample split along K (tcgen05 engine)
    DevArray<double> ypart64;  // same, fp64 engine
    DevArray<double> nl_scratch;  // f(coarse) per fragment entry (fp64 engine, nonlinear targets)
};

struct RunArgs {
    const Model* model;
    int target;
    double target_param;
    uint64_t seed;
    cudaStream_t stream;
    Workspace* ws;
    // coupling probe: copy the index sets of replications k < probe_k
    int64_t probe_k;
    uint32_t* probe_host;  // [probe_k][c] for this level, or nullptr
};

// Engines.  Both consume segments in order and update `st`.
void exact_run(const RunArgs& a, const LevelSpec& lv, const std::vector<Segment>& segs, LevelState& st);

// One level's share of a round for the fused engine.
struct FusedJob {
    LevelSpec lv;
    std::vector<Segment> segs;
    LevelState* st;
    uint32_t* probe_host;  // [probe_k][c] or nullptr
};
// A sampled-GEMM engine as seen by the pipelined batch loop (mlsk_fused.cu):
// a panel generator and a GEMM + fused level epilogue + fixed-order reduction.
// K-range of a batch: chunks [kc0, kc0 + nkc) of each sample's K-chunks (nkc < 0:
// all).  part = 0: whole samples; otherwise the batch is ONE sample split along
// K, part = 1 first / 2 middle / 3 last segment, with the partial Y carried
// between segments in device memory (samples whose panels exceed a batch).
//
// Merged sampled columns (round 2): a level-sample's contraction is
//     Y = sum_t w_t a_{j_t} b_{j_t}^T = sum_j W_j a_j b_j^T,  W_j = sum_{t: j_t = j} w_t,
// because a duplicated index gathers the same drawn column (sketch.cpp:60-71)
// -- so the K dimension can run over the DISTINCT sampled columns with summed
// weights, and a column whose fine and coarse weights cancel (M = 2: w_coarse
// = -w_fine, drawn once in the prefix and once in the suffix) drops out.  At
// c = n that is 0.53 c columns instead of c.  A device pre-pass
// (fused_run_round) builds per sample the ordered list of (j, W_j); `mk`
// points at the batch's first sample (mk_stride entries per sample, padding
// entries j = -1, w = 0), mk_info at its (len, neg_kc) and nkc is the merged
// chunk count of the job (the maximum over its samples; slots >= len are
// padding).  neg_kc (tcgen05 engine, shared RFF panel): the sample's leading
// K-chunks that hold its negative-weight columns; there an entry's w is the
// signed column scale sqrt(|W_j| / |w|) applied to the one panel both operand
// roles read (Y = |w| sum_j sign_j (s_j z_j)(s_j z_j)^T).
struct MkEntry {
    int32_t j, reps;  // 0-based column (-1: padding); reps = |cnt_fine - cnt_coarse| (informational)
    double w;
};
struct MkInfo {
    int32_t len, neg_kc;
};
struct KRange {
    int64_t kc0 = 0, nkc = -1;
    int part = 0;
    bool finish = true;  // the level's last batch of this pass (symmetric outputs are mirrored then)
    const MkEntry* mk = nullptr;
    int64_t mk_stride = 0;
    const MkInfo* mk_info = nullptr;
};
struct PanelEngine {
    virtual ~PanelEngine() = default;
    virtual int64_t chunk_cols() const = 0;   // K columns per chunk
    virtual int64_t chunk_bytes() const = 0;  // panel bytes of one chunk of one sample
    // K-chunks of one level-sample (c indices, coarse prefix cc)
    virtual int64_t nchunks(int64_t c, int64_t cc) const {
        (void)cc;
        return (c + chunk_cols() - 1) / chunk_cols();
    }
    int64_t panel_bytes(int64_t c, int64_t cc) const { return nchunks(c, cc) * chunk_bytes(); }
    virtual bool splits_k() const { return false; }
    // merged sampled columns: 0 = not supported for this (c, cc, weights);
    // 1 = one group, weights summed; 2 = sign groups (negative first, each
    // padded to whole K-chunks), columns scaled by sqrt(|W_j| / |w|)
    virtual int merge_mode(int64_t c, int64_t cc, double w_fine, double w_coarse) const {
        (void)c; (void)cc; (void)w_fine; (void)w_coarse;
        return 0;
    }
    virtual int64_t group_size() const = 0;   // samples per round of the CTA groups
    virtual void gen(cudaStream_t s, uint64_t seed, uint64_t tag, const int64_t* ks, int nb, int64_t c, int64_t cc,
                     double w_fine, double w_coarse, void* panels, uint32_t* idx, const KRange& kr) = 0;
    virtual void gemm(cudaStream_t s, const void* panels, int nb, int64_t c, int64_t cc, double w_fine,
                      double w_coarse, LevelState& st, const KRange& kr) = 0;
};
std::unique_ptr<PanelEngine> make_tc_engine(const Model& M, Workspace& ws);  // mlsk_tc.cu

// Runs all jobs of a round as one software pipeline (panel generation of
// batch i+1 overlapped with the GEMM of batch i on two streams).  Work is
// ordered after `a.stream`'s prior work and `a.stream` waits for its end;
// the call returns without a host synchronisation unless a probe is requested.
void fused_run_round(const RunArgs& a, std::vector<FusedJob>& jobs);
bool fused_supported(const Model& M, int target);

// Device-side sketch primitives used by the KAT entry points.
void exact_gather_sample(const Model& M, uint64_t seed, uint64_t tag, int64_t k, int64_t c,
                         uint32_t* idx_host, double* a_host, double* b_host, cudaStream_t st,
                         Workspace& ws);

}  // namespace mlsk
