// mlsk.hpp -- header-only C++ wrapper restoring the reference's estimator
// signatures (/root/reference/proj/include/mlsketch/estimators.hpp:58-80) on
// top of the C-ABI (mlsk.h).  Status codes are rethrown as the reference's
// exception classes: MLSK_EINVAL -> std::invalid_argument, anything else ->
// std::runtime_error.  Link with paper_1904_00429_b200/_lib/libmlsk.so.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "mlsk.h"

namespace mlsketch_b200 {

inline void check(int rc) {
    if (rc == MLSK_OK) return;
    if (rc == MLSK_EINVAL) throw std::invalid_argument(mlsk_last_error());
    throw std::runtime_error(mlsk_last_error());
}

// models.hpp:17-31 -- the std::function draw plugin becomes a descriptor
struct Model {
    mlsk_model_desc desc{};
    std::vector<double> mean_a, mean_b;  // optional host means (fp64 models)
    std::size_t rows() const { return desc.m == 0 && desc.p == 0 ? 1 : (std::size_t)desc.m; }
    std::size_t cols() const { return desc.m == 0 && desc.p == 0 ? 1 : (std::size_t)desc.p; }
};

inline Model paper_inner_model() {  // models.cpp:12-27
    Model m;
    m.desc.kind = MLSK_MODEL_PAPER_INNER;
    m.desc.n = 1000;
    m.desc.stream_mode = MLSK_STREAM_REF;
    return m;
}
inline Model paper_matrix_model() {  // models.cpp:29-52
    Model m;
    m.desc.kind = MLSK_MODEL_PAPER_MATRIX;
    m.desc.m = 10;
    m.desc.n = 1000;
    m.desc.p = 10;
    m.desc.stream_mode = MLSK_STREAM_REF;
    return m;
}
inline Model constant_ones_model(std::size_t n) {  // models.cpp:54-61
    if (n == 0) throw std::invalid_argument("constant_ones_model: n must be positive");
    Model m;
    m.desc.kind = MLSK_MODEL_CONSTANT_ONES;
    m.desc.n = (int64_t)n;
    m.desc.stream_mode = MLSK_STREAM_REF;
    return m;
}
inline Model deterministic_matrix_model() {  // models.cpp:88-97: A = [[1,2],[3,4]], B = [[5,6],[7,8]]
    Model m;
    m.desc.kind = MLSK_MODEL_DETERMINISTIC;
    m.desc.m = 2;
    m.desc.n = 2;
    m.desc.p = 2;
    m.desc.stream_mode = MLSK_STREAM_REF;
    return m;
}
inline Model gaussian_mean_matrix_model(std::size_t m_, std::size_t n, std::size_t p, double sd, double lo, double hi,
                                        std::uint64_t data_seed) {  // BASELINE configs 2-3
    Model m;
    m.desc.kind = MLSK_MODEL_GAUSS_MEAN;
    m.desc.m = (int64_t)m_;
    m.desc.n = (int64_t)n;
    m.desc.p = (int64_t)p;
    m.desc.sd = sd;
    m.desc.mean_lo = lo;
    m.desc.mean_hi = hi;
    m.desc.data_seed = data_seed;
    return m;
}

// models.hpp:35-39
struct TargetFunction {
    int32_t kind;
    double param;
};
inline TargetFunction target_identity() { return {MLSK_TARGET_IDENTITY, 0.0}; }
inline TargetFunction target_f1() { return {MLSK_TARGET_F1, 0.0}; }
inline TargetFunction target_f2(double zeta = 1e-12) {
    if (!(zeta > 0.0)) throw std::invalid_argument("target_f2: zeta must be positive");
    return {MLSK_TARGET_F2, zeta};
}

// planner.hpp:12-20 (+ c0; the reference is c0 = 1)
struct LevelPlan {
    std::size_t M;
    std::size_t L;
    std::vector<long long> N;
    std::size_t c0 = 1;
};

// estimators.hpp:20-36
template <class ValueT>
struct LevelStatistic {
    std::size_t level;
    ValueT estimate;
    long long replication_count;
    double sample_mean_of_squares;
    long long cost_units;
};
template <class ValueT>
struct EstimateReport {
    ValueT value;
    std::vector<LevelStatistic<ValueT>> per_level;
    long long total_cost_units;
    double wall_time_seconds;
    std::uint64_t seed;
};

struct EstimatorOptions {
    int device = -1;
    int engine = MLSK_ENGINE_AUTO;
    int rank = 0, world = 1;
    // several GPUs inside one call (mlsk_exec_opts.n_devices / device_ids; the
    // reference's threads, parallel.hpp:18-52); deterministic: fixed virtual
    // shards, bit-identical results for any device count dividing vshards
    std::vector<int32_t> devices;
    bool deterministic = false;
    int vshards = 0;
};

namespace detail {
inline mlsk_model_desc desc_of(const Model& m) {
    mlsk_model_desc d = m.desc;
    if (!m.mean_a.empty()) d.mean_a = m.mean_a.data();
    if (!m.mean_b.empty()) d.mean_b = m.mean_b.data();
    return d;
}
inline mlsk_exec_opts opts_of(const EstimatorOptions& o) {
    mlsk_exec_opts x{};
    x.device = o.device;
    x.engine = o.engine;
    x.rank = o.rank;
    x.world = o.world;
    if (!o.devices.empty()) {
        x.n_devices = (int32_t)o.devices.size();
        x.device_ids = o.devices.data();  // `o` outlives the call
    }
    x.deterministic = o.deterministic ? 1 : 0;
    x.vshards = o.vshards;
    return x;
}
}  // namespace detail

// mlmc_matmul(model, f, plan, seed, options) -- estimators.hpp:62-67; the
// matrix values are row-major vectors of rows() x cols()
inline EstimateReport<std::vector<double>> mlmc_matmul(const Model& model, const TargetFunction& f,
                                                       const LevelPlan& plan, std::uint64_t seed,
                                                       const EstimatorOptions& options = {}) {
    if (plan.N.size() != plan.L + 1) throw std::invalid_argument("estimator: malformed plan");
    const std::size_t cells = model.rows() * model.cols(), levels = plan.L + 1;
    std::vector<int64_t> N(plan.N.begin(), plan.N.end());
    mlsk_plan p{(int64_t)plan.M, (int64_t)plan.c0, (int64_t)plan.L, N.data()};
    std::vector<double> value(cells), est(levels * cells), msq(levels);
    std::vector<int64_t> cnt(levels), cost(levels);
    mlsk_report r{};
    r.value = value.data();
    r.level_estimate = est.data();
    r.level_mean_sq = msq.data();
    r.level_count = cnt.data();
    r.cost_units = cost.data();
    const mlsk_model_desc d = detail::desc_of(model);
    const mlsk_exec_opts o = detail::opts_of(options);
    check(mlsk_mlmc_matmul(&d, f.kind, f.param, &p, seed, &o, &r));
    EstimateReport<std::vector<double>> out{value, {}, r.total_cost_units, r.wall_time_s, r.seed};
    for (std::size_t l = 0; l < levels; ++l)
        out.per_level.push_back({l, std::vector<double>(est.begin() + l * cells, est.begin() + (l + 1) * cells),
                                 cnt[l], msq[l], cost[l]});
    return out;
}

// mlmc_inner(model, f, plan, seed, options) -- estimators.hpp:52-60
inline EstimateReport<double> mlmc_inner(const Model& model, const TargetFunction& f, const LevelPlan& plan,
                                         std::uint64_t seed, const EstimatorOptions& options = {}) {
    if (plan.N.size() != plan.L + 1) throw std::invalid_argument("estimator: malformed plan");
    const std::size_t levels = plan.L + 1;
    std::vector<int64_t> N(plan.N.begin(), plan.N.end());
    mlsk_plan p{(int64_t)plan.M, (int64_t)plan.c0, (int64_t)plan.L, N.data()};
    double value = 0.0;
    std::vector<double> est(levels), msq(levels);
    std::vector<int64_t> cnt(levels), cost(levels);
    mlsk_report r{};
    r.value = &value;
    r.level_estimate = est.data();
    r.level_mean_sq = msq.data();
    r.level_count = cnt.data();
    r.cost_units = cost.data();
    const mlsk_model_desc d = detail::desc_of(model);
    const mlsk_exec_opts o = detail::opts_of(options);
    check(mlsk_mlmc_inner(&d, f.kind, f.param, &p, seed, &o, &r));
    EstimateReport<double> out{value, {}, r.total_cost_units, r.wall_time_s, r.seed};
    for (std::size_t l = 0; l < levels; ++l) out.per_level.push_back({l, est[l], cnt[l], msq[l], cost[l]});
    return out;
}

// reference_inner / reference_matmul -- models.hpp:78-100 (threads ignored)
struct ScalarReference {
    double value;
    double std_error;
    std::size_t sample_count;
};
struct MatrixReference {
    std::vector<double> value;  // row-major rows() x cols()
    double std_error;
    std::size_t sample_count;
};

inline ScalarReference reference_inner(const Model& model, const TargetFunction& f, std::size_t count,
                                       std::uint64_t seed, const EstimatorOptions& options = {}) {
    ScalarReference r{0.0, 0.0, count};
    const mlsk_model_desc d = detail::desc_of(model);
    const mlsk_exec_opts o = detail::opts_of(options);
    check(mlsk_reference_inner(&d, f.kind, f.param, (int64_t)count, seed, &o, &r.value, &r.std_error));
    return r;
}

inline MatrixReference reference_matmul(const Model& model, const TargetFunction& f, std::size_t count,
                                        std::uint64_t seed, const EstimatorOptions& options = {}) {
    MatrixReference r{std::vector<double>(model.rows() * model.cols()), 0.0, count};
    const mlsk_model_desc d = detail::desc_of(model);
    const mlsk_exec_opts o = detail::opts_of(options);
    check(mlsk_reference_matmul(&d, f.kind, f.param, (int64_t)count, seed, &o, r.value.data(), &r.std_error));
    return r;
}

// Round-based session (adaptive MLMC; no reference analogue): run_round(dN)
// continues every level's replication index; stats() as mlmc_matmul's report;
// checkpoint() / restore() serialise the accumulators (same run only).
class Session {
   public:
    Session(const Model& model, const TargetFunction& f, std::size_t M, std::size_t L, std::uint64_t seed,
            std::size_t c0 = 1, const EstimatorOptions& options = {})
        : L_(L), cells_(model.rows() * model.cols()) {
        const mlsk_model_desc d = detail::desc_of(model);
        const mlsk_exec_opts o = detail::opts_of(options);
        check(mlsk_session_create(&d, f.kind, f.param, (int64_t)M, (int64_t)c0, (int64_t)L, seed, &o, &s_));
    }
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;
    ~Session() {
        if (s_) mlsk_session_destroy(s_);
    }
    void run_round(const std::vector<long long>& dN) {
        if (dN.size() != L_ + 1) throw std::invalid_argument("session: dN must have L+1 entries");
        std::vector<int64_t> d(dN.begin(), dN.end());
        check(mlsk_session_run_round(s_, d.data()));
    }
    EstimateReport<std::vector<double>> stats() {
        const std::size_t levels = L_ + 1;
        std::vector<double> value(cells_), est(levels * cells_), msq(levels);
        std::vector<int64_t> cnt(levels), cost(levels);
        mlsk_report r{};
        r.value = value.data();
        r.level_estimate = est.data();
        r.level_mean_sq = msq.data();
        r.level_count = cnt.data();
        r.cost_units = cost.data();
        check(mlsk_session_stats(s_, &r));
        EstimateReport<std::vector<double>> out{value, {}, r.total_cost_units, r.wall_time_s, r.seed};
        for (std::size_t l = 0; l < levels; ++l)
            out.per_level.push_back({l, std::vector<double>(est.begin() + l * cells_, est.begin() + (l + 1) * cells_),
                                     cnt[l], msq[l], cost[l]});
        return out;
    }
    std::vector<unsigned char> checkpoint() {
        int64_t n = 0;
        check(mlsk_session_checkpoint(s_, nullptr, &n));
        std::vector<unsigned char> img((std::size_t)n);
        check(mlsk_session_checkpoint(s_, img.data(), &n));
        return img;
    }
    void restore(const std::vector<unsigned char>& img) {
        check(mlsk_session_restore(s_, img.data(), (int64_t)img.size()));
    }

   private:
    mlsk_session* s_ = nullptr;
    std::size_t L_, cells_;
};

}  // namespace mlsketch_b200
