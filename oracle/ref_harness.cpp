// ref_harness.cpp -- drives the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/) through
// its public API, to pin the CPU oracle and to serve as the CPU baseline.
//
// TEST INFRASTRUCTURE ONLY.  Nothing here is product code.  The reference
// hard-wires level sizes to M^l (estimators.cpp:57-58,121); the BASELINE
// configs use c_l = c0 * M^l, so `ref_mlmc` composes the reference's own
// public pieces -- RngStream::derive, the model plugin draw,
// draw_realization, sketch_inner / sketch_matmul and detail::parallel_chunks
// -- in the loop of estimators.cpp:105-179 with fine = c0 * M^l.  For c0 = 1
// `ref_mlmc_native` calls mlmc_inner / mlmc_matmul themselves so the tests can
// prove the composed loop equals the reference's.  The configs' data models
// are supplied through the reference's plugin API (models.hpp:17-31).
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <atomic>
#include <memory>
#include <thread>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "mlsketch/estimators.hpp"
#include "mlsketch/models.hpp"
#include "mlsketch/parallel.hpp"
#include "mlsketch/planner.hpp"
#include "mlsketch/tensor.hpp"
#include "mlsketch/rng.hpp"
#include "mlsketch/sampling.hpp"
#include "mlsketch/sketch.hpp"

#include "../include/mlsk.h"

using namespace mlsketch;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return MLSK_EINVAL;
}

bool is_vector(const mlsk_model_desc* d) {
    const int k = d->kind;
    return k == MLSK_MODEL_PAPER_INNER ||
           ((k == MLSK_MODEL_CONSTANT_ONES || k == MLSK_MODEL_DETERMINISTIC ||
             k == MLSK_MODEL_GAUSS_MEAN) &&
            d->m == 0 && d->p == 0);
}

// Config models (BASELINE.json configs 1-2) written against the reference's
// plugin API: a = mean_a + sd * N(0,1) then b = mean_b + sd * N(0,1), drawn in
// the documented order (models.hpp:14-16,23-24).
VectorPairModel vector_model(const mlsk_model_desc* d) {
    switch (d->kind) {
    case MLSK_MODEL_PAPER_INNER: return paper_inner_model();
    case MLSK_MODEL_CONSTANT_ONES: return constant_ones_model(d->n);
    case MLSK_MODEL_DETERMINISTIC: return deterministic_model(d->n);
    case MLSK_MODEL_GAUSS_MEAN: {
        const std::size_t n = d->n;
        const double sd = d->sd;
        std::vector<double> ma((const double*)d->mean_a, (const double*)d->mean_a + n);
        std::vector<double> mb((const double*)d->mean_b, (const double*)d->mean_b + n);
        return VectorPairModel{n, "gauss-mean", [n, sd, ma, mb](RngStream& rng) {
                                   std::vector<double> a(n), b(n);
                                   for (std::size_t j = 0; j < n; ++j) a[j] = ma[j] + sd * rng.normal();
                                   for (std::size_t j = 0; j < n; ++j) b[j] = mb[j] + sd * rng.normal();
                                   return std::make_pair(DenseVector(std::move(a)),
                                                         DenseVector(std::move(b)));
                               }};
    }
    }
    throw std::invalid_argument("harness: unsupported vector model");
}

MatrixPairModel matrix_model(const mlsk_model_desc* d) {
    switch (d->kind) {
    case MLSK_MODEL_PAPER_MATRIX: return paper_matrix_model();
    case MLSK_MODEL_CONSTANT_ONES: return constant_ones_matrix_model(d->m, d->n, d->p);
    case MLSK_MODEL_DETERMINISTIC: return deterministic_matrix_model();
    case MLSK_MODEL_GAUSS_MEAN: {
        const std::size_t m = d->m, n = d->n, p = d->p;
        const double sd = d->sd;
        std::vector<double> ma((const double*)d->mean_a, (const double*)d->mean_a + m * n);
        std::vector<double> mb((const double*)d->mean_b, (const double*)d->mean_b + n * p);
        return MatrixPairModel{m, n, p, "gauss-mean", [m, n, p, sd, ma, mb](RngStream& rng) {
                                   std::vector<double> A(m * n), B(n * p);
                                   for (std::size_t e = 0; e < m * n; ++e) A[e] = ma[e] + sd * rng.normal();
                                   for (std::size_t e = 0; e < n * p; ++e) B[e] = mb[e] + sd * rng.normal();
                                   return std::make_pair(DenseMatrix(m, n, std::move(A)),
                                                         DenseMatrix(n, p, std::move(B)));
                               }};
    }
    }
    throw std::invalid_argument("harness: unsupported matrix model");
}

TargetFunction target(int32_t t, double p) {
    switch (t) {
    case MLSK_TARGET_F1: return target_f1();
    case MLSK_TARGET_F2: return target_f2(p > 0.0 ? p : 1e-12);
    default: return target_identity();
    }
}

long long ipow(long long M, long long l) {
    long long r = 1;
    while (l-- > 0) r *= M;
    return r;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_derive_seed(uint64_t master, uint64_t a, uint64_t b) {
    return RngStream::derive_seed(master, a, b);
}

void ref_u64_stream(uint64_t seed, int64_t count, uint64_t* out) {
    RngStream rng(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = rng.next_u64();
}

void ref_normals(uint64_t seed, int64_t count, double* out) {
    RngStream rng(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = rng.normal();
}

void ref_indices(uint64_t seed, int64_t n, int64_t count, uint32_t* out) {
    RngStream rng(seed);
    const auto dist = IndexDistribution::uniform(n);
    const auto r = draw_realization(dist, count, rng);
    std::memcpy(out, r.indices.data(), sizeof(uint32_t) * count);
}

int ref_sketch_inner(const double* a, const double* b, int64_t n, const uint32_t* idx, int64_t s,
                     double* out) {
    try {
        DenseVector va(std::vector<double>(a, a + n)), vb(std::vector<double>(b, b + n));
        *out = sketch_inner(va, vb, std::span<const uint32_t>(idx, s), IndexDistribution::uniform(n));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_sketch_matmul(const double* A, const double* B, int64_t m, int64_t n, int64_t d,
                      const uint32_t* idx, int64_t s, double* out) {
    try {
        DenseMatrix MA(m, n, std::vector<double>(A, A + m * n));
        DenseMatrix MB(n, d, std::vector<double>(B, B + n * d));
        const auto o = sketch_matmul(MA, MB, std::span<const uint32_t>(idx, s),
                                     IndexDistribution::uniform(n));
        std::memcpy(out, o.data().data(), sizeof(double) * m * d);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// model.draw + draw_realization for replication k of stream tag (estimators.cpp:134-136)
int ref_draw_sample(const mlsk_model_desc* d, uint64_t seed, uint64_t tag, int64_t k, int64_t c,
                    uint32_t* idx, double* a_cols, double* b_rows) {
    try {
        RngStream rng = RngStream::derive(seed, tag, k);
        if (is_vector(d)) {
            const auto model = vector_model(d);
            auto [a, b] = model.draw(rng);
            const auto dist = IndexDistribution::uniform(model.n);
            const Realization r = draw_realization(dist, c, rng);
            for (int64_t i = 0; i < c; ++i) {
                if (idx) idx[i] = r.indices[i];
                if (a_cols) a_cols[i] = a(r.indices[i]);
                if (b_rows) b_rows[i] = b(r.indices[i]);
            }
        } else {
            const auto model = matrix_model(d);
            auto [A, B] = model.draw(rng);
            const auto dist = IndexDistribution::uniform(model.n);
            const Realization r = draw_realization(dist, c, rng);
            for (int64_t i = 0; i < c; ++i) {
                const std::size_t j = r.indices[i];
                if (idx) idx[i] = (uint32_t)j;
                if (a_cols)
                    for (std::size_t row = 1; row <= model.m; ++row) a_cols[(row - 1) * c + i] = A(row, j);
                if (b_rows)
                    for (std::size_t q = 1; q <= model.d; ++q) b_rows[i * model.d + q - 1] = B(j, q);
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}


// The estimators.cpp:105-179 loop composed from reference parts, c_l = c0 M^l.
int ref_mlmc(const mlsk_model_desc* d, int32_t tgt, double tp, const mlsk_plan* plan,
             uint64_t seed, int32_t threads, mlsk_report* rep) {
    try {
        if (plan->M < 2 || plan->L < 0 || plan->c0 < 1) throw std::invalid_argument("estimator: malformed plan");
        for (int64_t l = 0; l <= plan->L; ++l)
            if (plan->N[l] < 1) throw std::invalid_argument("estimator: all N_l must be at least 1");
        const TargetFunction f = target(tgt, tp);
        const bool vec = is_vector(d);
        std::unique_ptr<VectorPairModel> vm;
        std::unique_ptr<MatrixPairModel> mm;
        std::size_t cells, n;
        if (vec) {
            vm = std::make_unique<VectorPairModel>(vector_model(d));
            cells = 1;
            n = vm->n;
        } else {
            mm = std::make_unique<MatrixPairModel>(matrix_model(d));
            cells = mm->m * mm->d;
            n = mm->n;
        }
        const IndexDistribution dist = IndexDistribution::uniform(n);
        if (rep->value) std::fill(rep->value, rep->value + cells, 0.0);
        rep->total_cost_units = 0;
        for (int64_t l = 0; l <= plan->L; ++l) {
            const std::size_t fine = (std::size_t)(plan->c0 * ipow(plan->M, l));
            const std::size_t coarse = l > 0 ? fine / plan->M : 0;
            const std::size_t count = (std::size_t)plan->N[l];
            const std::size_t n_chunks = (count + detail::kReductionChunk - 1) / detail::kReductionChunk;
            std::vector<std::vector<double>> sums(n_chunks);
            std::vector<double> sq_sums(n_chunks, 0.0);
            detail::parallel_chunks(
                count, detail::kReductionChunk, threads,
                [&](std::size_t ch, std::size_t begin, std::size_t end) {
                    std::vector<double> s(cells, 0.0);
                    double s2 = 0.0;
                    for (std::size_t k = begin; k < end; ++k) {
                        RngStream rng = RngStream::derive(seed, l, k);
                        if (vec) {
                            auto [a, b] = vm->draw(rng);
                            const Realization r = draw_realization(dist, fine, rng);
                            double v = f.f(sketch_inner(a, b, r, dist));
                            if (l > 0) {
                                const std::span<const std::uint32_t> pre(r.indices.data(), coarse);
                                v -= f.f(sketch_inner(a, b, pre, dist));
                            }
                            s[0] += v;
                            s2 += v * v;
                        } else {
                            auto [A, B] = mm->draw(rng);
                            const Realization r = draw_realization(dist, fine, rng);
                            DenseMatrix v = sketch_matmul(A, B, r, dist);
                            for (double& x : v.data()) x = f.f(x);
                            if (l > 0) {
                                const std::span<const std::uint32_t> pre(r.indices.data(), coarse);
                                const DenseMatrix cv = sketch_matmul(A, B, pre, dist);
                                for (std::size_t t = 0; t < cells; ++t) v.data()[t] -= f.f(cv.data()[t]);
                            }
                            for (std::size_t t = 0; t < cells; ++t) {
                                const double x = v.data()[t];
                                s[t] += x;
                                s2 += x * x;
                            }
                        }
                    }
                    sums[ch] = std::move(s);
                    sq_sums[ch] = s2;
                });
            std::vector<double> sum(cells, 0.0);
            double sq = 0.0;
            for (std::size_t ch = 0; ch < n_chunks; ++ch) {
                for (std::size_t t = 0; t < cells; ++t) sum[t] += sums[ch][t];
                sq += sq_sums[ch];
            }
            const double inv_n = 1.0 / static_cast<double>(count);
            const long long cost = (long long)count * (long long)(fine + coarse) * (long long)cells;
            for (std::size_t t = 0; t < cells; ++t) {
                if (rep->level_sum) rep->level_sum[l * cells + t] = sum[t];
                if (rep->level_estimate) rep->level_estimate[l * cells + t] = sum[t] * inv_n;
                if (rep->value) rep->value[t] += sum[t] * inv_n;
            }
            if (rep->level_sumsq) rep->level_sumsq[l] = sq;
            if (rep->level_mean_sq) rep->level_mean_sq[l] = sq * inv_n;
            if (rep->level_count) rep->level_count[l] = plan->N[l];
            if (rep->cost_units) rep->cost_units[l] = cost;
            rep->total_cost_units += cost;
        }
        rep->seed = seed;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The reference's own mlmc_inner / mlmc_matmul (c0 = 1 only).
int ref_mlmc_native(const mlsk_model_desc* d, int32_t tgt, double tp, const mlsk_plan* plan,
                    uint64_t seed, int32_t threads, mlsk_report* rep) {
    try {
        if (plan->c0 != 1) throw std::invalid_argument("native reference: c0 must be 1");
        LevelPlan lp{(std::size_t)plan->M, (std::size_t)plan->L,
                     std::vector<long long>(plan->N, plan->N + plan->L + 1), 0.1, 1.0, 1.0, false};
        EstimatorOptions opt;
        opt.threads = threads;
        if (is_vector(d)) {
            const auto r = mlmc_inner(vector_model(d), target(tgt, tp), lp, seed, opt);
            if (rep->value) rep->value[0] = r.value;
            for (std::size_t l = 0; l < r.per_level.size(); ++l) {
                if (rep->level_estimate) rep->level_estimate[l] = r.per_level[l].estimate;
                if (rep->level_mean_sq) rep->level_mean_sq[l] = r.per_level[l].sample_mean_of_squares;
                if (rep->level_count) rep->level_count[l] = r.per_level[l].replication_count;
                if (rep->cost_units) rep->cost_units[l] = r.per_level[l].cost_units;
            }
            rep->total_cost_units = r.total_cost_units;
            rep->wall_time_s = r.wall_time_seconds;
        } else {
            const auto r = mlmc_matmul(matrix_model(d), target(tgt, tp), lp, seed, opt);
            const std::size_t cells = r.value.rows() * r.value.cols();
            if (rep->value) std::memcpy(rep->value, r.value.data().data(), sizeof(double) * cells);
            for (std::size_t l = 0; l < r.per_level.size(); ++l) {
                if (rep->level_estimate)
                    std::memcpy(rep->level_estimate + l * cells, r.per_level[l].estimate.data().data(),
                                sizeof(double) * cells);
                if (rep->level_mean_sq) rep->level_mean_sq[l] = r.per_level[l].sample_mean_of_squares;
                if (rep->level_count) rep->level_count[l] = r.per_level[l].replication_count;
                if (rep->cost_units) rep->cost_units[l] = r.per_level[l].cost_units;
            }
            rep->total_cost_units = r.total_cost_units;
            rep->wall_time_s = r.wall_time_seconds;
        }
        rep->seed = seed;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The reference's own mc_inner / mc_matmul (sample size M^L).
int ref_mc_native(const mlsk_model_desc* d, int32_t tgt, double tp, int64_t L, int64_t N,
                  int64_t M, uint64_t seed, int32_t threads, mlsk_report* rep) {
    try {
        EstimatorOptions opt;
        opt.threads = threads;
        if (is_vector(d)) {
            const auto r = mc_inner(vector_model(d), target(tgt, tp), L, N, M, seed, opt);
            if (rep->value) rep->value[0] = r.value;
            rep->total_cost_units = r.total_cost_units;
        } else {
            const auto r = mc_matmul(matrix_model(d), target(tgt, tp), L, N, M, seed, opt);
            const std::size_t cells = r.value.rows() * r.value.cols();
            if (rep->value) std::memcpy(rep->value, r.value.data().data(), sizeof(double) * cells);
            rep->total_cost_units = r.total_cost_units;
        }
        rep->seed = seed;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// CPU-baseline throughput run: every (level, replication) item of the plan
// executes the reference's per-replication body (estimators.cpp:133-158:
// RngStream::derive, model.draw, draw_realization, sketch fine + coarse
// prefix, f, accumulate) and the items are spread over `threads` host
// threads with an atomic counter (the reference's parallel_chunks caps a
// level at ceil(N_l / 64) threads, which would idle most cores on a bounded
// sample).  Returns the wall time in seconds; *checksum gets sum of ||Y||^2.
double ref_throughput(const mlsk_model_desc* d, int32_t tgt, double tp, const mlsk_plan* plan,
                      uint64_t seed, int32_t threads, double* checksum) {
    try {
        const TargetFunction f = target(tgt, tp);
        const bool vec = is_vector(d);
        std::unique_ptr<VectorPairModel> vm;
        std::unique_ptr<MatrixPairModel> mm;
        std::size_t n;
        if (vec) { vm = std::make_unique<VectorPairModel>(vector_model(d)); n = vm->n; }
        else { mm = std::make_unique<MatrixPairModel>(matrix_model(d)); n = mm->n; }
        const IndexDistribution dist = IndexDistribution::uniform(n);
        std::vector<std::pair<int64_t, int64_t>> items;  // (level, k)
        for (int64_t l = 0; l <= plan->L; ++l)
            for (int64_t k = 0; k < plan->N[l]; ++k) items.emplace_back(l, k);
        std::atomic<std::size_t> next{0};
        std::vector<double> part(std::max(1, threads), 0.0);
        const auto t0 = std::chrono::steady_clock::now();
        auto worker = [&](int w) {
            double acc = 0.0;
            for (;;) {
                const std::size_t i = next.fetch_add(1);
                if (i >= items.size()) break;
                const auto [l, k] = items[i];
                const std::size_t fine = (std::size_t)(plan->c0 * ipow(plan->M, l));
                const std::size_t coarse = l > 0 ? fine / plan->M : 0;
                RngStream rng = RngStream::derive(seed, l, k);
                if (vec) {
                    auto [a, b] = vm->draw(rng);
                    const Realization r = draw_realization(dist, fine, rng);
                    double v = f.f(sketch_inner(a, b, r, dist));
                    if (l > 0) v -= f.f(sketch_inner(a, b, std::span<const uint32_t>(r.indices.data(), coarse), dist));
                    acc += v * v;
                } else {
                    auto [A, B] = mm->draw(rng);
                    const Realization r = draw_realization(dist, fine, rng);
                    DenseMatrix v = sketch_matmul(A, B, r, dist);
                    for (double& x : v.data()) x = f.f(x);
                    if (l > 0) {
                        const DenseMatrix cv =
                            sketch_matmul(A, B, std::span<const uint32_t>(r.indices.data(), coarse), dist);
                        for (std::size_t t = 0; t < v.data().size(); ++t) v.data()[t] -= f.f(cv.data()[t]);
                    }
                    for (double x : v.data()) acc += x * x;
                }
            }
            part[w] = acc;
        };
        std::vector<std::thread> pool;
        for (int w = 0; w < std::max(1, threads); ++w) pool.emplace_back(worker, w);
        for (auto& t : pool) t.join();
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        double sum = 0.0;
        for (double x : part) sum += x;
        if (checksum) *checksum = sum;
        return dt;
    } catch (const std::exception& e) {
        fail(e);
        return -1.0;
    }
}

// Reference sketch_matmul throughput probe for the CPU baseline of the large
// configs: sketch of pre-drawn A (m x n), B (n x d) on c indices.
double ref_time_sketch_matmul(int64_t m, int64_t n, int64_t d, int64_t c, uint64_t seed, int32_t reps) {
    std::vector<double> a(m * n), b(n * d);
    RngStream rng(seed);
    for (auto& x : a) x = rng.uniform01();
    for (auto& x : b) x = rng.uniform01();
    DenseMatrix A(m, n, std::move(a)), B(n, d, std::move(b));
    const auto dist = IndexDistribution::uniform(n);
    const Realization r = draw_realization(dist, c, rng);
    double chk = 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) chk += sketch_matmul(A, B, r, dist)(1, 1);
    const auto t1 = std::chrono::steady_clock::now();
    if (chk == 12345.678) g_err = "unlikely";
    return std::chrono::duration<double>(t1 - t0).count() / reps;
}

// ---- CLI output restatement (the reference CLI itself cannot be built here:
// CLI11.hpp is missing).  These compose the reference library's public
// functions exactly as mlsketch_main.cpp's cmd_sweep (:112-198) and
// cmd_estimate (:250-316) do and format the same text, to produce golden
// outputs for the B200 CLI (paper_1904_00429_b200/cli.py).

namespace {
std::string fmtd(const char* spec, double v) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), spec, v);
    return buf;
}
int copy_out(const std::string& text, char* buf, int64_t cap) {
    if ((int64_t)text.size() + 1 > cap) {
        g_err = "output buffer too small";
        return -(int)text.size() - 1;
    }
    std::memcpy(buf, text.c_str(), text.size() + 1);
    return (int)text.size();
}
}  // namespace

// reference_inner / reference_matmul (models.cpp:140-227)
int ref_reference_value(const mlsk_model_desc* d, int32_t tgt, double tp, int64_t count, uint64_t seed,
                        int32_t threads, double* mean, double* se) {
    try {
        if (is_vector(d)) {
            const auto r = reference_inner(vector_model(d), target(tgt, tp), (std::size_t)count, seed, threads);
            mean[0] = r.value;
            *se = r.std_error;
        } else {
            const auto r = reference_matmul(matrix_model(d), target(tgt, tp), (std::size_t)count, seed, threads);
            std::memcpy(mean, r.value.data().data(), sizeof(double) * r.value.rows() * r.value.cols());
            *se = r.std_error;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// make_plan / plan_N_mc (planner.cpp:83-100); N_out holds up to `cap` levels
int ref_make_plan(double eps, int64_t M, double c1, double c2, int64_t n, int64_t* L, int64_t* N_out, int64_t cap,
                  int32_t* n_cap_applied, int64_t* N_mc) {
    try {
        const LevelPlan p = make_plan(eps, (std::size_t)M, c1, c2, (std::size_t)n);
        *L = (int64_t)p.L;
        for (std::size_t l = 0; l < p.N.size() && (int64_t)l < cap; ++l) N_out[l] = p.N[l];
        *n_cap_applied = p.n_cap_applied ? 1 : 0;
        *N_mc = plan_N_mc(eps, c2);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// cmd_sweep (mlsketch_main.cpp:112-198) with --no-timing; returns the CSV length
int ref_sweep_csv(const char* mode, const char* model_key, const char* target_key, const int64_t* m_list, int32_t nm,
                  double eps, double c1, double c2, uint64_t seed, int32_t reps, int64_t n_ref, int32_t threads,
                  char* buf, int64_t cap) {
    try {
        const std::string md(mode);
        auto t = target_by_key(target_key);
        if (!t) throw std::invalid_argument("unknown target");
        // plain snprintf (no iostreams: the harness is loaded into processes
        // that carry their own libstdc++)
        std::string out = "M,L,M_pow_L,RE_mlmc,time_mlmc_s,cost_units_mlmc,RE_mc,time_mc_s,cost_units_mc,seed\n";
        const std::uint64_t ref_seed = RngStream::derive_seed(seed, 999983, 0);
        EstimatorOptions opts;
        opts.threads = threads;
        auto row = [&](std::size_t M, std::size_t L, double re1, long long c1u, double re2, long long c2u,
                       std::uint64_t rs) {
            char line[512];
            std::snprintf(line, sizeof(line), "%zu,%zu,%lld,%s,%s,%lld,%s,%s,%lld,%" PRIu64 "\n", M, L, int_pow(M, L),
                          fmtd("%.6e", re1).c_str(), fmtd("%.3f", 0.0).c_str(), c1u, fmtd("%.6e", re2).c_str(),
                          fmtd("%.3f", 0.0).c_str(), c2u, rs);
            out += line;
        };
        if (md == "inner") {
            auto model = vector_model_by_key(model_key);
            if (!model) throw std::invalid_argument("unknown vector model");
            const auto ref = reference_inner(*model, *t, (std::size_t)n_ref, ref_seed, threads);
            for (int32_t i = 0; i < nm; ++i) {
                const std::size_t M = (std::size_t)m_list[i];
                const auto plan = make_plan(eps, M, c1, c2, model->n);
                const long long N_mc = plan_N_mc(eps, c2);
                for (int rep = 0; rep < reps; ++rep) {
                    const std::uint64_t rs = RngStream::derive_seed(seed, M, rep);
                    const auto ml = mlmc_inner(*model, *t, plan, RngStream::derive_seed(rs, 1, 0), opts);
                    const auto mc = mc_inner(*model, *t, plan.L, N_mc, M, RngStream::derive_seed(rs, 2, 0), opts);
                    row(M, plan.L, relative_error(ml.value, ref.value), ml.total_cost_units,
                        relative_error(mc.value, ref.value), mc.total_cost_units, rs);
                }
            }
        } else {
            auto model = matrix_model_by_key(model_key);
            if (!model) throw std::invalid_argument("unknown matrix model");
            const auto ref = reference_matmul(*model, *t, (std::size_t)n_ref, ref_seed, threads);
            for (int32_t i = 0; i < nm; ++i) {
                const std::size_t M = (std::size_t)m_list[i];
                const auto plan = make_plan(eps, M, c1, c2, model->n);
                const long long N_mc = plan_N_mc(eps, c2);
                for (int rep = 0; rep < reps; ++rep) {
                    const std::uint64_t rs = RngStream::derive_seed(seed, M, rep);
                    const auto ml = mlmc_matmul(*model, *t, plan, RngStream::derive_seed(rs, 1, 0), opts);
                    const auto mc = mc_matmul(*model, *t, plan.L, N_mc, M, RngStream::derive_seed(rs, 2, 0), opts);
                    row(M, plan.L, relative_error(ml.value, ref.value), ml.total_cost_units,
                        relative_error(mc.value, ref.value), mc.total_cost_units, rs);
                }
            }
        }
        return copy_out(out, buf, cap);
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

// cmd_estimate (mlsketch_main.cpp:250-316); the wall_time_s line is written as 0.000
int ref_estimate_text(const char* mode, const char* model_key, const char* target_key, int64_t M, double eps,
                      double c1, double c2, uint64_t seed, int32_t threads, char* buf, int64_t cap) {
    try {
        const std::string md(mode);
        auto t = target_by_key(target_key);
        if (!t) throw std::invalid_argument("unknown target");
        EstimatorOptions opts;
        opts.threads = threads;
        std::string o;
        char line[512];
        std::snprintf(line, sizeof(line), "mode=%s model=%s target=%s\n", mode, model_key, target_key);
        o += line;
        if (md == "inner") {
            auto model = vector_model_by_key(model_key);
            if (!model) throw std::invalid_argument("unknown vector model");
            const auto plan = make_plan(eps, (std::size_t)M, c1, c2, model->n);
            const auto rep = mlmc_inner(*model, *t, plan, seed, opts);
            std::snprintf(line, sizeof(line), "M=%zu L=%zu epsilon=%g n=%zu%s\n", plan.M, plan.L, plan.epsilon,
                          model->n, plan.n_cap_applied ? " (depth set by dimension cap)" : "");
            o += line;
            o += "level  N          estimate        mean_sq_diff    cost_units\n";
            for (const auto& st : rep.per_level) {
                std::snprintf(line, sizeof(line), "%-5zu  %-9lld  %-14.8g  %-14.8g  %lld\n", st.level,
                              st.replication_count, st.estimate, st.sample_mean_of_squares, st.cost_units);
                o += line;
            }
            std::snprintf(line, sizeof(line), "estimate=%.10g\ntotal_cost_units=%lld\nwall_time_s=%.3f\nseed=%" PRIu64 "\n",
                          rep.value, rep.total_cost_units, 0.0, rep.seed);
            o += line;
        } else {
            auto model = matrix_model_by_key(model_key);
            if (!model) throw std::invalid_argument("unknown matrix model");
            const auto plan = make_plan(eps, (std::size_t)M, c1, c2, model->n);
            const auto rep = mlmc_matmul(*model, *t, plan, seed, opts);
            std::snprintf(line, sizeof(line), "M=%zu L=%zu epsilon=%g n=%zu m=%zu d=%zu%s\n", plan.M, plan.L,
                          plan.epsilon, model->n, model->m, model->d,
                          plan.n_cap_applied ? " (depth set by dimension cap)" : "");
            o += line;
            o += "level  N          frob_estimate   mean_sq_diff    cost_units\n";
            for (const auto& st : rep.per_level) {
                std::snprintf(line, sizeof(line), "%-5zu  %-9lld  %-14.8g  %-14.8g  %lld\n", st.level,
                              st.replication_count, std::sqrt(frobenius_norm_sq(st.estimate)),
                              st.sample_mean_of_squares, st.cost_units);
                o += line;
            }
            std::snprintf(line, sizeof(line), "estimate (%zux%zu):\n", rep.value.rows(), rep.value.cols());
            o += line;
            for (std::size_t i = 1; i <= rep.value.rows(); ++i) {
                for (std::size_t j = 1; j <= rep.value.cols(); ++j) {
                    std::snprintf(line, sizeof(line), "%s%.8g", j == 1 ? "  " : " ", rep.value(i, j));
                    o += line;
                }
                o += "\n";
            }
            std::snprintf(line, sizeof(line), "total_cost_units=%lld\nwall_time_s=%.3f\nseed=%" PRIu64 "\n",
                          rep.total_cost_units, 0.0, rep.seed);
            o += line;
        }
        return copy_out(o, buf, cap);
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

}  // extern "C"
