// mlsk_api.cu -- the C-ABI of include/mlsk.h.
//
// Mirrors the reference entry points (estimators.hpp:58-80, sketch.hpp:17-51)
// with the reference's validation order and error classes; maps internal
// exceptions to status codes and keeps a thread-local last-error message.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <thread>

#include "mlsk_internal.h"

namespace mlsk {
thread_local int64_t g_launches = 0;
thread_local int64_t g_columns[2] = {0, 0};
int run_guarded(const std::function<void()>& body);
}

using namespace mlsk;

namespace {

thread_local std::string g_last_error;

// The caller's current device is restored on return: entry points select
// their device (mlsk_exec_opts.device / the session's) only for the call.
struct DeviceRestore {
    int dev = -1;
    DeviceRestore() {
        if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
    }
    ~DeviceRestore() {
        int now = -1;
        if (dev >= 0 && cudaGetDevice(&now) == cudaSuccess && now != dev) cudaSetDevice(dev);
    }
};

int guard(const std::function<void()>& body) {
    DeviceRestore restore;
    try {
        body();
        return MLSK_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return MLSK_ERUNTIME;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return MLSK_ERUNTIME;
    }
}

// MLSK_TRACE=1: per-phase host (enqueue) and device (event) times of an
// estimator call, printed to stderr (diagnostics only).
struct Trace {
    bool on;
    cudaStream_t s;
    std::vector<std::pair<std::string, cudaEvent_t>> ev;
    std::vector<double> host;
    std::chrono::steady_clock::time_point t0;
    explicit Trace(cudaStream_t st) : on(getenv("MLSK_TRACE") != nullptr), s(st) {
        if (on) {
            t0 = std::chrono::steady_clock::now();
            mark("start");
        }
    }
    void mark(const char* name) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        ev.emplace_back(name, e);
        host.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    void report() {
        if (!on) return;
        cudaEventSynchronize(ev.back().second);
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
            fprintf(stderr, "[mlsk trace] %-16s host %8.3f ms  device %8.3f ms\n", ev[i].first.c_str(),
                    host[i] - host[i - 1], ms);
        }
        for (auto& e : ev) cudaEventDestroy(e.second);
        ev.clear();
    }
};

// Per-call execution context: device selection and stream.
// One library stream per (host thread, device), destroyed with the thread
// (a host thread pool calling the library does not leak streams).
struct LibStreams {
    std::map<int, cudaStream_t> by_device;
    cudaStream_t get(int device) {
        auto it = by_device.find(device);
        if (it == by_device.end()) {
            cudaStream_t st;
            MLSK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            it = by_device.emplace(device, st).first;
        }
        return it->second;
    }
    ~LibStreams() {
        int cur = -1;
        if (cudaGetDevice(&cur) != cudaSuccess) return;  // runtime already torn down
        for (auto& kv : by_device) {
            if (cudaSetDevice(kv.first) == cudaSuccess) {
                cudaStreamSynchronize(kv.second);
                cudaStreamDestroy(kv.second);
            }
        }
        cudaSetDevice(cur);
    }
};

struct Exec {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool owns = false;
    int engine = MLSK_ENGINE_AUTO;
    int rank = 0, world = 1;
    int64_t probe_k = 0;
    uint32_t* probe_out = nullptr;
    std::vector<int> slots;  // device slots (multi-GPU inside the call); empty: one device
    bool deterministic = false;
    int vshards = 8;

    // the options' multi-device request, validated (no device is touched)
    static void multi_of(const mlsk_exec_opts* o, std::vector<int>& slots, bool& det, int& vsh) {
        slots.clear();
        det = false;
        vsh = 8;
        if (!o) return;
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
        if (o->n_devices < 0) invalid("exec: n_devices must be non-negative");
        if (o->n_devices > 1 || o->deterministic) {
            const int nd = o->n_devices > 1 ? o->n_devices : 1;
            for (int i = 0; i < nd; ++i) {
                const int d = o->device_ids ? o->device_ids[i] : (o->n_devices > 1 ? i : std::max(0, o->device));
                if (d < 0 || d >= ndev) invalid("exec: device id out of range");
                slots.push_back(d);
            }
        }
        det = o->deterministic != 0;
        vsh = o->vshards > 0 ? o->vshards : 8;
        if (det) {
            const int world = o->world <= 0 ? 1 : o->world;
            if (world != 1) invalid("exec: deterministic mode needs world == 1 (across processes: ShardedSession)");
            if (vsh % (int)slots.size() != 0) invalid("exec: n_devices must divide vshards");
        }
    }

    explicit Exec(const mlsk_exec_opts* o) {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw Error(MLSK_ERUNTIME, "no CUDA device available (the library has no CPU fallback)");
        if (o) {
            engine = o->engine;
            rank = o->rank;
            world = o->world <= 0 ? 1 : o->world;
            probe_k = o->probe_k;
            probe_out = o->probe_out;
            multi_of(o, slots, deterministic, vshards);
            if (rank < 0 || rank >= world) invalid("exec: rank out of range");
            if (engine < MLSK_ENGINE_AUTO || engine > MLSK_ENGINE_FUSED) invalid("exec: unknown engine");
        }
        if (o && o->device >= 0) {
            if (o->device >= ndev) invalid("exec: device ordinal out of range");
            device = o->device;
            MLSK_CUDA(cudaSetDevice(device));
        } else {
            MLSK_CUDA(cudaGetDevice(&device));
        }
        if (o && o->stream) {
            stream = (cudaStream_t)o->stream;
        } else {
            // one library stream per (thread, device), reused by every call: the
            // stream-ordered pool then recycles the per-call allocations in order
            // (a fresh stream per call made pool reuse opportunistic and call
            // times erratic)
            static thread_local LibStreams streams;
            stream = streams.get(device);
            owns = true;  // library stream: calls synchronise before returning
        }
    }
};

void check_plan(const mlsk_plan* plan) {  // estimators.cpp:23-32
    if (!plan || !plan->N || plan->M < 2 || plan->L < 0) invalid("estimator: malformed plan");
    if (plan->c0 < 1) invalid("estimator: c0 must be at least 1");
    for (int64_t l = 0; l <= plan->L; ++l)
        if (plan->N[l] < 1) invalid("estimator: all N_l must be at least 1");
    // c_L = c0 M^L must be representable
    double cl = (double)plan->c0;
    for (int64_t l = 0; l < plan->L; ++l) cl *= (double)plan->M;
    if (cl > 4.0e9) invalid("estimator: c0 * M^L exceeds the index-count limit");
}

void check_target(int32_t target, double param) {
    if (target < MLSK_TARGET_IDENTITY || target > MLSK_TARGET_F2) invalid("target: unknown target");
    if (target == MLSK_TARGET_F2 && !(param > 0.0)) invalid("target_f2: zeta must be positive");
}

// Workspaces of the one-shot estimator calls are cached per host thread and
// device, so repeated calls reuse the panel buffers and pipeline streams.
Workspace& cached_workspace(int device) {
    static thread_local std::map<int, std::unique_ptr<Workspace>> cache;
    auto& w = cache[device];
    if (!w) w.reset(new Workspace());
    return *w;
}

// Level driver shared by the estimators and the sessions.
struct Runner {
    Model model;
    Workspace own_ws;
    Workspace* wsp = &own_ws;
    int target;
    double tparam;
    uint64_t seed;
    int engine;  // resolved
    int rank, world;

    void resolve_engine(int requested) {
        const bool fused_ok = fused_supported(model, target);
        if (requested == MLSK_ENGINE_FUSED && !fused_ok)
            invalid("engine: the fused engine needs the philox stream and a supported model (fp32 models: identity target)");
        engine = requested == MLSK_ENGINE_AUTO ? (fused_ok ? MLSK_ENGINE_FUSED : MLSK_ENGINE_EXACT) : requested;
    }

    // one level (estimators) or several levels (a session round) at once
    struct Item {
        LevelSpec lv;
        int64_t k0, k1;
        LevelState* st;
        uint32_t* probe;
    };
    void run(const std::vector<Item>& items, cudaStream_t s, int64_t probe_k) {
        if (engine == MLSK_ENGINE_FUSED) {
            std::vector<FusedJob> jobs;
            for (const auto& it : items) {
                // the fused engines need only which replications run (no open
                // 64-chunk bookkeeping): at world 1 one segment per level (per-chunk
                // segments cost ~16 k host objects per config-1 round)
                std::vector<Segment> segs;
                if (world == 1) {
                    if (it.k1 > it.k0) segs.push_back(Segment{it.k0 / 64, it.k0, it.k1 - it.k0, false, false});
                } else {
                    segs = plan_segments(it.k0, it.k1, rank, world, *it.st);
                }
                jobs.push_back(FusedJob{it.lv, std::move(segs), it.st, it.probe});
            }
            RunArgs a{&model, target, tparam, seed, s, wsp, probe_k, nullptr};
            fused_run_round(a, jobs);
            return;
        }
        for (const auto& it : items) {
            const auto segs = plan_segments(it.k0, it.k1, rank, world, *it.st);
            RunArgs a{&model, target, tparam, seed, s, wsp, probe_k, it.probe};
            exact_run(a, it.lv, segs, *it.st);
        }
    }
};

// All levels' sums / sums of squares in one pass: one device->host copy per
// level into pinned staging (only [total | total_sq] unless a chunk is
// open), one synchronisation.
void read_levels(const std::vector<LevelState>& sts, cudaStream_t s, Workspace& ws, std::vector<const double*>& sums,
                 std::vector<double>& sqs) {
    size_t need = 0;
    for (const auto& st : sts) need += (st.open_count > 0 ? 2 : 1) * (size_t)(st.cells + 1);
    double* h = ws.host.ensure(std::max<size_t>(need, 1));
    size_t off = 0;
    for (const auto& st : sts) {
        const size_t n = (st.open_count > 0 ? 2 : 1) * (size_t)(st.cells + 1);
        MLSK_CUDA(cudaMemcpyAsync(h + off, st.buf.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        off += n;
    }
    MLSK_CUDA(cudaStreamSynchronize(s));
    sums.resize(sts.size());
    sqs.resize(sts.size());
    off = 0;
    for (size_t l = 0; l < sts.size(); ++l) {
        const int64_t cells = sts[l].cells;
        double* b = h + off;  // the level's sums, read in place from the staging buffer
        if (sts[l].open_count > 0) {  // fold the open chunk in (last in order)
            for (int64_t t = 0; t < cells; ++t) b[t] += b[cells + 1 + t];
            b[cells] += b[2 * cells + 1];
        }
        sums[l] = b;
        sqs[l] = b[cells];
        off += (sts[l].open_count > 0 ? 2 : 1) * (size_t)(cells + 1);
    }
}

// level sum / sum of squares on the host: total (+ open chunk, last in order)
void read_level(const LevelState& st, cudaStream_t s, std::vector<double>& sum, double& sq) {
    const int64_t cells = st.cells;
    std::vector<double> h(2 * cells + 2);
    MLSK_CUDA(cudaMemcpyAsync(h.data(), st.buf.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
    MLSK_CUDA(cudaStreamSynchronize(s));
    sum.assign(h.begin(), h.begin() + cells);
    sq = h[cells];
    if (st.open_count > 0) {
        for (int64_t t = 0; t < cells; ++t) sum[t] += h[cells + 1 + t];
        sq += h[2 * cells + 1];
    }
}

int mlmc_impl(bool matrix, const mlsk_model_desc* model, int32_t target, double tparam, const mlsk_plan* plan,
              uint64_t seed, const mlsk_exec_opts* opts, mlsk_report* rep) {
    return guard([&] {
        const auto t0 = std::chrono::steady_clock::now();
        check_plan(plan);
        check_target(target, tparam);
        if (!model) invalid("model: null descriptor");
        if (model_is_vector(model) == matrix) invalid("estimator: model kind does not match the estimator");
        if (opts && (opts->n_devices > 1 || opts->deterministic)) {
            // multi-GPU inside the call: a multi-device session, one round
            mlsk_session* s = nullptr;
            int rc = mlsk_session_create(model, target, tparam, plan->M, plan->c0, plan->L, seed, opts, &s);
            if (rc == MLSK_OK) rc = mlsk_session_run_round(s, plan->N);
            if (rc == MLSK_OK && rep) rc = mlsk_session_stats(s, rep);
            const std::string msg = rc == MLSK_OK ? "" : mlsk_last_error();
            if (s) mlsk_session_destroy(s);
            if (rc != MLSK_OK) throw Error(rc, msg);
            if (rep) rep->wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            return;
        }
        Exec ex(opts);
        Trace tr(ex.stream);
        Runner R;
        R.wsp = &cached_workspace(ex.device);
        tr.mark("exec+workspace");
        build_model(R.model, model, ex.stream);
        tr.mark("build_model");
        R.target = target;
        R.tparam = tparam;
        R.seed = seed;
        R.rank = ex.rank;
        R.world = ex.world;
        R.resolve_engine(ex.engine);
        const int64_t cells = R.model.rows * R.model.cols;
        std::vector<double> value(cells, 0.0);
        int64_t total_cost = 0;
        const int64_t cL = plan->c0 * ipow(plan->M, plan->L);
        std::vector<LevelState> states(plan->L + 1);
        std::vector<Runner::Item> items;
        for (int64_t l = 0; l <= plan->L; ++l) {
            const int64_t fine = plan->c0 * ipow(plan->M, l);
            const int64_t coarse = l > 0 ? fine / plan->M : 0;
            states[l].init(cells, ex.stream);
            uint32_t* probe = nullptr;
            if (ex.probe_out && ex.probe_k > 0 && l > 0) probe = ex.probe_out + l * ex.probe_k * cL;
            items.push_back({LevelSpec{(uint64_t)l, fine, coarse}, 0, plan->N[l], &states[l], probe});
        }
        tr.mark("level states");
        R.run(items, ex.stream, ex.probe_k);  // all levels as one round
        tr.mark("round");
        std::vector<const double*> sums;
        std::vector<double> sqs;
        read_levels(states, ex.stream, *R.wsp, sums, sqs);
        tr.mark("level d2h");
        double* const lsum = rep ? rep->level_sum : nullptr;
        double* const lest = rep ? rep->level_estimate : nullptr;
        for (int64_t l = 0; l <= plan->L; ++l) {
            const int64_t fine = plan->c0 * ipow(plan->M, l);
            const int64_t coarse = l > 0 ? fine / plan->M : 0;
            const LevelState& st = states[l];
            const double* sum = sums[l];
            const double sq = sqs[l];
            const double inv_n = 1.0 / (double)plan->N[l];
            const int64_t cost = plan->N[l] * (fine + coarse) * cells;  // estimators.cpp:34-40
            total_cost += cost;
            if (lsum) std::memcpy(lsum + l * cells, sum, sizeof(double) * cells);
            if (lest)
                for (int64_t t = 0; t < cells; ++t) lest[l * cells + t] = sum[t] * inv_n;
            if (rep) {
                if (rep->level_sumsq) rep->level_sumsq[l] = sq;
                if (rep->level_mean_sq) rep->level_mean_sq[l] = sq * inv_n;
                if (rep->level_count) rep->level_count[l] = st.count;
                if (rep->cost_units) rep->cost_units[l] = cost;
            }
            for (int64_t t = 0; t < cells; ++t) value[t] += sum[t] * inv_n;  // estimators.cpp:179-184
        }
        MLSK_CUDA(cudaStreamSynchronize(ex.stream));
        tr.mark("read levels");
        tr.report();
        if (rep) {
            if (rep->value) std::memcpy(rep->value, value.data(), sizeof(double) * cells);
            rep->total_cost_units = total_cost;
            rep->seed = seed;
            rep->wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

int mc_impl(bool matrix, const mlsk_model_desc* model, int32_t target, double tparam, int64_t L, int64_t N,
            int64_t M, int64_t c0, uint64_t seed, const mlsk_exec_opts* opts, mlsk_report* rep) {
    return guard([&] {
        const auto t0 = std::chrono::steady_clock::now();
        if (M < 2 || N < 1 || L < 0 || c0 < 1) invalid(matrix ? "mc_matmul: need M >= 2 and N >= 1"
                                                               : "mc_inner: need M >= 2 and N >= 1");
        check_target(target, tparam);
        if (!model) invalid("model: null descriptor");
        if (model_is_vector(model) == matrix) invalid("estimator: model kind does not match the estimator");
        Exec ex(opts);
        Runner R;
        R.wsp = &cached_workspace(ex.device);
        build_model(R.model, model, ex.stream);
        R.target = target;
        R.tparam = tparam;
        R.seed = seed;
        R.rank = ex.rank;
        R.world = ex.world;
        R.resolve_engine(ex.engine);
        const int64_t cells = R.model.rows * R.model.cols;
        const int64_t s = c0 * ipow(M, L);
        LevelState st;
        st.init(cells, ex.stream);
        R.run({{LevelSpec{MLSK_TAG_MC, s, 0}, 0, N, &st, nullptr}}, ex.stream, 0);
        std::vector<double> sum;
        double sq;
        read_level(st, ex.stream, sum, sq);
        if (rep) {
            for (int64_t t = 0; t < cells; ++t) {
                if (rep->value) rep->value[t] = sum[t] / (double)N;  // estimators.cpp:219,265
                if (rep->level_sum) rep->level_sum[t] = sum[t];
                if (rep->level_estimate) rep->level_estimate[t] = sum[t] / (double)N;
            }
            if (rep->level_sumsq) rep->level_sumsq[0] = sq;
            if (rep->level_mean_sq) rep->level_mean_sq[0] = sq / (double)N;
            if (rep->level_count) rep->level_count[0] = st.count;
            if (rep->cost_units) rep->cost_units[0] = N * s * cells;
            rep->total_cost_units = N * s * cells;
            rep->seed = seed;
            rep->wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

int reference_impl(bool matrix, const mlsk_model_desc* model, int32_t target, double tparam, int64_t count,
                   uint64_t seed, const mlsk_exec_opts* opts, double* mean, double* se) {
    return guard([&] {
        if (count < 1) invalid(matrix ? "reference_matmul: count must be positive"
                                      : "reference_inner: count must be positive");
        check_target(target, tparam);
        if (!model) invalid("model: null descriptor");
        if (model_is_vector(model) == matrix) invalid("estimator: model kind does not match the estimator");
        Exec ex(opts);
        Runner R;
        R.wsp = &cached_workspace(ex.device);
        build_model(R.model, model, ex.stream);
        R.target = target;
        R.tparam = tparam;
        R.seed = seed;
        R.rank = 0;  // every rank computes the whole reference value
        R.world = 1;
        R.engine = MLSK_ENGINE_EXACT;
        const int64_t cells = R.model.rows * R.model.cols;
        LevelState st;
        st.init(cells, ex.stream);
        LevelSpec lv{0, R.model.desc.n, 0};  // key (seed, 0, k), models.cpp:152,193
        lv.full = true;
        R.run({{lv, 0, count, &st, nullptr}}, ex.stream, 0);
        std::vector<double> sum;
        double sq;
        read_level(st, ex.stream, sum, sq);
        const double cnt = (double)count;
        double mean_sq = 0.0;  // frobenius_norm_sq(mean) (tensor.cpp:141-147); inner: mean * mean
        std::vector<double> mv(cells);
        for (int64_t t = 0; t < cells; ++t) {
            mv[t] = sum[t] / cnt;
            mean_sq += mv[t] * mv[t];
        }
        double err = 0.0;
        if (count > 1) {
            const double var = matrix ? std::max(0.0, (sq - cnt * mean_sq) / (double)(count - 1))
                                      : std::max(0.0, (sq - cnt * mv[0] * mv[0]) / (double)(count - 1));
            err = std::sqrt(var / cnt);
        }
        if (mean) std::memcpy(mean, mv.data(), sizeof(double) * cells);
        if (se) *se = err;
    });
}

}  // namespace

int mlsk::run_guarded(const std::function<void()>& body) { return guard(body); }

namespace {
// packed[0..cells] = total (+ open), packed[cells] = sum of squares, packed[cells+1] = count
__global__ void k_pack_level(const double* __restrict__ total, const double* __restrict__ open, int64_t cells,
                             int has_open, double count, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= cells + 1;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i <= cells) out[i] = has_open ? __dadd_rn(total[i], open[i]) : total[i];
        else out[i] = count;
    }
}
}  // namespace

struct mlsk_session {
    std::unique_ptr<Exec> ex;
    Runner R;
    int64_t M, c0, L;
    std::vector<LevelState> levels;
    std::vector<int64_t> next_k;
    DevArray<double> packed;
    // multi-GPU session (mlsk_exec_opts.n_devices > 1 or deterministic): the
    // shards, each a one-device session, in the fixed order their sums are
    // added; shard_slot[i] = the device slot (host thread) that runs shard i
    std::vector<std::unique_ptr<mlsk_session>> shards;
    std::vector<int> shard_slot;
    int nslots = 0;
    bool multi() const { return !shards.empty(); }
};

namespace {

std::unique_ptr<mlsk_session> session_single(const mlsk_model_desc* model, int32_t target, double tp, int64_t M,
                                             int64_t c0, int64_t L, uint64_t seed, const mlsk_exec_opts* opts) {
    auto s = std::make_unique<mlsk_session>();
    s->ex = std::make_unique<Exec>(opts);
    build_model(s->R.model, model, s->ex->stream);
    s->R.target = target;
    s->R.tparam = tp;
    s->R.seed = seed;
    s->R.rank = s->ex->rank;
    s->R.world = s->ex->world;
    s->R.resolve_engine(s->ex->engine);
    s->M = M;
    s->c0 = c0;
    s->L = L;
    const int64_t cells = s->R.model.rows * s->R.model.cols;
    s->levels.resize(L + 1);
    for (auto& st : s->levels) st.init(cells, s->ex->stream);
    s->next_k.assign(L + 1, 0);
    s->packed.alloc((size_t)(L + 1) * (cells + 2));
    s->packed.zero(s->ex->stream);
    return s;
}

// A multi-GPU session: one single-device session per shard.  Plain mode:
// shard i = device slot i, chunk sharding rank' = rank * n + i of world * n.
// Deterministic mode: shard v = virtual shard v (rank' = v, world' = vshards)
// on slot v mod n; shards are summed in v order, so the result does not
// depend on n.
std::unique_ptr<mlsk_session> session_multi(const mlsk_model_desc* model, int32_t target, double tp, int64_t M,
                                            int64_t c0, int64_t L, uint64_t seed, const mlsk_exec_opts* opts) {
    std::vector<int> slots;
    bool det;
    int vsh;
    Exec::multi_of(opts, slots, det, vsh);
    if (opts->probe_k > 0) invalid("exec: the coupling probe needs a single device");
    const int n = (int)slots.size();
    const int world = opts->world <= 0 ? 1 : opts->world;
    mlsk_exec_opts home = *opts;
    home.n_devices = 0;
    home.device_ids = nullptr;
    home.deterministic = 0;
    home.device = slots[0];
    home.stream = nullptr;  // every shard runs on its device's library stream
    auto s = session_single(model, target, tp, M, c0, L, seed, &home);  // shape, packed buffer
    s->nslots = n;
    const int nshards = det ? vsh : n;
    for (int i = 0; i < nshards; ++i) {
        mlsk_exec_opts so = home;
        so.device = slots[i % n];
        so.rank = det ? i : opts->rank * n + i;
        so.world = det ? vsh : world * n;
        s->shards.push_back(session_single(model, target, tp, M, c0, L, seed, &so));
        s->shard_slot.push_back(i % n);
    }
    return s;
}

// run `f(shard)` for every shard: one host thread per device slot, each
// running its shards in order; the first error is rethrown
void for_shards(mlsk_session* s, const std::function<void(mlsk_session*)>& f) {
    std::vector<std::thread> pool;
    std::vector<std::string> err(s->nslots);
    std::vector<int> code(s->nslots, MLSK_OK);
    for (int slot = 0; slot < s->nslots; ++slot) {
        pool.emplace_back([&, slot] {
            try {
                for (size_t i = 0; i < s->shards.size(); ++i)
                    if (s->shard_slot[i] == slot) {
                        MLSK_CUDA(cudaSetDevice(s->shards[i]->ex->device));
                        f(s->shards[i].get());
                    }
            } catch (const Error& e) {
                err[slot] = e.what();
                code[slot] = e.code;
            } catch (const std::exception& e) {
                err[slot] = e.what();
                code[slot] = MLSK_ERUNTIME;
            }
        });
    }
    for (auto& t : pool) t.join();
    for (int slot = 0; slot < s->nslots; ++slot)
        if (code[slot] != MLSK_OK) throw Error(code[slot], err[slot]);
}

// the shards' level sums / sums of squares / counts added in shard order
void multi_levels(mlsk_session* s, std::vector<std::vector<double>>& sums, std::vector<double>& sqs,
                  std::vector<int64_t>& counts) {
    const int64_t cells = s->R.model.rows * s->R.model.cols;
    sums.assign(s->L + 1, std::vector<double>(cells, 0.0));
    sqs.assign(s->L + 1, 0.0);
    counts.assign(s->L + 1, 0);
    for (auto& sh : s->shards) {
        MLSK_CUDA(cudaSetDevice(sh->ex->device));
        std::vector<const double*> ps;
        std::vector<double> pq;
        read_levels(sh->levels, sh->ex->stream, *sh->R.wsp, ps, pq);
        for (int64_t l = 0; l <= s->L; ++l) {
            for (int64_t t = 0; t < cells; ++t) sums[l][t] += ps[l][t];
            sqs[l] += pq[l];
            counts[l] += sh->levels[l].count;
        }
    }
}

}  // namespace

extern "C" {

int mlsk_mlmc_inner(const mlsk_model_desc* model, int32_t target, double tp, const mlsk_plan* plan,
                    uint64_t seed, const mlsk_exec_opts* opts, mlsk_report* report) {
    return mlmc_impl(false, model, target, tp, plan, seed, opts, report);
}

int mlsk_mlmc_matmul(const mlsk_model_desc* model, int32_t target, double tp, const mlsk_plan* plan,
                     uint64_t seed, const mlsk_exec_opts* opts, mlsk_report* report) {
    return mlmc_impl(true, model, target, tp, plan, seed, opts, report);
}

int mlsk_mc_inner(const mlsk_model_desc* model, int32_t target, double tp, int64_t L, int64_t N, int64_t M,
                  int64_t c0, uint64_t seed, const mlsk_exec_opts* opts, mlsk_report* report) {
    return mc_impl(false, model, target, tp, L, N, M, c0, seed, opts, report);
}

int mlsk_mc_matmul(const mlsk_model_desc* model, int32_t target, double tp, int64_t L, int64_t N, int64_t M,
                   int64_t c0, uint64_t seed, const mlsk_exec_opts* opts, mlsk_report* report) {
    return mc_impl(true, model, target, tp, L, N, M, c0, seed, opts, report);
}

int mlsk_reference_inner(const mlsk_model_desc* model, int32_t target, double tp, int64_t count, uint64_t seed,
                         const mlsk_exec_opts* opts, double* mean, double* std_error) {
    return reference_impl(false, model, target, tp, count, seed, opts, mean, std_error);
}

int mlsk_reference_matmul(const mlsk_model_desc* model, int32_t target, double tp, int64_t count, uint64_t seed,
                          const mlsk_exec_opts* opts, double* mean, double* std_error) {
    return reference_impl(true, model, target, tp, count, seed, opts, mean, std_error);
}

int mlsk_session_create(const mlsk_model_desc* model, int32_t target, double tp, int64_t M, int64_t c0, int64_t L,
                        uint64_t seed, const mlsk_exec_opts* opts, mlsk_session** out) {
    return guard([&] {
        if (!out) invalid("session: null output pointer");
        if (M < 2 || L < 0 || c0 < 1) invalid("estimator: malformed plan");
        check_target(target, tp);
        if (!model) invalid("model: null descriptor");
        const bool multi = opts && (opts->n_devices > 1 || opts->deterministic);
        auto s = multi ? session_multi(model, target, tp, M, c0, L, seed, opts)
                       : session_single(model, target, tp, M, c0, L, seed, opts);
        *out = s.release();
    });
}

int mlsk_session_run_round(mlsk_session* s, const int64_t* dN) {
    return guard([&] {
        if (!s || !dN) invalid("session: null argument");
        for (int64_t l = 0; l <= s->L; ++l)
            if (dN[l] < 0) invalid("session: dN must be non-negative");
        MLSK_CUDA(cudaSetDevice(s->ex->device));
        std::vector<Runner::Item> items;
        for (int64_t l = 0; l <= s->L; ++l) {
            if (dN[l] == 0) continue;
            const int64_t fine = s->c0 * ipow(s->M, l), coarse = l > 0 ? fine / s->M : 0;
            items.push_back({LevelSpec{(uint64_t)l, fine, coarse}, s->next_k[l], s->next_k[l] + dN[l], &s->levels[l],
                             nullptr});
            s->next_k[l] += dN[l];
        }
        if (s->multi()) {
            // every shard runs the round's replication ranges (its chunks of them)
            for_shards(s, [&](mlsk_session* sh) {
                std::vector<Runner::Item> its;
                for (const auto& it : items) {
                    const int64_t l = (int64_t)it.lv.tag;
                    its.push_back({it.lv, it.k0, it.k1, &sh->levels[l], nullptr});
                }
                sh->R.run(its, sh->ex->stream, 0);
                MLSK_CUDA(cudaStreamSynchronize(sh->ex->stream));
            });
            return;
        }
        s->R.run(items, s->ex->stream, 0);
        // without a caller stream the call is synchronous; with one, the round is
        // ordered on that stream and the call returns once it is enqueued
        if (s->ex->owns) MLSK_CUDA(cudaStreamSynchronize(s->ex->stream));
    });
}

int mlsk_session_stats(mlsk_session* s, mlsk_report* rep) {
    return guard([&] {
        if (!s || !rep) invalid("session: null argument");
        MLSK_CUDA(cudaSetDevice(s->ex->device));
        const int64_t cells = s->R.model.rows * s->R.model.cols;
        std::vector<double> value(cells, 0.0);
        int64_t total_cost = 0;
        std::vector<const double*> sums;
        std::vector<double> sqs;
        std::vector<std::vector<double>> msums;
        std::vector<int64_t> mcounts;
        if (s->multi()) {
            multi_levels(s, msums, sqs, mcounts);
            for (auto& v : msums) sums.push_back(v.data());
        } else {
            read_levels(s->levels, s->ex->stream, *s->R.wsp, sums, sqs);
        }
        for (int64_t l = 0; l <= s->L; ++l) {
            const double* sum = sums[l];
            const double sq = sqs[l];
            const int64_t n = s->multi() ? mcounts[l] : s->levels[l].count;
            const int64_t fine = s->c0 * ipow(s->M, l), coarse = l > 0 ? fine / s->M : 0;
            const double inv_n = n > 0 ? 1.0 / (double)n : 0.0;
            const int64_t cost = n * (fine + coarse) * cells;
            total_cost += cost;
            if (rep->level_sum) std::memcpy(rep->level_sum + l * cells, sum, sizeof(double) * cells);
            if (rep->level_estimate)
                for (int64_t t = 0; t < cells; ++t) rep->level_estimate[l * cells + t] = sum[t] * inv_n;
            for (int64_t t = 0; t < cells; ++t) value[t] += sum[t] * inv_n;
            if (rep->level_sumsq) rep->level_sumsq[l] = sq;
            if (rep->level_mean_sq) rep->level_mean_sq[l] = sq * inv_n;
            if (rep->level_count) rep->level_count[l] = n;
            if (rep->cost_units) rep->cost_units[l] = cost;
        }
        if (rep->value) std::memcpy(rep->value, value.data(), sizeof(double) * cells);
        rep->total_cost_units = total_cost;
        rep->seed = s->R.seed;
    });
}

int mlsk_session_level_buffer(mlsk_session* s, void** device_ptr, int64_t* n_doubles) {
    return guard([&] {
        if (!s || !device_ptr || !n_doubles) invalid("session: null argument");
        MLSK_CUDA(cudaSetDevice(s->ex->device));
        const int64_t cells = s->R.model.rows * s->R.model.cols;
        if (s->multi()) {
            // the shards' sums (added on the host in shard order) into the home device's buffer
            std::vector<std::vector<double>> ms;
            std::vector<double> mq;
            std::vector<int64_t> mc;
            multi_levels(s, ms, mq, mc);
            std::vector<double> h((size_t)(s->L + 1) * (cells + 2));
            for (int64_t l = 0; l <= s->L; ++l) {
                std::memcpy(h.data() + l * (cells + 2), ms[l].data(), sizeof(double) * cells);
                h[l * (cells + 2) + cells] = mq[l];
                h[l * (cells + 2) + cells + 1] = (double)mc[l];
            }
            MLSK_CUDA(cudaSetDevice(s->ex->device));
            MLSK_CUDA(cudaMemcpy(s->packed.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
            *device_ptr = s->packed.p;
            *n_doubles = (int64_t)h.size();
            return;
        }
        // pack [(sum Y, sum ||Y||^2, count)] per level on the device (sum includes the open chunk)
        for (int64_t l = 0; l <= s->L; ++l) {
            const LevelState& st = s->levels[l];
            k_pack_level<<<(int)std::min<int64_t>((cells + 256) / 256, 1184), 256, 0, s->ex->stream>>>(
                st.total(), st.open(), cells, st.open_count > 0 ? 1 : 0, (double)st.count,
                s->packed.p + l * (cells + 2));
            launched();
        }
        // library-owned stream: nothing outside the library can order itself
        // after the pack, so the buffer is complete when the call returns.  With
        // a caller stream the pack is ordered on that stream (the caller's
        // collective must run on it or wait on it).
        if (s->ex->owns) MLSK_CUDA(cudaStreamSynchronize(s->ex->stream));
        *device_ptr = s->packed.p;
        *n_doubles = (int64_t)(s->L + 1) * (cells + 2);
    });
}

// ---- checkpoint / resume ---------------------------------------------------
// A session's state is its per-level accumulators and replication counters:
// per level the device buffer [total | total_sq | open chunk | open_sq] and
// (count, open_count, open_chunk), plus the next replication index of every
// level.  The image is plain host bytes (little-endian PODs): a header that
// identifies the run (plan shape, seed, target, model scalars, sharding), then
// next_k[L+1], then for every accumulator unit (the session itself, or each
// shard of a multi-device session in shard order) its levels.  Restoring into
// a session created with the same arguments and continuing gives the same bits
// as a run that never stopped.
namespace {

constexpr uint64_t kCkptMagic = 0x31504B43534B4C4DULL;  // "MLSKCKP1"

struct CkptHeader {
    uint64_t magic, version;
    int64_t M, c0, L, cells, units;
    uint64_t seed;
    int32_t target, kind, dtype, stream_mode;
    double tparam;
    int64_t m, n, p, rff_dim;
    uint64_t data_seed;
    double sd, mean_lo, mean_hi, nu, sigma;
    int64_t rank, world, host_means;
};

std::vector<mlsk_session*> ckpt_units(mlsk_session* s) {
    std::vector<mlsk_session*> u;
    if (s->multi())
        for (auto& sh : s->shards) u.push_back(sh.get());
    else
        u.push_back(s);
    return u;
}

CkptHeader ckpt_header(mlsk_session* s) {
    CkptHeader h{};
    const mlsk_model_desc& d = s->R.model.desc;
    h.magic = kCkptMagic;
    h.version = 1;
    h.M = s->M;
    h.c0 = s->c0;
    h.L = s->L;
    h.cells = s->R.model.rows * s->R.model.cols;
    h.units = (int64_t)ckpt_units(s).size();
    h.seed = s->R.seed;
    h.target = s->R.target;
    h.tparam = s->R.tparam;
    h.kind = d.kind;
    h.dtype = d.dtype;
    h.stream_mode = d.stream_mode;
    h.m = d.m;
    h.n = d.n;
    h.p = d.p;
    h.rff_dim = d.rff_dim;
    h.data_seed = d.data_seed;
    h.sd = d.sd;
    h.mean_lo = d.mean_lo;
    h.mean_hi = d.mean_hi;
    h.nu = d.nu;
    h.sigma = d.sigma;
    h.rank = s->R.rank;
    h.world = s->R.world;
    h.host_means = (d.mean_a || d.mean_b) ? 1 : 0;
    return h;
}

int64_t ckpt_bytes(mlsk_session* s) {
    const CkptHeader h = ckpt_header(s);
    const int64_t per_level = 3 * (int64_t)sizeof(int64_t) + (2 * h.cells + 2) * (int64_t)sizeof(double);
    return (int64_t)sizeof(CkptHeader) + (h.L + 1) * (int64_t)sizeof(int64_t) + h.units * (h.L + 1) * per_level;
}

}  // namespace

int mlsk_session_checkpoint(mlsk_session* s, void* buf, int64_t* bytes) {
    return guard([&] {
        if (!s || !bytes) invalid("session: null argument");
        const int64_t need = ckpt_bytes(s);
        if (!buf) {  // size query
            *bytes = need;
            return;
        }
        if (*bytes < need) invalid("session_checkpoint: buffer too small");
        const CkptHeader h = ckpt_header(s);
        unsigned char* o = static_cast<unsigned char*>(buf);
        std::memcpy(o, &h, sizeof h);
        o += sizeof h;
        std::memcpy(o, s->next_k.data(), sizeof(int64_t) * (h.L + 1));
        o += sizeof(int64_t) * (h.L + 1);
        for (mlsk_session* u : ckpt_units(s)) {
            MLSK_CUDA(cudaSetDevice(u->ex->device));
            for (const LevelState& st : u->levels) {
                const int64_t meta[3] = {st.count, st.open_count, st.open_chunk};
                std::memcpy(o, meta, sizeof meta);
                o += sizeof meta;
                MLSK_CUDA(cudaMemcpyAsync(o, st.buf.p, sizeof(double) * (2 * h.cells + 2), cudaMemcpyDeviceToHost,
                                          u->ex->stream));
                o += sizeof(double) * (2 * h.cells + 2);
            }
            MLSK_CUDA(cudaStreamSynchronize(u->ex->stream));
        }
        MLSK_CUDA(cudaSetDevice(s->ex->device));
        *bytes = need;
    });
}

int mlsk_session_restore(mlsk_session* s, const void* buf, int64_t bytes) {
    return guard([&] {
        if (!s || !buf) invalid("session: null argument");
        const CkptHeader mine = ckpt_header(s);
        if (bytes < (int64_t)sizeof(CkptHeader)) invalid("session_restore: not a session checkpoint");
        CkptHeader h;
        std::memcpy(&h, buf, sizeof h);
        if (h.magic != kCkptMagic || h.version != 1) invalid("session_restore: not a session checkpoint");
        // the run must be the same: plan shape, seed, target, model and sharding
        if (h.M != mine.M || h.c0 != mine.c0 || h.L != mine.L || h.cells != mine.cells || h.units != mine.units ||
            h.seed != mine.seed || h.target != mine.target || h.tparam != mine.tparam || h.kind != mine.kind ||
            h.dtype != mine.dtype || h.stream_mode != mine.stream_mode || h.m != mine.m || h.n != mine.n ||
            h.p != mine.p || h.rff_dim != mine.rff_dim || h.data_seed != mine.data_seed || h.sd != mine.sd ||
            h.mean_lo != mine.mean_lo || h.mean_hi != mine.mean_hi || h.nu != mine.nu || h.sigma != mine.sigma ||
            h.rank != mine.rank || h.world != mine.world || h.host_means != mine.host_means)
            invalid("session_restore: the checkpoint belongs to a different run (model, plan, seed, target or "
                    "sharding differ)");
        if (bytes < ckpt_bytes(s)) invalid("session_restore: truncated checkpoint");
        const unsigned char* i = static_cast<const unsigned char*>(buf) + sizeof h;
        std::vector<int64_t> nk(h.L + 1);
        std::memcpy(nk.data(), i, sizeof(int64_t) * (h.L + 1));
        i += sizeof(int64_t) * (h.L + 1);
        for (int64_t l = 0; l <= h.L; ++l)
            if (nk[l] < 0) invalid("session_restore: corrupt checkpoint");
        for (mlsk_session* u : ckpt_units(s)) {
            MLSK_CUDA(cudaSetDevice(u->ex->device));
            for (LevelState& st : u->levels) {
                int64_t meta[3];
                std::memcpy(meta, i, sizeof meta);
                i += sizeof meta;
                if (meta[0] < 0 || meta[1] < 0 || meta[1] > 64 || meta[2] < -1)
                    invalid("session_restore: corrupt checkpoint");
                st.count = meta[0];
                st.open_count = meta[1];
                st.open_chunk = meta[2];
                MLSK_CUDA(cudaMemcpyAsync(st.buf.p, i, sizeof(double) * (2 * h.cells + 2), cudaMemcpyHostToDevice,
                                          u->ex->stream));
                i += sizeof(double) * (2 * h.cells + 2);
            }
            MLSK_CUDA(cudaStreamSynchronize(u->ex->stream));
        }
        MLSK_CUDA(cudaSetDevice(s->ex->device));
        s->next_k = nk;
    });
}

int mlsk_session_synchronize(mlsk_session* s) {
    return guard([&] {
        if (!s) invalid("session: null argument");
        for (auto& sh : s->shards) {
            MLSK_CUDA(cudaSetDevice(sh->ex->device));
            MLSK_CUDA(cudaStreamSynchronize(sh->ex->stream));
        }
        MLSK_CUDA(cudaSetDevice(s->ex->device));
        MLSK_CUDA(cudaStreamSynchronize(s->ex->stream));
    });
}

int mlsk_session_destroy(mlsk_session* s) {
    return guard([&] {
        if (!s) return;
        for (auto& sh : s->shards) {
            cudaSetDevice(sh->ex->device);
            cudaStreamSynchronize(sh->ex->stream);
        }
        cudaSetDevice(s->ex->device);
        cudaStreamSynchronize(s->ex->stream);
        delete s;
    });
}

int mlsk_draw_sample(const mlsk_model_desc* model, uint64_t seed, uint64_t tag, int64_t k, int64_t c,
                     uint32_t* indices, double* a_cols, double* b_rows) {
    return guard([&] {
        if (c <= 0) invalid("draw_realization: size must be positive");
        Exec ex(nullptr);
        Model M;
        build_model(M, model, ex.stream);
        Workspace ws;
        exact_gather_sample(M, seed, tag, k, c, indices, a_cols, b_rows, ex.stream, ws);
    });
}

int mlsk_model_data(const mlsk_model_desc* model, int32_t which, void* out, int64_t* count) {
    return guard([&] {
        if (!count) invalid("model_data: null count");
        Exec ex(nullptr);
        Model M;
        build_model(M, model, ex.stream);
        const void* src = nullptr;
        size_t elem = 8, n = 0;
        const bool f32 = M.dm.dtype == MLSK_F32;
        if (M.dm.kind == MLSK_MODEL_GAUSS_MEAN) {
            if (which == 0) { src = f32 ? (const void*)M.mean_a_f.p : (const void*)M.mean_a.p; n = f32 ? M.mean_a_f.n : M.mean_a.n; }
            if (which == 1) { src = f32 ? (const void*)M.mean_b_f.p : (const void*)M.mean_b.p; n = f32 ? M.mean_b_f.n : M.mean_b.n; }
            elem = f32 ? 4 : 8;
        } else if (M.dm.kind == MLSK_MODEL_RFF) {
            elem = 4;
            if (which == 0) { src = M.rff_x.p; n = M.rff_x.n; }
            if (which == 1) { src = M.rff_w.p; n = M.rff_w.n; }
            if (which == 2) { src = M.rff_b.p; n = M.rff_b.n; }
        }
        if (!src) invalid("model_data: this model has no such stored data");
        if (out) {
            if ((size_t)*count < n) invalid("model_data: output buffer too small");
            MLSK_CUDA(cudaMemcpyAsync(out, src, n * elem, cudaMemcpyDeviceToHost, ex.stream));
            MLSK_CUDA(cudaStreamSynchronize(ex.stream));
        }
        *count = (int64_t)n;
    });
}

uint64_t mlsk_derive_seed(uint64_t master, uint64_t a, uint64_t b) { return derive_seed(master, a, b); }

const char* mlsk_last_error(void) { return g_last_error.c_str(); }

const char* mlsk_version(void) { return MLSK_VERSION_STRING; }

int mlsk_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int64_t mlsk_kernel_launch_count(void) { return g_launches; }

int mlsk_contraction_columns(int64_t out[2], int reset) {
    if (out) {
        out[0] = g_columns[0];
        out[1] = g_columns[1];
    }
    if (reset) g_columns[0] = g_columns[1] = 0;
    return MLSK_OK;
}

}  // extern "C"
