/*
 * mlsk.h -- C-ABI of the B200-native MLMC sampled-product level estimator.
 *
 * Drop-in boundary for the hot path of the reference library `mlsketch`
 * (/root/reference/proj).  Every entry point below replaces one reference
 * interface; the citation is given beside it.  Only plain C types cross the
 * boundary: host pointers + sizes in, caller-allocated host report buffers out.
 * Device memory, streams and kernels are owned by the library
 * (paper_1904_00429_b200/csrc); there is no CPU fallback -- if no CUDA device
 * is usable every compute entry point returns MLSK_ERUNTIME.
 *
 * Error behaviour mirrors the reference: conditions under which the
 * reference throws std::invalid_argument (malformed plan, N_l < 1, M < 2,
 * bad dimensions, out-of-range indices, empty realizations, NaN inputs)
 * return MLSK_EINVAL (the CLI's exit code 1, mlsketch_main.cpp:415-417);
 * CUDA/NCCL/runtime failures return MLSK_ERUNTIME (exit code 3).  The message
 * of the last failure on the calling thread is returned by mlsk_last_error().
 */
#ifndef MLSK_H
#define MLSK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLSK_VERSION_STRING "mlsk-b200 0.1.0"

/* status codes */
#define MLSK_OK 0
#define MLSK_EINVAL 1   /* std::invalid_argument in the reference */
#define MLSK_ERUNTIME 3 /* CUDA / NCCL / allocation failure */

/* model kinds -- the reference's std::function draw plugins
 * (models.hpp:17-31) become device-side descriptors. */
#define MLSK_MODEL_CONSTANT_ONES 1  /* models.cpp:54-74  a=b=1 / A=B=1            */
#define MLSK_MODEL_DETERMINISTIC 2  /* models.cpp:76-97  a_j=j, b_j=n+j / 2x2 pair */
#define MLSK_MODEL_PAPER_INNER 3    /* models.cpp:12-27  n=1000 paper sec. 4.1     */
#define MLSK_MODEL_PAPER_MATRIX 4   /* models.cpp:29-52  10x1000x10 paper sec. 4.2 */
#define MLSK_MODEL_GAUSS_MEAN 5     /* configs 1-3: entry = mean + sd*N(0,1)        */
#define MLSK_MODEL_RFF 6            /* config 4: z_k(x) = sqrt2 cos(w_k.x + b_k)    */
#define MLSK_MODEL_STUDENT_T 7      /* config 5: entry = mean + t_nu                */

/* arithmetic type of the path */
#define MLSK_F64 0
#define MLSK_F32 1

/* stream definitions */
#define MLSK_STREAM_PHILOX 0 /* counter-based Philox4x32-10, keyed (seed, l, k) */
#define MLSK_STREAM_REF 1    /* the reference's mt19937_64 substreams (rng.hpp)  */

/* target functions (models.cpp:99-117) */
#define MLSK_TARGET_IDENTITY 0
#define MLSK_TARGET_F1 1 /* |x| H(x-10)                 */
#define MLSK_TARGET_F2 2 /* x^2 sin(1/(|x|+zeta)), zeta = target_param */

/* execution engines */
#define MLSK_ENGINE_AUTO 0  /* fused tensor-core engine when applicable, else exact */
#define MLSK_ENGINE_EXACT 1 /* reference arithmetic order, bit-exact given the draws */
#define MLSK_ENGINE_FUSED 2 /* DMMA / tcgen05 sampled GEMM with fused level epilogue */

/*
 * Model descriptor.  Vector models (mlmc_inner) use n only.  Fixed model data
 * (means, RFF weights) is generated on the device from data_seed unless the
 * caller passes host arrays in mean_a / mean_b (row-major, dtype as `dtype`).
 */
typedef struct mlsk_model_desc {
    int32_t kind;        /* MLSK_MODEL_* */
    int32_t dtype;       /* MLSK_F64 / MLSK_F32 */
    int32_t stream_mode; /* MLSK_STREAM_* */
    int32_t reserved0;
    int64_t m, n, p;     /* A is m x n, B is n x p (reference `d` == p) */
    uint64_t data_seed;  /* seed of the fixed-from-seed data */
    double sd;           /* noise standard deviation (gauss_mean) */
    double mean_lo;      /* generated means ~ U(mean_lo, mean_hi) */
    double mean_hi;
    double nu;           /* Student-t degrees of freedom */
    double sigma;        /* RFF kernel bandwidth */
    int64_t rff_dim;     /* RFF input dimension D */
    const void* mean_a;  /* optional host means of a / A (len n or m*n) */
    const void* mean_b;  /* optional host means of b / B (len n or n*p) */
} mlsk_model_desc;

/*
 * Level plan: c_l = c0 * M^l sampled indices at level l, coarse level = the
 * first c_l / M of them.  The reference is c0 = 1 (estimators.cpp:57-58,121).
 * N points at L+1 replication counts (planner.hpp:12-20 LevelPlan::N).
 */
typedef struct mlsk_plan {
    int64_t M;
    int64_t c0;
    int64_t L;
    const int64_t* N;
} mlsk_plan;

/* Execution options (EstimatorOptions, estimators.hpp:45-50). */
typedef struct mlsk_exec_opts {
    int32_t device;      /* CUDA ordinal, -1 = current device */
    int32_t engine;      /* MLSK_ENGINE_* */
    void* stream;        /* cudaStream_t to order the work on; NULL = a library stream
                            and every call returns only when its work is done.  With
                            a caller stream, mlsk_session_run_round returns once the
                            round is enqueued (results ordered on that stream); a
                            round whose deep levels run on merged sampled columns
                            (mlsk_contraction_columns) waits once for a small device
                            pre-pass before it enqueues the rest (MLSK_MERGE=0: never). */
    int32_t rank;        /* sample sharding: 64-sample chunk q runs on rank q % world */
    int32_t world;       /* 1 for a single GPU */
    int64_t probe_k;     /* coupling probe: dump index sets of the first probe_k
                            replications of every level >= 1 (estimators.hpp:38-48) */
    uint32_t* probe_out; /* host [(L+1)][probe_k][c_L] 1-based indices, row l holds c_l */
    /* Multi-GPU inside one call (the reference parallelises inside the library,
     * parallel.hpp:18-52).  n_devices > 1: the replications are dealt to
     * n_devices device slots (device_ids[i], NULL = 0 .. n_devices-1; an ordinal
     * may repeat), one host thread per slot; slot i of this process is shard
     * rank * n_devices + i of world * n_devices.  The per-level sums of the
     * slots are added on the host in slot order.  Estimators and sessions only
     * (mc_* / reference_* run on the first device). */
    int32_t n_devices;         /* 0 or 1: one device (`device`) */
    const int32_t* device_ids;
    /* deterministic = 1: the samples go to `vshards` fixed virtual shards
     * (chunk q -> shard q mod vshards), each accumulated on its own and added
     * in shard order, so results are bit-identical for every n_devices that
     * divides vshards (the reference's thread-count invariance,
     * README.md:109-119).  Needs world == 1 (across processes: the Python
     * driver's ShardedSession). */
    int32_t deterministic;
    int32_t vshards;           /* 0: 8 */
} mlsk_exec_opts;

/*
 * Report (EstimateReport / LevelStatistic, estimators.hpp:20-36).  All
 * pointers are caller-allocated host buffers and may be NULL when not wanted.
 * `cells` = m*p (1 for the inner-product estimators).
 */
typedef struct mlsk_report {
    double* value;           /* [cells]           sum_l estimate_l                 */
    double* level_estimate;  /* [(L+1)*cells]     sum_l * (1/N_l)                  */
    double* level_sum;       /* [(L+1)*cells]     raw sum of Y over replications   */
    double* level_sumsq;     /* [L+1]             raw sum of ||Y||_F^2             */
    double* level_mean_sq;   /* [L+1]             sample_mean_of_squares           */
    int64_t* level_count;    /* [L+1]             replication_count                */
    int64_t* cost_units;     /* [L+1]             N_l (c_l + c_{l-1}) cells        */
    int64_t total_cost_units;
    double wall_time_s;
    uint64_t seed;
} mlsk_report;

/* ---- estimators (estimators.hpp:58-80) ---------------------------------- */

/* mlmc_inner(model, f, plan, seed, options)  estimators.cpp:44-103 */
int mlsk_mlmc_inner(const mlsk_model_desc* model, int32_t target, double target_param,
                    const mlsk_plan* plan, uint64_t seed, const mlsk_exec_opts* opts,
                    mlsk_report* report);

/* mlmc_matmul(model, f, plan, seed, options)  estimators.cpp:105-187 */
int mlsk_mlmc_matmul(const mlsk_model_desc* model, int32_t target, double target_param,
                     const mlsk_plan* plan, uint64_t seed, const mlsk_exec_opts* opts,
                     mlsk_report* report);

/* mc_inner(model, f, L, N, M, seed, options)  estimators.cpp:189-226
 * (sample size c0 * M^L; c0 = 1 is the reference) */
int mlsk_mc_inner(const mlsk_model_desc* model, int32_t target, double target_param,
                  int64_t L, int64_t N, int64_t M, int64_t c0, uint64_t seed,
                  const mlsk_exec_opts* opts, mlsk_report* report);

/* mc_matmul(model, f, L, N, M, seed, options)  estimators.cpp:228-275 */
int mlsk_mc_matmul(const mlsk_model_desc* model, int32_t target, double target_param,
                   int64_t L, int64_t N, int64_t M, int64_t c0, uint64_t seed,
                   const mlsk_exec_opts* opts, mlsk_report* report);

/* reference_inner(model, f, count, seed, threads)  models.cpp:140-175 and
 * reference_matmul(...)  models.cpp:177-227: the MC reference value -- count
 * full draws keyed (seed, 0, k), the exact product of each (tensor.cpp:97-131,
 * columns in order, no sampling), f per entry, 64-replication chunk sums.
 * mean[cells] = sum / count; *std_error = sqrt(max(0, (sq - count*|mean|^2) /
 * (count - 1)) / count) (0 when count == 1).  Always the exact engine. */
int mlsk_reference_inner(const mlsk_model_desc* model, int32_t target, double target_param,
                         int64_t count, uint64_t seed, const mlsk_exec_opts* opts,
                         double* mean, double* std_error);
int mlsk_reference_matmul(const mlsk_model_desc* model, int32_t target, double target_param,
                          int64_t count, uint64_t seed, const mlsk_exec_opts* opts,
                          double* mean, double* std_error);

/* ---- round API for adaptive MLMC --------------- */

typedef struct mlsk_session mlsk_session;

int mlsk_session_create(const mlsk_model_desc* model, int32_t target, double target_param,
                        int64_t M, int64_t c0, int64_t L, uint64_t seed,
                        const mlsk_exec_opts* opts, mlsk_session** out);
/* Run dN[l] more replications of every level l (continuing the replication
 * index k where the previous round stopped). */
int mlsk_session_run_round(mlsk_session* s, const int64_t* dN);
/* Fill `report` from the accumulated sums (estimate = sum * (1/count)). */
int mlsk_session_stats(mlsk_session* s, mlsk_report* report);
/* Packed per-level device buffer [(L+1)][cells + 2] = (sum Y, sum ||Y||^2,
 * count) in fp64, for an in-place NCCL all-reduce across ranks. */
int mlsk_session_level_buffer(mlsk_session* s, void** device_ptr, int64_t* n_doubles);
/* Checkpoint / resume: the session's accumulators and
 * replication counters as host bytes.  buf = NULL: *bytes = the size needed.
 * Restore into a session created with the same model, target, plan shape,
 * seed and sharding (else MLSK_EINVAL); continuing it then gives the same bits
 * as an uninterrupted run. */
int mlsk_session_checkpoint(mlsk_session* s, void* buf, int64_t* bytes);
int mlsk_session_restore(mlsk_session* s, const void* buf, int64_t bytes);
int mlsk_session_synchronize(mlsk_session* s);
int mlsk_session_destroy(mlsk_session* s);

/* ---- reference-function analogues on the device (for known-answer tests) --- */

/* sketch_inner(a, b, indices, dist)  sketch.cpp:22-38.  inv_probs NULL = uniform (n). */
int mlsk_sketch_inner(const double* a, const double* b, int64_t n, const uint32_t* indices,
                      int64_t s, const double* inv_probs, double* out);

/* sketch_matmul(A, B, indices, dist)  sketch.cpp:45-77.  A m x n, B n x d row-major. */
int mlsk_sketch_matmul(const double* A, const double* B, int64_t m, int64_t n, int64_t d,
                       const uint32_t* indices, int64_t s, const double* inv_probs,
                       double* out);

/* One level-sample's draw (model.draw + draw_realization, estimators.cpp:134-136):
 * the c sampled indices (1-based) and the gathered data a_S (rows x c) and
 * b_S (c x cols) for replication k of stream tag `tag` (level l, or 0xFFFFFFFF
 * for the MC baseline).  Any output pointer may be NULL. */
int mlsk_draw_sample(const mlsk_model_desc* model, uint64_t seed, uint64_t tag, int64_t k,
                     int64_t c, uint32_t* indices, double* a_cols, double* b_rows);

/* Fixed model data as generated on the device (for ground truth): which = 0
 * means of A / a (RFF: points X, m x D), 1 means of B / b (RFF: W, D x n),
 * 2 RFF phases.  With out == NULL only *count is set; else *count values of
 * the model dtype are copied to out. */
int mlsk_model_data(const mlsk_model_desc* model, int32_t which, void* out, int64_t* count);

/* RngStream::derive_seed (rng.hpp:31-37) -- pure host arithmetic. */
uint64_t mlsk_derive_seed(uint64_t master, uint64_t a, uint64_t b);

/* ---- misc ----------------------------------------------------------------- */
const char* mlsk_last_error(void);
const char* mlsk_version(void);
int mlsk_device_count(void);
/* Number of kernels this thread's library calls have launched so far. */
int64_t mlsk_kernel_launch_count(void);

/* ---- measurement (bench.py) ----------------------------------------------- */
/* Per-kernel CUDA-event timing on the launching stream: enable, reset, then
 * read entry i (returns the number of entries): name, launches, total ms. */
int mlsk_profile_enable(int on);
int mlsk_profile_reset(void);
int mlsk_profile_read(int i, char* name, int name_len, int64_t* launches, double* ms);
/* Start / end (ms since the last reset) of profiled launch i; returns the count. */
int mlsk_profile_timeline(int i, char* name, int name_len, double* t0, double* t1);
/* Merged sampled columns (identity target, the deep levels -- c >= n / 16 or
 * so -- where it saves K-chunks: a
 * level-sample's contraction runs over its DISTINCT sampled columns with
 * summed weights -- a duplicated index gathers the same drawn column,
 * sketch.cpp:60-71 -- and columns whose fine and coarse weights cancel drop
 * out).  out[0] = K-columns the GEMMs of this thread's calls executed since
 * the last reset, out[1] = the sampled indices they stand for (sum of c_l over
 * the level-samples); reset != 0 clears both after the read. */
int mlsk_contraction_columns(int64_t out[2], int reset);
/* fp64 tensor-pipe (DMMA) throughput measured on the device, TFLOP/s. */
double mlsk_measure_fp64_peak(int device);
/* Dense TF32 tcgen05 throughput (M=128, N=n, one CTA per SM), TFLOP/s. */
double mlsk_measure_tf32_peak(int device, int n);
/* RNG roofline of the inner-product path: index-samples/s of its per-index
 * work alone (index draw, Philox + Box-Muller pair, mean gathers), config 1. */
double mlsk_measure_index_rate(int device);

#ifdef __cplusplus
}
#endif

#endif /* MLSK_H */
