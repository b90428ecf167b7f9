/*
 * mlsk_oracle.h -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker the CUDA product is
 * compared against; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product
 * (paper_1904_00429_b200) never links or calls it.
 *
 * It restates, in plain C, the reference's per-sample level estimator:
 *   rng.hpp:17-90        SplitMix64 derive, mt19937_64, uniform01/uniform_pos,
 *                        Box-Muller normal, exponential, poisson
 *   sampling.cpp:32-134  uniform distribution, cumulative table, sample, prefix
 *   sketch.cpp:22-77     sketch_inner / sketch_matmul arithmetic order
 *   models.cpp:12-117    built-in models and targets (draw order)
 *   estimators.cpp:44-275  mlmc_inner / mlmc_matmul / mc_inner / mc_matmul,
 *                        64-replication chunks, chunk-order reduction, 1/N
 *   parallel.hpp:18-55   (sequential: chunk order is the determinism contract)
 * plus the philox-mode stream of include/mlsk_stream_spec.h.
 *
 * Parity pins: the ref-stream mode is checked bit for bit against the
 * reference compiled from /root/reference (oracle/_ref and the JSON fixtures in tests/golden);
 * Philox4x32-10 is checked against libcudacxx's std::philox4x32 and the
 * C++26 10000th-value known answer (tests/golden/philox_kat.json).
 */
#ifndef MLSK_ORACLE_H
#define MLSK_ORACLE_H

#include <stdint.h>
#include "../include/mlsk.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp ------------------------------------------------------------- */
uint64_t orc_mix(uint64_t z);
uint64_t orc_derive_seed(uint64_t master, uint64_t a, uint64_t b);

typedef struct orc_ref_rng {
    uint64_t mt[312];
    int idx;
    int have_cached;
    double cached;
} orc_ref_rng;

void orc_ref_init(orc_ref_rng* r, uint64_t seed);
uint64_t orc_ref_next_u64(orc_ref_rng* r);
double orc_ref_uniform01(orc_ref_rng* r);
double orc_ref_uniform_pos(orc_ref_rng* r);
double orc_ref_normal(orc_ref_rng* r);
double orc_ref_exponential(orc_ref_rng* r);
long orc_ref_poisson(orc_ref_rng* r, double mean);
/* first `count` outputs of std::mt19937_64(seed) */
void orc_mt64_stream(uint64_t seed, int64_t count, uint64_t* out);

/* ---- philox-mode stream (include/mlsk_stream_spec.h) --------------------- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double orc_log_unit(double x);                 /* portable log on (0, 1] */
void orc_sincos_turn(double u, double* c, double* s); /* cos, sin of 2 pi u */
void orc_box_muller(uint64_t ua, uint64_t ub, double* z0, double* z1);
float orc_log_unit_f(float x);
void orc_sincos_turn_f(float u, float* c, float* s);
void orc_box_muller_f(uint32_t ua, uint32_t ub, float* z0, float* z1);

/* ---- sampling.cpp -------------------------------------------------------- */
void orc_uniform_cumulative(int64_t n, double* cum);
uint32_t orc_index_from_u64(uint64_t x, int64_t n, const double* cum);

/* ---- sketch.cpp ---------------------------------------------------------- */
/* return 0 ok, MLSK_EINVAL on bad indices / empty realization */
int orc_sketch_inner(const double* a, const double* b, int64_t n, const uint32_t* idx,
                     int64_t s, const double* inv_probs, double* out);
int orc_sketch_matmul(const double* A, const double* B, int64_t m, int64_t n, int64_t d,
                      const uint32_t* idx, int64_t s, const double* inv_probs, double* out);

/* ---- models + estimators ------------------------------------------------- */
typedef struct orc_model orc_model;
int orc_model_create(const mlsk_model_desc* desc, orc_model** out);
void orc_model_destroy(orc_model* m);
/* fixed data arrays (means / rff weights) as generated for this model */
const double* orc_model_mean_a(const orc_model* m);
const double* orc_model_mean_b(const orc_model* m);

/* One level-sample's draw: indices (1-based) and the gathered columns of A
 * (rows x c, row-major) and rows of B (c x cols).  Vector models: rows = cols = 1. */
int orc_draw_sample(const orc_model* m, uint64_t seed, uint64_t tag, int64_t k, int64_t c,
                    uint32_t* idx, double* a_cols, double* b_rows);

int orc_mlmc(const orc_model* m, int32_t target, double target_param, const mlsk_plan* plan,
             uint64_t seed, int matrix, mlsk_report* rep);
int orc_mc(const orc_model* m, int32_t target, double target_param, int64_t L, int64_t N,
           int64_t M, int64_t c0, uint64_t seed, int matrix, mlsk_report* rep);

/* Per-sample coupled difference Y for replication k at level l (c_l indices,
 * coarse = first c_l / M) of the fused-formulation (identity target) -- used
 * by the fp32 / large-shape tests on a subset of output rows / columns.
 * rows: list of output rows, cols: list of output columns; y[r*ncols + c]. */
int orc_sample_y_subset(const orc_model* m, uint64_t seed, uint64_t tag, int64_t k,
                        int64_t c, int64_t coarse, int32_t target, double target_param,
                        const int64_t* rows, int64_t nrows, const int64_t* cols,
                        int64_t ncols, double* y);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
