/*
 * mlsk_oracle.c -- CPU restatement of the reference's MLMC level estimator.
 *
 * TEST INFRASTRUCTURE ONLY (see mlsk_oracle.h).  Compiled with
 * -ffp-contract=off and no -march so that every multiply and add rounds
 * exactly as in the reference build (proj/CMakeLists.txt:8-16, x86-64
 * baseline ISA, no FMA contraction).  Explicit fma() appears only in the
 * philox-mode transforms, whose definition uses fused operations.
 */
#include "mlsk_oracle.h"
#include "../include/mlsk_stream_spec.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- rng.hpp */

/* rng.hpp:22-27 SplitMix64 finalizer */
uint64_t orc_mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.hpp:31-37 chained asymmetric absorption */
uint64_t orc_derive_seed(uint64_t master, uint64_t a, uint64_t b) {
    uint64_t h = orc_mix(master);
    h = orc_mix(h ^ (a + 0x9e3779b97f4a7c15ULL));
    h = orc_mix(h ^ (b + 0xbf58476d1ce4e5b9ULL));
    return h;
}

/* std::mt19937_64 (ISO C++ [rand.eng.mers], the engine behind rng.hpp:19,87):
 * w=64 n=312 m=156 r=31 a=0xB5026F5AA96619E9 u=29 d=0x5555555555555555 s=17
 * b=0x71D67FFFEDA60000 t=37 c=0xFFF7EEE000000000 l=43 f=6364136223846793005 */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void orc_ref_init(orc_ref_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i) {
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    }
    r->idx = MT_N;
    r->have_cached = 0;
    r->cached = 0.0;
}

static void mt_twist(uint64_t* mt) {
    for (int k = 0; k < MT_N; ++k) {
        const uint64_t y = (mt[k] & MT_UPPER) | (mt[(k + 1) % MT_N] & MT_LOWER);
        mt[k] = mt[(k + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    }
}

uint64_t orc_ref_next_u64(orc_ref_rng* r) {
    if (r->idx >= MT_N) {
        mt_twist(r->mt);
        r->idx = 0;
    }
    uint64_t z = r->mt[r->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= (z >> 43);
    return z;
}

void orc_mt64_stream(uint64_t seed, int64_t count, uint64_t* out) {
    orc_ref_rng r;
    orc_ref_init(&r, seed);
    for (int64_t i = 0; i < count; ++i) out[i] = orc_ref_next_u64(&r);
}

/* rng.hpp:46-51 */
double orc_ref_uniform01(orc_ref_rng* r) {
    return (double)(orc_ref_next_u64(r) >> 11) * 0x1.0p-53;
}
double orc_ref_uniform_pos(orc_ref_rng* r) { return 1.0 - orc_ref_uniform01(r); }

/* rng.hpp:55-65 Box-Muller with a cached second value (glibc libm) */
double orc_ref_normal(orc_ref_rng* r) {
    if (r->have_cached) {
        r->have_cached = 0;
        return r->cached;
    }
    const double rad = sqrt(-2.0 * log(orc_ref_uniform_pos(r)));
    const double theta = 6.283185307179586476925286766559 * orc_ref_uniform01(r);
    r->cached = rad * sin(theta);
    r->have_cached = 1;
    return rad * cos(theta);
}

/* rng.hpp:68 */
double orc_ref_exponential(orc_ref_rng* r) { return -log(orc_ref_uniform_pos(r)); }

/* rng.hpp:73-84 sequential CDF inversion capped at k < 1000 */
long orc_ref_poisson(orc_ref_rng* r, double mean) {
    const double u = orc_ref_uniform01(r);
    double p = exp(-mean);
    double cdf = p;
    long k = 0;
    while (u > cdf && k < 1000) {
        ++k;
        p *= mean / (double)k;
        cdf += p;
    }
    return k;
}

/* ------------------------------------------------ philox-mode (spec header) */

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        const uint64_t p0 = (uint64_t)MLSK_PHILOX_M0 * x0;
        const uint64_t p1 = (uint64_t)MLSK_PHILOX_M1 * x2;
        const uint32_t y0 = (uint32_t)(p1 >> 32) ^ x1 ^ k0;
        const uint32_t y1 = (uint32_t)p1;
        const uint32_t y2 = (uint32_t)(p0 >> 32) ^ x3 ^ k1;
        const uint32_t y3 = (uint32_t)p0;
        x0 = y0; x1 = y1; x2 = y2; x3 = y3;
        k0 += MLSK_PHILOX_W0;
        k1 += MLSK_PHILOX_W1;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

static double as_double(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }
static uint64_t as_u64(double d) { uint64_t b; memcpy(&b, &d, 8); return b; }
static float as_float(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t as_u32(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

static const double T_SINCOS_D[512] = {MLSK_SINCOS_D_INIT};
static const double T_LOG_D[256] = {MLSK_LOG_D_INIT};
static const float T_SINCOS_F[128] = {MLSK_SINCOS_F_INIT};
static const float T_LOG_F[128] = {MLSK_LOG_F_INIT};

/* log(x) for normal x in (0, 1]: the table-driven sequence of the spec */
double orc_log_unit(double x) {
    const uint64_t ix = as_u64(x);
    const uint64_t tmp = ix - 0x3fe6000000000000ULL;
    const int i = (int)((tmp >> 45) & 127);
    const int64_t k = (int64_t)tmp >> 52;
    const double z = as_double(ix - (tmp & 0xfff0000000000000ULL));
    const double invc = T_LOG_D[2 * i], logc = T_LOG_D[2 * i + 1];
    const double r = fma(z, invc, -1.0);
    double p = MLSK_L1P_D_8;
    p = fma(p, r, MLSK_L1P_D_7);
    p = fma(p, r, MLSK_L1P_D_6);
    p = fma(p, r, MLSK_L1P_D_5);
    p = fma(p, r, MLSK_L1P_D_4);
    p = fma(p, r, MLSK_L1P_D_3);
    p = fma(p, r, MLSK_L1P_D_2);
    const double y = fma(p, r * r, r);
    const double kd = (double)k;
    const double hi = fma(kd, MLSK_LN2_HI, logc);
    const double lo = fma(kd, MLSK_LN2_LO, y);
    return hi + lo;
}

/* (cos, sin)(2 pi (iv + f) / 1024) */
static void sincos_iv(int iv, double f, double* c, double* s) {
    const int q = iv >> 8, i = iv & 255;
    const double C = T_SINCOS_D[2 * i], S = T_SINCOS_D[2 * i + 1];
    const double d = f * MLSK_SINCOS_D_STEP;
    const double d2 = d * d;
    const double sd = fma(d * d2, fma(d2, MLSK_SC_S5, MLSK_SC_S3), d);
    const double cd = fma(d2, fma(d2, MLSK_SC_C4, MLSK_SC_C2), 1.0);
    const double c1 = fma(C, cd, -(S * sd));
    const double s1 = fma(S, cd, C * sd);
    switch (q & 3) {
    case 0: *c = c1; *s = s1; break;
    case 1: *c = -s1; *s = c1; break;
    case 2: *c = -c1; *s = -s1; break;
    default: *c = s1; *s = -c1; break;
    }
}

/* (cos, sin)(2 pi u) for u in [0, 1) with at most 52 fraction bits */
void orc_sincos_turn(double u, double* c, double* s) {
    const double v = u * 1024.0;
    const int iv = (int)v;
    sincos_iv(iv, v - (double)iv, c, s);
}

/* 52-bit uniforms from the bit patterns (spec header, box_muller) */
void orc_box_muller(uint64_t ua, uint64_t ub, double* z0, double* z1) {
    const double u1 = 2.0 - as_double(0x3ff0000000000000ULL | (ua >> 12));
    const uint64_t f2 = ub >> 12;
    const int iv = (int)(f2 >> 42);
    const double f = as_double(0x3ff0000000000000ULL | ((f2 & 0x3ffffffffffULL) << 10)) - 1.0;
    const double rad = sqrt(-2.0 * orc_log_unit(u1));
    double c, s;
    sincos_iv(iv, f, &c, &s);
    *z0 = rad * c;
    *z1 = rad * s;
}

float orc_log_unit_f(float x) {
    const uint32_t ix = as_u32(x);
    const uint32_t tmp = ix - 0x3f300000u;
    const int i = (int)((tmp >> 17) & 63);
    const int32_t k = (int32_t)tmp >> 23;
    const float z = as_float(ix - (tmp & 0xff800000u));
    const float invc = T_LOG_F[2 * i], logc = T_LOG_F[2 * i + 1];
    const float r = fmaf(z, invc, -1.0f);
    float p = MLSK_L1P_F_5;
    p = fmaf(p, r, MLSK_L1P_F_4);
    p = fmaf(p, r, MLSK_L1P_F_3);
    p = fmaf(p, r, MLSK_L1P_F_2);
    const float y = fmaf(p, r * r, r);
    const float kf = (float)k;
    const float hi = fmaf(kf, MLSK_LN2_F_HI, logc);
    const float lo = fmaf(kf, MLSK_LN2_F_LO, y);
    return hi + lo;
}

void orc_sincos_turn_f(float u, float* c, float* s) {
    const float v = u * 256.0f;
    const int iv = (int)v;
    const float f = v - (float)iv;
    const int q = iv >> 6, i = iv & 63;
    const float C = T_SINCOS_F[2 * i], S = T_SINCOS_F[2 * i + 1];
    const float d = f * MLSK_SINCOS_F_STEP;
    const float d2 = d * d;
    const float sd = fmaf(d * d2, MLSK_SC_S3_F, d);
    const float cd = fmaf(d2, fmaf(d2, MLSK_SC_C4_F, MLSK_SC_C2_F), 1.0f);
    const float c1 = fmaf(C, cd, -(S * sd));
    const float s1 = fmaf(S, cd, C * sd);
    switch (q & 3) {
    case 0: *c = c1; *s = s1; break;
    case 1: *c = -s1; *s = c1; break;
    case 2: *c = -c1; *s = -s1; break;
    default: *c = s1; *s = -c1; break;
    }
}

void orc_box_muller_f(uint32_t ua, uint32_t ub, float* z0, float* z1) {
    const float u1 = 1.0f - (float)(ua >> 8) * 0x1.0p-24f;
    const float u2 = (float)(ub >> 8) * 0x1.0p-24f;
    const float rad = sqrtf(-2.0f * orc_log_unit_f(u1));
    float c, s;
    orc_sincos_turn_f(u2, &c, &s);
    *z0 = rad * c;
    *z1 = rad * s;
}

static void philox_block(uint64_t key64, uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3,
                         uint32_t out[4]) {
    const uint32_t ctr[4] = {x0, x1, x2, x3};
    const uint32_t key[2] = {(uint32_t)key64, (uint32_t)(key64 >> 32)};
    orc_philox4x32_10(ctr, key, out);
}

static uint64_t lo_u64(const uint32_t r[4]) { return (uint64_t)r[0] | ((uint64_t)r[1] << 32); }
static uint64_t hi_u64(const uint32_t r[4]) { return (uint64_t)r[2] | ((uint64_t)r[3] << 32); }

/* ----------------------------------------------------------- sampling.cpp */

/* sampling.cpp:32-42 (probs = 1/n) + 96-105 (running sum, last forced to 1) */
void orc_uniform_cumulative(int64_t n, double* cum) {
    const double p = 1.0 / (double)n;
    double run = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        run += p;
        cum[j] = run;
    }
    cum[n - 1] = 1.0;
}

static int is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
static int log2i(int64_t n) { int k = 0; while ((1LL << k) < n) ++k; return k; }

/* sampling.cpp:107-112: upper_bound(cum, u01) + 1, clamped to n */
uint32_t orc_index_from_u64(uint64_t x, int64_t n, const double* cum) {
    const double u = (double)(x >> 11) * 0x1.0p-53;
    if (is_pow2(n)) {
        const int k = log2i(n);
        return k == 0 ? 1u : (uint32_t)(x >> (64 - k)) + 1u;
    }
    int64_t lo = 0, hi = n; /* first j with cum[j] > u */
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (cum[mid] > u) hi = mid; else lo = mid + 1;
    }
    if (lo > n - 1) lo = n - 1;
    return (uint32_t)lo + 1u;
}

/* ------------------------------------------------------------- sketch.cpp */

static int check_indices(const uint32_t* idx, int64_t s, int64_t n) {
    if (s <= 0) return fail(MLSK_EINVAL, "sketch: realization must be non-empty");
    for (int64_t i = 0; i < s; ++i) {
        if (idx[i] < 1 || (int64_t)idx[i] > n) return fail(MLSK_EINVAL, "sketch: index out of range");
    }
    return 0;
}

/* sketch.cpp:22-38: sum += a_j * b_j * inv_j in index order; sum / s */
int orc_sketch_inner(const double* a, const double* b, int64_t n, const uint32_t* idx,
                     int64_t s, const double* inv, double* out) {
    const int rc = check_indices(idx, s, n);
    if (rc) return rc;
    double sum = 0.0;
    for (int64_t i = 0; i < s; ++i) {
        const int64_t j = idx[i] - 1;
        const double w = inv ? inv[j] : (double)n;
        sum += a[j] * b[j] * w;
    }
    *out = sum / (double)s;
    return 0;
}

/* sketch.cpp:45-77: o[i][k] += (a[i][j] * inv_j) * b[j][k] per index in order; o *= 1/s */
int orc_sketch_matmul(const double* A, const double* B, int64_t m, int64_t n, int64_t d,
                      const uint32_t* idx, int64_t s, const double* inv, double* out) {
    const int rc = check_indices(idx, s, n);
    if (rc) return rc;
    for (int64_t t = 0; t < m * d; ++t) out[t] = 0.0;
    for (int64_t q = 0; q < s; ++q) {
        const int64_t j = idx[q] - 1;
        const double w = inv ? inv[j] : (double)n;
        for (int64_t i = 0; i < m; ++i) {
            const double scaled = A[i * n + j] * w;
            for (int64_t k = 0; k < d; ++k) out[i * d + k] += scaled * B[j * d + k];
        }
    }
    const double scale = 1.0 / (double)s;
    for (int64_t t = 0; t < m * d; ++t) out[t] *= scale;
    return 0;
}

/* ----------------------------------------------------------------- models */

struct orc_model {
    mlsk_model_desc d;
    int vector;          /* inner-product model */
    int64_t rows, cols;  /* output shape (1x1 for vectors) */
    double* mean_a;      /* gauss / student-t means, rff X */
    double* mean_b;      /* gauss / student-t means, rff W */
    double* rff_b;       /* rff phases */
    double* cum;         /* cumulative table (non power-of-two n) */
    double exp_m10;      /* exp(-10) for the paper models' poisson */
    double rff_scale;
};

const double* orc_model_mean_a(const orc_model* m) { return m->mean_a; }
const double* orc_model_mean_b(const orc_model* m) { return m->mean_b; }

static double data_uniform(uint64_t key64, int64_t e, int f32) {
    uint32_t r[4];
    philox_block(key64, (uint32_t)e, (uint32_t)((uint64_t)e >> 32), 0, MLSK_CTR_DATA, r);
    if (f32) return (double)((float)(r[0] >> 8) * 0x1.0p-24f);
    return (double)(lo_u64(r) >> 11) * 0x1.0p-53;
}

static void gen_means(double* out, int64_t count, uint64_t data_seed, uint64_t which,
                      double lo, double hi, int f32) {
    const uint64_t key = orc_derive_seed(data_seed, MLSK_TAG_DATA, which);
    if (f32) {
        const float flo = (float)lo, w = (float)(hi - lo);
        for (int64_t e = 0; e < count; ++e) {
            const float u = (float)data_uniform(key, e, 1);
            out[e] = (double)(flo + w * u);
        }
    } else {
        const double w = hi - lo;
        for (int64_t e = 0; e < count; ++e) out[e] = lo + w * data_uniform(key, e, 0);
    }
}

/* data normals for the RFF model: element e uses block e/2, z0 / z1 */
static void gen_normals(double* out, int64_t count, uint64_t data_seed, uint64_t which) {
    const uint64_t key = orc_derive_seed(data_seed, MLSK_TAG_DATA, which);
    for (int64_t e = 0; e < count; e += 2) {
        uint32_t r[4];
        philox_block(key, (uint32_t)(e >> 1), (uint32_t)((uint64_t)(e >> 1) >> 32), 1,
                     MLSK_CTR_DATA, r);
        double z0, z1;
        orc_box_muller(lo_u64(r), hi_u64(r), &z0, &z1);
        out[e] = z0;
        if (e + 1 < count) out[e + 1] = z1;
    }
}

int orc_model_create(const mlsk_model_desc* desc, orc_model** out) {
    if (!desc || !out) return fail(MLSK_EINVAL, "model: null descriptor");
    orc_model* m = (orc_model*)calloc(1, sizeof(orc_model));
    m->d = *desc;
    const int k = desc->kind;
    /* vector-pair models (models.hpp:17-21): paper-inner, or a generic kind
     * with m = p = 0; everything else is a matrix-pair model */
    m->vector = k == MLSK_MODEL_PAPER_INNER ||
                ((k == MLSK_MODEL_CONSTANT_ONES || k == MLSK_MODEL_DETERMINISTIC ||
                  k == MLSK_MODEL_GAUSS_MEAN) && desc->m == 0 && desc->p == 0);
    if (k == MLSK_MODEL_PAPER_INNER) { m->d.n = 1000; m->vector = 1; }
    if (k == MLSK_MODEL_PAPER_MATRIX) { m->d.m = 10; m->d.n = 1000; m->d.p = 10; m->vector = 0; }
    if (k == MLSK_MODEL_DETERMINISTIC && !m->vector) { m->d.m = 2; m->d.n = 2; m->d.p = 2; }
    if (m->d.n <= 0 || (!m->vector && (m->d.m <= 0 || m->d.p <= 0))) {
        free(m);
        return fail(MLSK_EINVAL, "model: dimensions must be positive");
    }
    m->rows = m->vector ? 1 : m->d.m;
    m->cols = m->vector ? 1 : m->d.p;
    const int64_t n = m->d.n;
    const int f32 = desc->dtype == MLSK_F32;
    if (k == MLSK_MODEL_STUDENT_T && (desc->mean_a || desc->mean_b)) {
        free(m);
        return fail(MLSK_EINVAL, "student-t: means are generated from data_seed");
    }
    if (k == MLSK_MODEL_GAUSS_MEAN) {
        const int64_t na = m->vector ? n : m->d.m * n;
        const int64_t nb = m->vector ? n : n * m->d.p;
        m->mean_a = (double*)malloc(sizeof(double) * na);
        m->mean_b = (double*)malloc(sizeof(double) * nb);
        if (desc->mean_a) {
            for (int64_t e = 0; e < na; ++e)
                m->mean_a[e] = f32 ? (double)((const float*)desc->mean_a)[e] : ((const double*)desc->mean_a)[e];
        } else {
            gen_means(m->mean_a, na, desc->data_seed, 0, desc->mean_lo, desc->mean_hi, f32);
        }
        if (desc->mean_b) {
            for (int64_t e = 0; e < nb; ++e)
                m->mean_b[e] = f32 ? (double)((const float*)desc->mean_b)[e] : ((const double*)desc->mean_b)[e];
        } else {
            gen_means(m->mean_b, nb, desc->data_seed, 1, desc->mean_lo, desc->mean_hi, f32);
        }
    } else if (k == MLSK_MODEL_RFF) {
        /* X: m x D ~ N(0,1), W: D x n ~ N(0, 1/sigma^2), b: n ~ U(0, 2 pi) */
        const int64_t D = desc->rff_dim;
        if (D <= 0 || !(desc->sigma > 0.0)) { free(m); return fail(MLSK_EINVAL, "rff: bad D / sigma"); }
        m->mean_a = (double*)malloc(sizeof(double) * m->d.m * D);
        m->mean_b = (double*)malloc(sizeof(double) * D * n);
        m->rff_b = (double*)malloc(sizeof(double) * n);
        gen_normals(m->mean_a, m->d.m * D, desc->data_seed, 2);
        gen_normals(m->mean_b, D * n, desc->data_seed, 3);
        const double inv_sigma = 1.0 / desc->sigma;
        for (int64_t e = 0; e < D * n; ++e) m->mean_b[e] = (double)(float)(m->mean_b[e] * inv_sigma);
        for (int64_t e = 0; e < m->d.m * D; ++e) m->mean_a[e] = (double)(float)m->mean_a[e];
        const uint64_t key = orc_derive_seed(desc->data_seed, MLSK_TAG_DATA, 4);
        for (int64_t e = 0; e < n; ++e)
            m->rff_b[e] = (double)(float)(6.283185307179586 * data_uniform(key, e, 0));
        m->rff_scale = sqrt(2.0 / (double)n);
    }
    if (!is_pow2(n)) {
        m->cum = (double*)malloc(sizeof(double) * n);
        orc_uniform_cumulative(n, m->cum);
    }
    m->exp_m10 = exp(-10.0);
    *out = m;
    return 0;
}

void orc_model_destroy(orc_model* m) {
    if (!m) return;
    free(m->mean_a);
    free(m->mean_b);
    free(m->rff_b);
    free(m->cum);
    free(m);
}

static double heaviside(double x) { return x >= 0.0 ? 1.0 : 0.0; }

/* Reference-order full draw for the ref stream (models.hpp:14-16,23-24):
 * all of a then b / A row-major then B row-major.  Fills full A (m x n) and
 * B (n x p), or a and b for vector models. */
static int ref_full_draw(const orc_model* m, orc_ref_rng* rng, double* A, double* B) {
    const int64_t n = m->d.n;
    switch (m->d.kind) {
    case MLSK_MODEL_CONSTANT_ONES:  /* models.cpp:54-74 (no stream use) */
        for (int64_t e = 0; e < m->rows * n; ++e) A[e] = 1.0;
        for (int64_t e = 0; e < n * m->cols; ++e) B[e] = 1.0;
        return 0;
    case MLSK_MODEL_DETERMINISTIC:  /* models.cpp:76-97 */
        if (m->vector) {
            for (int64_t j = 0; j < n; ++j) { A[j] = (double)(j + 1); B[j] = (double)(n + j + 1); }
        } else {
            A[0] = 1; A[1] = 2; A[2] = 3; A[3] = 4;
            B[0] = 5; B[1] = 6; B[2] = 7; B[3] = 8;
        }
        return 0;
    case MLSK_MODEL_PAPER_INNER:    /* models.cpp:12-27 */
        for (int64_t j = 0; j < n; ++j) {
            const double z = orc_ref_normal(rng);
            A[j] = ((double)(j + 1) / 50.0) * (0.5 - z);
        }
        for (int64_t j = 0; j < n; ++j) {
            const double w = (double)orc_ref_poisson(rng, 10.0);
            const double e = orc_ref_exponential(rng);
            B[j] = cos(w + 2.0 * e);
        }
        return 0;
    case MLSK_MODEL_PAPER_MATRIX: { /* models.cpp:29-52 */
        const int64_t mm = m->d.m, d = m->d.p;
        for (int64_t i = 0; i < mm; ++i) {
            for (int64_t j = 0; j < n; ++j) {
                const double z = orc_ref_normal(rng);
                const double x = ((double)(j + 1) / 100.0) * (0.5 - z);
                const double g = orc_ref_normal(rng);
                A[i * n + j] = sin(x) + g * x;
            }
        }
        for (int64_t j = 0; j < n; ++j) {
            for (int64_t k = 0; k < d; ++k) {
                const double p = (double)orc_ref_poisson(rng, 10.0);
                B[j * d + k] = cos(p) * heaviside(5.0 - p);
            }
        }
        return 0;
    }
    case MLSK_MODEL_GAUSS_MEAN: {   /* configs 1-2 written as reference plugins */
        if (m->d.dtype != MLSK_F64) return fail(MLSK_EINVAL, "ref stream: the reference is fp64 only");
        const double sd = m->d.sd;
        const int64_t na = m->rows * n, nb = n * m->cols;
        for (int64_t e = 0; e < na; ++e) A[e] = m->mean_a[e] + sd * orc_ref_normal(rng);
        for (int64_t e = 0; e < nb; ++e) B[e] = m->mean_b[e] + sd * orc_ref_normal(rng);
        return 0;
    }
    default:
        return fail(MLSK_EINVAL, "ref stream: model kind has no reference-stream definition");
    }
}

/* philox-mode value of A[r][col] / a[col] (which = 0) or B[col][q] / b[col] (which = 1) */
static double philox_entry(const orc_model* m, uint64_t key, int which, int64_t col, int64_t rq) {
    const int64_t n = m->d.n;
    switch (m->d.kind) {
    case MLSK_MODEL_CONSTANT_ONES:
        return 1.0;
    case MLSK_MODEL_DETERMINISTIC:
        if (m->vector) return which == 0 ? (double)(col + 1) : (double)(n + col + 1);
        {
            static const double A[4] = {1, 2, 3, 4}, B[4] = {5, 6, 7, 8};
            return which == 0 ? A[rq * 2 + col] : B[col * 2 + rq];
        }
    case MLSK_MODEL_GAUSS_MEAN: {
        const int f32 = m->d.dtype == MLSK_F32;
        const double mean = which == 0 ? m->mean_a[m->vector ? col : rq * n + col]
                                       : m->mean_b[m->vector ? col : col * m->cols + rq];
        if (f32) {
            uint32_t r[4];
            float z[4];
            if (m->vector) { /* one block per column: a takes z0, b takes z1 */
                philox_block(key, (uint32_t)col, 0, 0, MLSK_CTR_A, r);
                orc_box_muller_f(r[0], r[1], &z[0], &z[1]);
                return (double)((float)mean + (float)m->d.sd * z[which]);
            }
            philox_block(key, (uint32_t)col, (uint32_t)(rq >> 2), 0,
                         which == 0 ? MLSK_CTR_A : MLSK_CTR_B, r);
            orc_box_muller_f(r[0], r[1], &z[0], &z[1]);
            orc_box_muller_f(r[2], r[3], &z[2], &z[3]);
            return (double)((float)mean + (float)m->d.sd * z[rq & 3]);
        }
        uint32_t r[4];
        if (m->vector) {
            philox_block(key, (uint32_t)col, 0, 0, MLSK_CTR_A, r);
        } else {
            philox_block(key, (uint32_t)col, (uint32_t)(rq >> 1), 0,
                         which == 0 ? MLSK_CTR_A : MLSK_CTR_B, r);
        }
        double z0, z1;
        orc_box_muller(lo_u64(r), hi_u64(r), &z0, &z1);
        const double z = m->vector ? (which == 0 ? z0 : z1) : ((rq & 1) ? z1 : z0);
        return mean + m->d.sd * z;
    }
    case MLSK_MODEL_STUDENT_T: {
        /* t_nu = z0 / sqrt((z1^2 + ... + z_nu^2) / nu), nu = 3: one block = 4
         * normals; the U(lo, hi) mean is generated on the fly (config 5 stores
         * nothing): element e = row*n + col of A / col*p + q of B */
        uint32_t r[4];
        philox_block(key, (uint32_t)col, (uint32_t)rq, (uint32_t)which, MLSK_CTR_T, r);
        float z[4];
        orc_box_muller_f(r[0], r[1], &z[0], &z[1]);
        orc_box_muller_f(r[2], r[3], &z[2], &z[3]);
        const float v = (z[1] * z[1] + z[2] * z[2]) + z[3] * z[3];
        const float t = z[0] / sqrtf(v / 3.0f);
        /* the mean of row rq (A) / entry rq of B's row col: component rq & 3 of
         * one block per row quad (include/mlsk_stream_spec.h, "student-t means") */
        const uint64_t dkey = orc_derive_seed(m->d.data_seed, MLSK_TAG_DATA, (uint64_t)which);
        uint32_t rd[4];
        philox_block(dkey, (uint32_t)col, (uint32_t)((uint64_t)rq >> 2), 0, MLSK_CTR_SMEAN, rd);
        const float flo = (float)m->d.mean_lo, fw = (float)(m->d.mean_hi - m->d.mean_lo);
        const float mean = flo + fw * ((float)(rd[rq & 3] >> 8) * 0x1.0p-24f);
        return (double)(mean + t);
    }
    case MLSK_MODEL_RFF: {
        /* A[x][col] = sqrt(2/n) cos(w_col . x + b_col); B = A^T */
        const int64_t D = m->d.rff_dim;
        double acc = 0.0;
        for (int64_t t = 0; t < D; ++t) acc += m->mean_a[rq * D + t] * m->mean_b[t * n + col];
        return m->rff_scale * cos(acc + m->rff_b[col]); /* glibc cos: tolerance-only parity */
    }
    default:
        return 0.0;
    }
}

int orc_draw_sample(const orc_model* m, uint64_t seed, uint64_t tag, int64_t k, int64_t c,
                    uint32_t* idx, double* a_cols, double* b_rows) {
    if (c <= 0) return fail(MLSK_EINVAL, "draw_realization: size must be positive");
    const int64_t n = m->d.n, rows = m->rows, cols = m->cols;
    const uint64_t key = orc_derive_seed(seed, tag, (uint64_t)k);
    uint32_t* ix = idx ? idx : (uint32_t*)malloc(sizeof(uint32_t) * c);
    if (m->d.stream_mode == MLSK_STREAM_REF) {
        orc_ref_rng rng;
        orc_ref_init(&rng, key);
        double* A = (double*)malloc(sizeof(double) * rows * n);
        double* B = (double*)malloc(sizeof(double) * n * cols);
        int rc = ref_full_draw(m, &rng, A, B);
        if (rc) { free(A); free(B); if (!idx) free(ix); return rc; }
        for (int64_t i = 0; i < c; ++i) ix[i] = orc_index_from_u64(orc_ref_next_u64(&rng), n, m->cum);
        for (int64_t i = 0; i < c; ++i) {
            const int64_t j = ix[i] - 1;
            if (a_cols) for (int64_t r = 0; r < rows; ++r) a_cols[r * c + i] = A[r * n + j];
            if (b_rows) for (int64_t q = 0; q < cols; ++q) b_rows[i * cols + q] = B[j * cols + q];
        }
        free(A);
        free(B);
    } else {
        if (m->d.kind == MLSK_MODEL_PAPER_INNER || m->d.kind == MLSK_MODEL_PAPER_MATRIX) {
            if (!idx) free(ix);
            return fail(MLSK_EINVAL, "philox stream: paper models are defined on the reference stream only");
        }
        for (int64_t i = 0; i < c; ++i) {
            uint32_t r[4];
            philox_block(key, (uint32_t)(i >> 1), 0, 0, MLSK_CTR_INDEX, r);
            ix[i] = orc_index_from_u64((i & 1) ? hi_u64(r) : lo_u64(r), n, m->cum);
        }
        for (int64_t i = 0; i < c; ++i) {
            const int64_t j = ix[i] - 1;
            if (a_cols) for (int64_t r = 0; r < rows; ++r) a_cols[r * c + i] = philox_entry(m, key, 0, j, r);
            if (b_rows) {
                if (m->d.kind == MLSK_MODEL_RFF) {
                    for (int64_t q = 0; q < cols; ++q) b_rows[i * cols + q] = philox_entry(m, key, 0, j, q);
                } else {
                    for (int64_t q = 0; q < cols; ++q) b_rows[i * cols + q] = philox_entry(m, key, 1, j, q);
                }
            }
        }
    }
    if (!idx) free(ix);
    return 0;
}

/* ------------------------------------------------------------ estimators */

static double apply_target(int32_t target, double tp, double x) {
    switch (target) {
    case MLSK_TARGET_F1: return fabs(x) * heaviside(x - 10.0);       /* models.cpp:103-106 */
    case MLSK_TARGET_F2: return x * x * sin(1.0 / (fabs(x) + tp));  /* models.cpp:108-117 */
    default: return x;                                               /* models.cpp:99-101 */
    }
}

static int64_t ipow(int64_t M, int64_t l) { int64_t r = 1; while (l-- > 0) r *= M; return r; }

#define CHUNK 64 /* parallel.hpp:55 kReductionChunk */

/* One replication's coupled difference v (cells values) from the gathered
 * data, in the reference's arithmetic order (sketch.cpp + estimators.cpp). */
static void sample_difference(const orc_model* m, const double* a_cols, const double* b_rows,
                              int64_t c, int64_t coarse, int32_t target, double tp, double* v) {
    const int64_t n = m->d.n;
    const double w = (double)n; /* uniform inv_probs, sampling.cpp:39 */
    if (m->vector) {
        double sum = 0.0, pre = 0.0;
        for (int64_t i = 0; i < c; ++i) {
            sum += a_cols[i] * b_rows[i] * w;
            if (i + 1 == coarse) pre = sum;
        }
        double x = apply_target(target, tp, sum / (double)c);
        if (coarse > 0) x -= apply_target(target, tp, pre / (double)coarse);
        v[0] = x;
        return;
    }
    const int64_t rows = m->rows, cols = m->cols;
    const double sf = 1.0 / (double)c;
    const double sc = coarse > 0 ? 1.0 / (double)coarse : 0.0;
    for (int64_t r = 0; r < rows; ++r) {
        for (int64_t q = 0; q < cols; ++q) {
            double o = 0.0, pre = 0.0;
            for (int64_t i = 0; i < c; ++i) {
                const double scaled = a_cols[r * c + i] * w;
                o += scaled * b_rows[i * cols + q];
                if (i + 1 == coarse) pre = o;
            }
            double x = apply_target(target, tp, o * sf);
            if (coarse > 0) x -= apply_target(target, tp, pre * sc);
            v[r * cols + q] = x;
        }
    }
}

/* Runs `count` replications of one level (tag, c, coarse) and returns the
 * chunk-order reduced sums (estimators.cpp:128-169). */
static int run_level(const orc_model* m, uint64_t seed, uint64_t tag, int64_t c, int64_t coarse,
                     int64_t count, int32_t target, double tp, double* sum, double* sq) {
    const int64_t rows = m->rows, cols = m->cols, cells = rows * cols;
    double* a_cols = (double*)malloc(sizeof(double) * rows * c);
    double* b_rows = (double*)malloc(sizeof(double) * c * cols);
    double* v = (double*)malloc(sizeof(double) * cells);
    double* s = (double*)malloc(sizeof(double) * cells);
    for (int64_t t = 0; t < cells; ++t) sum[t] = 0.0;
    *sq = 0.0;
    int rc = 0;
    for (int64_t begin = 0; begin < count && !rc; begin += CHUNK) {
        const int64_t end = begin + CHUNK < count ? begin + CHUNK : count;
        for (int64_t t = 0; t < cells; ++t) s[t] = 0.0;
        double s2 = 0.0;
        for (int64_t k = begin; k < end; ++k) {
            rc = orc_draw_sample(m, seed, tag, k, c, NULL, a_cols, b_rows);
            if (rc) break;
            sample_difference(m, a_cols, b_rows, c, coarse, target, tp, v);
            for (int64_t t = 0; t < cells; ++t) {
                const double x = v[t];
                s[t] += x;
                s2 += x * x;
            }
        }
        for (int64_t t = 0; t < cells; ++t) sum[t] += s[t];
        *sq += s2;
    }
    free(a_cols); free(b_rows); free(v); free(s);
    return rc;
}

int orc_mlmc(const orc_model* m, int32_t target, double tp, const mlsk_plan* plan,
             uint64_t seed, int matrix, mlsk_report* rep) {
    if (!plan || plan->M < 2 || plan->L < 0 || !plan->N || plan->c0 < 1)
        return fail(MLSK_EINVAL, "estimator: malformed plan");
    for (int64_t l = 0; l <= plan->L; ++l)
        if (plan->N[l] < 1) return fail(MLSK_EINVAL, "estimator: all N_l must be at least 1");
    if (matrix == m->vector) return fail(MLSK_EINVAL, "estimator: model kind does not match estimator");
    const int64_t cells = m->rows * m->cols;
    double* sum = (double*)malloc(sizeof(double) * cells);
    if (rep->value) for (int64_t t = 0; t < cells; ++t) rep->value[t] = 0.0;
    rep->total_cost_units = 0;
    for (int64_t l = 0; l <= plan->L; ++l) {
        const int64_t fine = plan->c0 * ipow(plan->M, l);
        const int64_t coarse = l > 0 ? fine / plan->M : 0;
        double sq;
        const int rc = run_level(m, seed, (uint64_t)l, fine, coarse, plan->N[l], target, tp, sum, &sq);
        if (rc) { free(sum); return rc; }
        const double inv_n = 1.0 / (double)plan->N[l];
        const int64_t cost = plan->N[l] * (fine + coarse) * cells;
        for (int64_t t = 0; t < cells; ++t) {
            if (rep->level_sum) rep->level_sum[l * cells + t] = sum[t];
            if (rep->level_estimate) rep->level_estimate[l * cells + t] = sum[t] * inv_n;
        }
        if (rep->level_sumsq) rep->level_sumsq[l] = sq;
        if (rep->level_mean_sq) rep->level_mean_sq[l] = sq * inv_n;
        if (rep->level_count) rep->level_count[l] = plan->N[l];
        if (rep->cost_units) rep->cost_units[l] = cost;
        rep->total_cost_units += cost;
        if (rep->value) for (int64_t t = 0; t < cells; ++t) rep->value[t] += sum[t] * inv_n;
    }
    rep->seed = seed;
    rep->wall_time_s = 0.0;
    free(sum);
    return 0;
}

int orc_mc(const orc_model* m, int32_t target, double tp, int64_t L, int64_t N, int64_t M,
           int64_t c0, uint64_t seed, int matrix, mlsk_report* rep) {
    if (M < 2 || N < 1 || c0 < 1 || L < 0) return fail(MLSK_EINVAL, "mc: need M >= 2 and N >= 1");
    if (matrix == m->vector) return fail(MLSK_EINVAL, "estimator: model kind does not match estimator");
    const int64_t cells = m->rows * m->cols;
    const int64_t s = c0 * ipow(M, L);
    double* sum = (double*)malloc(sizeof(double) * cells);
    double sq;
    const int rc = run_level(m, seed, MLSK_TAG_MC, s, 0, N, target, tp, sum, &sq);
    if (rc) { free(sum); return rc; }
    for (int64_t t = 0; t < cells; ++t) {
        if (rep->value) rep->value[t] = sum[t] / (double)N; /* estimators.cpp:219,265 divide */
        if (rep->level_sum) rep->level_sum[t] = sum[t];
    }
    if (rep->level_sumsq) rep->level_sumsq[0] = sq;
    if (rep->level_count) rep->level_count[0] = N;
    rep->total_cost_units = N * s * cells;
    rep->seed = seed;
    free(sum);
    return 0;
}

int orc_sample_y_subset(const orc_model* m, uint64_t seed, uint64_t tag, int64_t k, int64_t c,
                        int64_t coarse, int32_t target, double tp, const int64_t* rows,
                        int64_t nrows, const int64_t* cols, int64_t ncols, double* y) {
    /* gather only the requested rows / columns of the sampled panels */
    const int64_t n = m->d.n;
    const uint64_t key = orc_derive_seed(seed, tag, (uint64_t)k);
    if (m->d.stream_mode != MLSK_STREAM_PHILOX) return fail(MLSK_EINVAL, "subset: philox stream only");
    uint32_t* ix = (uint32_t*)malloc(sizeof(uint32_t) * c);
    for (int64_t i = 0; i < c; ++i) {
        uint32_t r[4];
        philox_block(key, (uint32_t)(i >> 1), 0, 0, MLSK_CTR_INDEX, r);
        ix[i] = orc_index_from_u64((i & 1) ? hi_u64(r) : lo_u64(r), n, m->cum);
    }
    double* a = (double*)malloc(sizeof(double) * nrows * c);
    double* b = (double*)malloc(sizeof(double) * c * ncols);
    const int bwhich = m->d.kind == MLSK_MODEL_RFF ? 0 : 1;
    for (int64_t i = 0; i < c; ++i) {
        const int64_t j = ix[i] - 1;
        for (int64_t r = 0; r < nrows; ++r) a[r * c + i] = philox_entry(m, key, 0, j, rows[r]);
        for (int64_t q = 0; q < ncols; ++q) b[i * ncols + q] = philox_entry(m, key, bwhich, j, cols[q]);
    }
    const double w = (double)n;
    const double sf = 1.0 / (double)c, sc = coarse > 0 ? 1.0 / (double)coarse : 0.0;
    for (int64_t r = 0; r < nrows; ++r) {
        for (int64_t q = 0; q < ncols; ++q) {
            double o = 0.0, pre = 0.0;
            for (int64_t i = 0; i < c; ++i) {
                o += (a[r * c + i] * w) * b[i * ncols + q];
                if (i + 1 == coarse) pre = o;
            }
            double x = apply_target(target, tp, o * sf);
            if (coarse > 0) x -= apply_target(target, tp, pre * sc);
            y[r * ncols + q] = x;
        }
    }
    free(ix); free(a); free(b);
    return 0;
}
