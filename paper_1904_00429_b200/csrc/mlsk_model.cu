// mlsk_model.cu -- device models: validation (the reference's constructor
// checks, tensor.cpp:12-60 / models.cpp:54-97) and generation of the fixed
// model data on the device (means, RFF weights) from the philox data stream.
#include <cmath>
#include <cstring>

#include <atomic>

#include "mlsk_internal.h"

namespace mlsk {

// Transform tables of the philox-mode stream (include/mlsk_stream_tables.h).
__device__ __align__(16) const double g_sincos_d[512] = {MLSK_SINCOS_D_INIT};
__device__ __align__(16) const double g_log_d[256] = {MLSK_LOG_D_INIT};
__device__ __align__(16) const float g_sincos_f[128] = {MLSK_SINCOS_F_INIT};
__device__ __align__(16) const float g_log_f[128] = {MLSK_LOG_F_INIT};

void configure_mempool() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;  // keep freed blocks pooled between calls
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done_dev = dev;
}

Tables device_tables() {
    // symbol addresses are per device (one module per device context)
    static std::mutex mu;
    static std::map<int, Tables> per_dev;
    int dev = 0;
    MLSK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    auto it = per_dev.find(dev);
    if (it != per_dev.end()) return it->second;
    Tables r{};
    void* p;
    MLSK_CUDA(cudaGetSymbolAddress(&p, g_sincos_d)); r.sincos_d = (const double*)p;
    MLSK_CUDA(cudaGetSymbolAddress(&p, g_log_d)); r.log_d = (const double*)p;
    MLSK_CUDA(cudaGetSymbolAddress(&p, g_sincos_f)); r.sincos_f = (const float*)p;
    MLSK_CUDA(cudaGetSymbolAddress(&p, g_log_f)); r.log_f = (const float*)p;
    per_dev[dev] = r;
    return r;
}

namespace {

__global__ void k_means_f64(double* out, int64_t count, uint64_t key, double lo, double w) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x) {
        const u32x4 r = philox((uint32_t)e, (uint32_t)((uint64_t)e >> 32), 0, MLSK_CTR_DATA, key);
        out[e] = __dadd_rn(lo, __dmul_rn(w, u01(lo64(r))));
    }
}

__global__ void k_means_f32(float* out, int64_t count, uint64_t key, float lo, float w) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x) {
        const u32x4 r = philox((uint32_t)e, (uint32_t)((uint64_t)e >> 32), 0, MLSK_CTR_DATA, key);
        const float u = __fmul_rn((float)(r.x >> 8), 0x1.0p-24f);
        out[e] = __fadd_rn(lo, __fmul_rn(w, u));
    }
}

// data normals (RFF X / W): element e takes z0 / z1 of block e / 2, scaled
__global__ void k_normals_f32(float* out, int64_t count, uint64_t key, double scale, Tables tab) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = e >> 1;
        const u32x4 r = philox((uint32_t)h, (uint32_t)((uint64_t)h >> 32), 1, MLSK_CTR_DATA, key);
        double z0, z1;
        box_muller(lo64(r), hi64(r), z0, z1, tab);
        const double z = (e & 1) ? z1 : z0;
        out[e] = scale == 1.0 ? (float)z : (float)__dmul_rn(z, scale);
    }
}

__global__ void k_phases_f32(float* out, int64_t count, uint64_t key) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x) {
        const u32x4 r = philox((uint32_t)e, (uint32_t)((uint64_t)e >> 32), 0, MLSK_CTR_DATA, key);
        out[e] = (float)__dmul_rn(6.283185307179586, u01(lo64(r)));
    }
}

template <class T>
__global__ void k_transpose(const T* __restrict__ in, T* __restrict__ out, int64_t rows, int64_t cols) {
    __shared__ T tile[32][33];
    const int64_t c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][i];
    }
}

__global__ void k_nan_count(const double* x, int64_t n, int* flag) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        if (x[e] != x[e]) *flag = 1;
}

int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

template <class T>
void transpose(const T* in, T* out, int64_t rows, int64_t cols, cudaStream_t st) {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    k_transpose<T><<<grid, dim3(32, 8), 0, st>>>(in, out, rows, cols);
    launched();
}

}  // namespace

bool model_is_vector(const mlsk_model_desc* d) {
    const int k = d->kind;
    return k == MLSK_MODEL_PAPER_INNER ||
           ((k == MLSK_MODEL_CONSTANT_ONES || k == MLSK_MODEL_DETERMINISTIC || k == MLSK_MODEL_GAUSS_MEAN) &&
            d->m == 0 && d->p == 0);
}

void build_model(Model& M, const mlsk_model_desc* d, cudaStream_t st) {
    if (!d) invalid("model: null descriptor");
    static std::atomic<uint64_t> next_serial{1};
    M.serial = next_serial.fetch_add(1);
    M.desc = *d;
    mlsk_model_desc& D = M.desc;
    const int k = D.kind;
    if (k < MLSK_MODEL_CONSTANT_ONES || k > MLSK_MODEL_STUDENT_T) invalid("model: unknown model kind");
    if (D.stream_mode != MLSK_STREAM_PHILOX && D.stream_mode != MLSK_STREAM_REF)
        invalid("model: unknown stream mode");
    if (D.dtype != MLSK_F64 && D.dtype != MLSK_F32) invalid("model: unknown dtype");
    M.vector = model_is_vector(d);
    if (k == MLSK_MODEL_PAPER_INNER) D.n = 1000;                              // models.cpp:13
    if (k == MLSK_MODEL_PAPER_MATRIX) { D.m = 10; D.n = 1000; D.p = 10; }    // models.cpp:30
    if (k == MLSK_MODEL_DETERMINISTIC && !M.vector) { D.m = 2; D.n = 2; D.p = 2; }  // models.cpp:88-96
    if (k == MLSK_MODEL_RFF) D.p = D.m;  // B = A^T
    if (D.n <= 0) invalid("model: n must be positive");
    if (!M.vector && (D.m <= 0 || D.p <= 0)) invalid("model: dimensions must be positive");
    if (D.n > (int64_t(1) << 32) || D.m > (int64_t(1) << 31) || D.p > (int64_t(1) << 31))
        invalid("model: dimensions exceed the 32-bit counter space");
    const bool f32 = D.dtype == MLSK_F32;
    if (f32 && !(k == MLSK_MODEL_GAUSS_MEAN || k == MLSK_MODEL_STUDENT_T || k == MLSK_MODEL_RFF))
        invalid("model: fp32 is defined for the gauss-mean, student-t and rff models only");
    if (!f32 && (k == MLSK_MODEL_STUDENT_T || k == MLSK_MODEL_RFF))
        invalid("model: student-t and rff models are fp32");
    if (D.stream_mode == MLSK_STREAM_REF &&
        (k == MLSK_MODEL_STUDENT_T || k == MLSK_MODEL_RFF || f32))
        invalid("ref stream: model kind has no reference-stream definition");
    if (D.stream_mode == MLSK_STREAM_PHILOX && (k == MLSK_MODEL_PAPER_INNER || k == MLSK_MODEL_PAPER_MATRIX))
        invalid("philox stream: paper models are defined on the reference stream only");
    if (k == MLSK_MODEL_GAUSS_MEAN && !(D.sd >= 0.0 && std::isfinite(D.sd))) invalid("model: sd must be finite");
    if (k == MLSK_MODEL_STUDENT_T && D.nu != 3.0) invalid("student-t: only nu = 3 is implemented");
    if (k == MLSK_MODEL_RFF && (D.rff_dim <= 0 || !(D.sigma > 0.0))) invalid("rff: bad dimension / sigma");

    M.rows = M.vector ? 1 : D.m;
    M.cols = M.vector ? 1 : D.p;
    M.ref_u64 = ref_model_u64(k, M.vector, D.m, D.n, D.p);

    DevModel& dm = M.dm;
    std::memset(&dm, 0, sizeof dm);
    dm.kind = k;
    dm.dtype = D.dtype;
    dm.stream = D.stream_mode;
    dm.vector = M.vector;
    dm.m = D.m; dm.n = D.n; dm.p = D.p;
    dm.rows = M.rows; dm.cols = M.cols;
    dm.sd = D.sd;
    dm.log2n = is_pow2(D.n) ? log2_exact(D.n) : -1;
    dm.exp_m10 = std::exp(-10.0);  // rng.hpp:75 with mean 10 (glibc)
    dm.tab = device_tables();

    if (!is_pow2(D.n)) {  // sampling.cpp:32-42,96-105
        std::vector<double> cum(D.n);
        const double p = 1.0 / (double)D.n;
        double run = 0.0;
        for (int64_t j = 0; j < D.n; ++j) { run += p; cum[j] = run; }
        cum[D.n - 1] = 1.0;
        M.cum.alloc_on(D.n, st);
        MLSK_CUDA(cudaMemcpyAsync(M.cum.p, cum.data(), sizeof(double) * D.n, cudaMemcpyHostToDevice, st));
        dm.cum = M.cum.p;
    }
    if (k == MLSK_MODEL_PAPER_MATRIX) {  // models.cpp:47-48 cos(p) * H(5 - p), p <= 1000
        std::vector<double> t(1001);
        for (int pz = 0; pz <= 1000; ++pz) t[pz] = std::cos((double)pz) * (5.0 - pz >= 0.0 ? 1.0 : 0.0);
        M.paper_b.alloc_on(1001, st);
        MLSK_CUDA(cudaMemcpyAsync(M.paper_b.p, t.data(), sizeof(double) * 1001, cudaMemcpyHostToDevice, st));
        dm.paper_b = M.paper_b.p;
    }
    if (k == MLSK_MODEL_STUDENT_T) {
        // means generated on the fly from the data stream (config 5: nothing stored)
        if (D.mean_a || D.mean_b) invalid("student-t: means are generated from data_seed");
        dm.st_key_a = derive_seed(D.data_seed, MLSK_TAG_DATA, 0);
        dm.st_key_b = derive_seed(D.data_seed, MLSK_TAG_DATA, 1);
        dm.st_lo = (float)D.mean_lo;
        dm.st_w = (float)(D.mean_hi - D.mean_lo);
    }
    if (k == MLSK_MODEL_GAUSS_MEAN) {
        const int64_t na = M.vector ? D.n : D.m * D.n;
        const int64_t nb = M.vector ? D.n : D.n * D.p;
        const double lo = D.mean_lo, w = D.mean_hi - D.mean_lo;
        if (f32) {
            M.mean_a_f.alloc_on(na, st);
            M.mean_b_f.alloc_on(nb, st);
            if (D.mean_a) {
                const float* h = (const float*)D.mean_a;
                for (int64_t e = 0; e < na; ++e) if (h[e] != h[e]) invalid("DenseMatrix: NaN entry rejected");
                MLSK_CUDA(cudaMemcpyAsync(M.mean_a_f.p, h, sizeof(float) * na, cudaMemcpyHostToDevice, st));
            } else {
                k_means_f32<<<grid_for(na), 256, 0, st>>>(M.mean_a_f.p, na, derive_seed(D.data_seed, MLSK_TAG_DATA, 0),
                                                          (float)lo, (float)w);
                launched();
            }
            if (D.mean_b) {
                const float* h = (const float*)D.mean_b;
                for (int64_t e = 0; e < nb; ++e) if (h[e] != h[e]) invalid("DenseMatrix: NaN entry rejected");
                MLSK_CUDA(cudaMemcpyAsync(M.mean_b_f.p, h, sizeof(float) * nb, cudaMemcpyHostToDevice, st));
            } else {
                k_means_f32<<<grid_for(nb), 256, 0, st>>>(M.mean_b_f.p, nb, derive_seed(D.data_seed, MLSK_TAG_DATA, 1),
                                                          (float)lo, (float)w);
                launched();
            }
            dm.mean_a_f = M.mean_a_f.p;
            dm.mean_b_f = M.mean_b_f.p;
            if (!M.vector) {
                M.mean_at_f.alloc_on(na, st);
                transpose<float>(M.mean_a_f.p, M.mean_at_f.p, D.m, D.n, st);
                dm.mean_at_f = M.mean_at_f.p;
            }
        } else {
            M.mean_a.alloc_on(na, st);
            M.mean_b.alloc_on(nb, st);
            DevArray<int> flag;
            flag.alloc_on(1, st);
            flag.zero(st);
            if (D.mean_a) {
                MLSK_CUDA(cudaMemcpyAsync(M.mean_a.p, D.mean_a, sizeof(double) * na, cudaMemcpyHostToDevice, st));
                k_nan_count<<<grid_for(na), 256, 0, st>>>(M.mean_a.p, na, flag.p);
                launched();
            } else {
                k_means_f64<<<grid_for(na), 256, 0, st>>>(M.mean_a.p, na, derive_seed(D.data_seed, MLSK_TAG_DATA, 0), lo, w);
                launched();
            }
            if (D.mean_b) {
                MLSK_CUDA(cudaMemcpyAsync(M.mean_b.p, D.mean_b, sizeof(double) * nb, cudaMemcpyHostToDevice, st));
                k_nan_count<<<grid_for(nb), 256, 0, st>>>(M.mean_b.p, nb, flag.p);
                launched();
            } else {
                k_means_f64<<<grid_for(nb), 256, 0, st>>>(M.mean_b.p, nb, derive_seed(D.data_seed, MLSK_TAG_DATA, 1), lo, w);
                launched();
            }
            if (D.mean_a || D.mean_b) {
                int h = 0;
                MLSK_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
                MLSK_CUDA(cudaStreamSynchronize(st));
                if (h) invalid("DenseMatrix: NaN entry rejected");
            }
            dm.mean_a = M.mean_a.p;
            dm.mean_b = M.mean_b.p;
            if (!M.vector) {
                M.mean_at.alloc_on(na, st);
                transpose<double>(M.mean_a.p, M.mean_at.p, D.m, D.n, st);
                dm.mean_at = M.mean_at.p;
            }
        }
    }
    if (k == MLSK_MODEL_RFF) {
        const int64_t Dd = D.rff_dim;
        M.rff_x.alloc_on(D.m * Dd, st);
        M.rff_w.alloc_on(Dd * D.n, st);
        M.rff_b.alloc_on(D.n, st);
        k_normals_f32<<<grid_for(D.m * Dd), 256, 0, st>>>(M.rff_x.p, D.m * Dd,
                                                          derive_seed(D.data_seed, MLSK_TAG_DATA, 2), 1.0,
                                                          dm.tab);
        k_normals_f32<<<grid_for(Dd * D.n), 256, 0, st>>>(M.rff_w.p, Dd * D.n,
                                                          derive_seed(D.data_seed, MLSK_TAG_DATA, 3), 1.0 / D.sigma,
                                                          dm.tab);
        k_phases_f32<<<grid_for(D.n), 256, 0, st>>>(M.rff_b.p, D.n, derive_seed(D.data_seed, MLSK_TAG_DATA, 4));
        launched(3);
        dm.rff_x = M.rff_x.p;
        M.rff_xt.alloc_on(D.m * Dd, st);
        transpose<float>(M.rff_x.p, M.rff_xt.p, D.m, Dd, st);
        dm.rff_xt = M.rff_xt.p;
        dm.rff_w = M.rff_w.p;
        dm.rff_b = M.rff_b.p;
        dm.rff_dim = Dd;
        dm.rff_scale = std::sqrt(2.0 / (double)D.n);
    }
}

}  // namespace mlsk
