// mlsk_sketch.cu -- device versions of the reference's sketch functions on
// caller-supplied data (sketch.cpp:22-77), for the known-answer tests of
// proj/tests/test_sketch.cpp.  Same validation (sketch.cpp:9-18,25-28,48-51)
// and the same operation order as the reference.
#include <algorithm>
#include <functional>
#include <vector>

#include "mlsk_internal.h"

namespace mlsk {
namespace {

__global__ void k_sketch_inner(const double* __restrict__ a, const double* __restrict__ b,
                               const double* __restrict__ inv, const uint32_t* __restrict__ idx, int64_t s,
                               double* out) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    double sum = 0.0;
    for (int64_t i = 0; i < s; ++i) {
        const int64_t j = (int64_t)idx[i] - 1;
        sum = __dadd_rn(sum, __dmul_rn(__dmul_rn(a[j], b[j]), inv[j]));
    }
    *out = __ddiv_rn(sum, (double)s);
}

__global__ void k_sketch_matmul(const double* __restrict__ A, const double* __restrict__ B,
                                const double* __restrict__ inv, const uint32_t* __restrict__ idx, int64_t m,
                                int64_t n, int64_t d, int64_t s, double scale, double* __restrict__ out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * d;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / d, k = e - i * d;
        double o = 0.0;
        for (int64_t q = 0; q < s; ++q) {
            const int64_t j = (int64_t)idx[q] - 1;
            o = __dadd_rn(o, __dmul_rn(__dmul_rn(A[i * n + j], inv[j]), B[j * d + k]));
        }
        out[e] = __dmul_rn(o, scale);
    }
}

void check_indices(const uint32_t* idx, int64_t s, int64_t n) {
    if (!idx || s <= 0) invalid("sketch: realization must be non-empty");
    for (int64_t i = 0; i < s; ++i)
        if (idx[i] < 1 || (int64_t)idx[i] > n) invalid("sketch: index out of range");
}

std::vector<double> inv_probs(const double* inv, int64_t n) {
    if (inv) {
        for (int64_t j = 0; j < n; ++j)
            if (!(inv[j] > 0.0)) invalid("IndexDistribution: probabilities must be strictly positive");
        return std::vector<double>(inv, inv + n);
    }
    return std::vector<double>(n, (double)n);  // sampling.cpp:39
}

template <class T>
T* upload(DevArray<T>& d, const T* h, int64_t n, cudaStream_t s) {
    d.alloc(n);
    MLSK_CUDA(cudaMemcpyAsync(d.p, h, sizeof(T) * n, cudaMemcpyHostToDevice, s));
    return d.p;
}

}  // namespace
}  // namespace mlsk

using namespace mlsk;

namespace mlsk {
int run_guarded(const std::function<void()>& body);  // mlsk_api.cu
}

namespace {
struct Stream {
    cudaStream_t s = nullptr;
    Stream() {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw Error(MLSK_ERUNTIME, "no CUDA device available (the library has no CPU fallback)");
        MLSK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    }
    ~Stream() { if (s) cudaStreamDestroy(s); }
};
}  // namespace


extern "C" int mlsk_sketch_inner(const double* a, const double* b, int64_t n, const uint32_t* idx, int64_t s,
                                 const double* inv, double* out) {
    return run_guarded([&] {
        if (!a || !b || !out || n <= 0) invalid("sketch_inner: dimension mismatch");
        check_indices(idx, s, n);
        const auto w = inv_probs(inv, n);
        Stream st;
        DevArray<double> da, db, dw, dout(1);
        DevArray<uint32_t> di;
        k_sketch_inner<<<1, 1, 0, st.s>>>(upload(da, a, n, st.s), upload(db, b, n, st.s),
                                          upload(dw, w.data(), n, st.s), upload(di, idx, s, st.s), s, dout.p);
        launched();
        MLSK_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double), cudaMemcpyDeviceToHost, st.s));
        MLSK_CUDA(cudaStreamSynchronize(st.s));
    });
}

extern "C" int mlsk_sketch_matmul(const double* A, const double* B, int64_t m, int64_t n, int64_t d,
                                  const uint32_t* idx, int64_t s, const double* inv, double* out) {
    return run_guarded([&] {
        if (!A || !B || !out || m <= 0 || n <= 0 || d <= 0) invalid("sketch_matmul: dimension mismatch");
        check_indices(idx, s, n);
        const auto w = inv_probs(inv, n);
        Stream st;
        DevArray<double> dA, dB, dw, dout(m * d);
        DevArray<uint32_t> di;
        const double scale = 1.0 / (double)s;  // sketch.cpp:72
        const int64_t cells = m * d;
        const int grid = (int)std::min<int64_t>((cells + 255) / 256, 148 * 16);
        k_sketch_matmul<<<grid, 256, 0, st.s>>>(upload(dA, A, m * n, st.s), upload(dB, B, n * d, st.s),
                                                upload(dw, w.data(), n, st.s), upload(di, idx, s, st.s), m, n, d,
                                                s, scale, dout.p);
        launched();
        MLSK_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double) * cells, cudaMemcpyDeviceToHost, st.s));
        MLSK_CUDA(cudaStreamSynchronize(st.s));
    });
}
