// Branch-free correctly rounded sqrt for the Box-Muller radius vs __dsqrt_rn.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sqrt_check sqrt_check.cu && ./sqrt_check
// Checks 2^32 inputs per sweep: random doubles in [2^-60, 2^8) (uniform
// exponent and mantissa) and the radius argument -2 log(u1) for 52-bit u1
// (computed with log(), the set of values of the Box-Muller path), plus edges.
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ double sqrt_nr(double x) {
    double y0;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
    const double e = __fma_rn(-x, __dmul_rn(y0, y0), 1.0);
    const double p = __fma_rn(e, 0.375, 0.5);
    const double y1 = __fma_rn(p, __dmul_rn(y0, e), y0);
    const double s = __dmul_rn(x, y1);
    const double r = __fma_rn(-s, s, x);
    const double res = __fma_rn(r, __dmul_rn(y1, 0.5), s);
    return x == 0.0 ? x : res;
}

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__global__ void k_check(uint64_t base, uint64_t n, int mode, unsigned long long* bad, double* ex) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = mix(base + i);
        double x;
        if (mode == 0) {
            const uint64_t expo = 1023 - 60 + (r >> 58) % 68;  // 2^-60 .. 2^7
            x = __longlong_as_double((long long)((expo << 52) | (r & 0xFFFFFFFFFFFFFULL)));
        } else {
            const double u1 = __dadd_rn(2.0, -__longlong_as_double((long long)(0x3ff0000000000000ULL | (r >> 12))));
            x = __dmul_rn(-2.0, log(u1));
        }
        const double a = sqrt_nr(x), b = __dsqrt_rn(x);
        if (__double_as_longlong(a) != __double_as_longlong(b)) {
            if (atomicAdd(bad, 1ULL) == 0) *ex = x;
        }
    }
}

__global__ void k_edges(unsigned long long* bad) {
    const double xs[] = {0.0, -0.0, 1.0, 2.0, 4.0, 0x1p-51, 0x1p-52, 72.0, 72.5, 73.0, 1e-300, 0x1.fffffffffffffp+7,
                         0x1.0000000000001p-60};
    for (double x : xs)
        if (__double_as_longlong(sqrt_nr(x)) != __double_as_longlong(__dsqrt_rn(x))) atomicAdd(bad, 1ULL);
}

int main() {
    unsigned long long* bad;
    double* ex;
    cudaMallocManaged(&bad, 8);
    cudaMallocManaged(&ex, 8);
    for (int mode = 0; mode < 2; ++mode) {
        *bad = 0;
        const uint64_t n = 1ULL << 32;
        k_check<<<148 * 16, 256>>>(0x1234567ULL + mode * (1ULL << 40), n, mode, bad, ex);
        cudaDeviceSynchronize();
        printf("{\"mode\": \"%s\", \"inputs\": %llu, \"mismatches\": %llu%s}\n",
               mode == 0 ? "random doubles [2^-60, 2^8)" : "-2 log(u1), 52-bit u1", (unsigned long long)n, *bad,
               *bad ? ", \"example\": 1" : "");
    }
    *bad = 0;
    k_edges<<<1, 1>>>(bad);
    cudaDeviceSynchronize();
    printf("{\"mode\": \"edges\", \"mismatches\": %llu}\n", *bad);
    return 0;
}
