// Throughput of the philox-mode normal-pair generator (diagnostics):
// pairs/s for philox alone, Box-Muller alone, and both, one pair per loop trip.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1904_00429_b200/csrc/mlsk_device.cuh"

using namespace mlsk;
__device__ __align__(16) const double g_sc[512] = {MLSK_SINCOS_D_INIT};
__device__ __align__(16) const double g_lg[256] = {MLSK_LOG_D_INIT};

template <int MODE>
__global__ void __launch_bounds__(256) k_pairs(uint64_t key, int iters, double* out) {
    __shared__ __align__(16) double2 s_sc[256];
    __shared__ __align__(16) double2 s_lg[128];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_sc[i] = reinterpret_cast<const double2*>(g_sc)[i];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) s_lg[i] = reinterpret_cast<const double2*>(g_lg)[i];
    __syncthreads();
    Tables T{reinterpret_cast<const double*>(s_sc), reinterpret_cast<const double*>(s_lg), nullptr, nullptr};
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0.0;
    uint64_t x = tid * 0x9E3779B97F4A7C15ULL;
    for (int i = 0; i < iters; ++i) {
        uint64_t ua, ub;
        if (MODE != 1) {
            const u32x4 r = philox((uint32_t)i, tid, 0, MLSK_CTR_A, key);
            ua = lo64(r);
            ub = hi64(r);
        } else {
            x += 0x9E3779B97F4A7C15ULL;
            ua = x;
            ub = x * 0xBF58476D1CE4E5B9ULL;
        }
        if (MODE != 0) {
            double z0, z1;
            box_muller(ua, ub, z0, z1, T);
            acc = __dadd_rn(acc, __dadd_rn(z0, z1));
        } else {
            acc += (double)(ua ^ ub);
        }
    }
    if (acc == 1.2345) out[0] = acc;
}

template <int MODE>
void run(const char* name) {
    double* out;
    cudaMalloc(&out, 8);
    const int grid = 148 * 8, iters = 2048;
    k_pairs<MODE><<<grid, 256>>>(1, 16, out);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_pairs<MODE><<<grid, 256>>>(1, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double pairs = (double)grid * 256 * iters;
    const double smsp_cycles = 148.0 * 4 * 1.965e9 * best * 1e-3;
    printf("{\"mode\":\"%s\",\"ms\":%.3f,\"Gpairs_per_s\":%.1f,\"smsp_cycles_per_pair\":%.2f}\n", name, best,
           pairs / best / 1e6, smsp_cycles / pairs * 32.0 / 32.0);
    cudaFree(out);
}

int main() {
    run<0>("philox_only");
    run<1>("box_muller_only");
    run<2>("philox+box_muller");
    return 0;
}
