// Pipe-throughput microbenchmark for the fp64 sampled-GEMM design decision:
// is DMMA (mma.sync f64 -> DMMA.8x8x4) a separate pipe from DFMA / FFMA / IMAD
// on sm_100a, and what are their peaks?  Prints one JSON line per experiment.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("{\"error\":\"%s\"}\n",cudaGetErrorString(e)); return 1;}}while(0)

// mode: 0 = dmma only, 1 = dfma only, 2 = half warps dmma / half dfma,
//       3 = half dmma / half ffma, 4 = ffma only, 5 = half dmma / half imad, 6 = imad only
template <int MODE>
__global__ void __launch_bounds__(256) pipes(double* out, int iters) {
    const int warp = threadIdx.x >> 5;
    const bool use_mma = (MODE == 0) || ((MODE == 2 || MODE == 3 || MODE == 5) && (warp & 1) == 0);
    double acc = 0.0;
    if (use_mma) {
        double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
        double c[8][2];
        #pragma unroll
        for (int j = 0; j < 8; ++j) { c[j][0] = 0; c[j][1] = 0; }
        for (int i = 0; i < iters; ++i) {
            #pragma unroll
            for (int j = 0; j < 8; ++j)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
        }
        #pragma unroll
        for (int j = 0; j < 8; ++j) acc += c[j][0] + c[j][1];
    } else if (MODE == 1 || MODE == 2) {
        double x[8];
        #pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
        const double m = 1.0000001, s = 1e-9;
        for (int i = 0; i < iters; ++i) {
            // 8 DMMA (2048 FMA/warp) vs 64 DFMA (2048 FMA/warp) per iteration: equal work
            #pragma unroll
            for (int r = 0; r < 8; ++r)
                #pragma unroll
                for (int j = 0; j < 8; ++j) x[j] = fma(x[j], m, s);
        }
        #pragma unroll
        for (int j = 0; j < 8; ++j) acc += x[j];
    } else if (MODE == 3 || MODE == 4) {
        float x[8];
        #pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
        const float m = 1.0000001f, s = 1e-9f;
        for (int i = 0; i < iters; ++i) {
            #pragma unroll
            for (int r = 0; r < 8; ++r)
                #pragma unroll
                for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], m, s);
        }
        #pragma unroll
        for (int j = 0; j < 8; ++j) acc += x[j];
    } else {
        uint32_t x[8];
        #pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
        for (int i = 0; i < iters; ++i) {
            #pragma unroll
            for (int r = 0; r < 8; ++r)
                #pragma unroll
                for (int j = 0; j < 8; ++j) x[j] = __umulhi(x[j], 0xD2511F53u) ^ (x[j] * 0xCD9E8D57u);
        }
        #pragma unroll
        for (int j = 0; j < 8; ++j) acc += x[j];
    }
    if (acc == 12345.678) out[0] = acc;
}

template <int MODE>
int run(const char* name, int blocks_per_sm) {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out; CK(cudaMalloc(&out, 8));
    const int iters = 4096;
    const int grid = sms * blocks_per_sm;
    pipes<MODE><<<grid, 256>>>(out, 16); CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        pipes<MODE><<<grid, 256>>>(out, iters);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    // per warp per iteration: 2048 FMA (= 4096 flop) for each of the op kinds
    const double warps = grid * 8.0;
    const double ops = warps * iters * 4096.0;
    printf("{\"exp\":\"%s\",\"blocks_per_sm\":%d,\"ms\":%.4f,\"tflops_total\":%.2f}\n",
           name, blocks_per_sm, best, ops / (best * 1e-3) / 1e12);
    cudaFree(out);
    return 0;
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("{\"device\":\"%s\",\"sms\":%d,\"clock_khz\":%d}\n", p.name, p.multiProcessorCount, p.clockRate);
    for (int b : {1, 2, 4}) {
        run<0>("dmma_only", b);
        run<1>("dfma_only", b);
        run<2>("dmma_half_dfma_half", b);
        run<3>("dmma_half_ffma_half", b);
        run<4>("ffma_only", b);
        run<5>("dmma_half_imad_half", b);
        run<6>("imad_only(umulhi+mul+xor)", b);
    }
    return 0;
}
