// tcgen05.mma kind::tf32 issue-rate microbenchmark for the 3xTF32 GEMM design:
// single CTA (M128 N256) vs CTA pair (cta_group::2, M256 N256), SWIZZLE_64B vs
// SWIZZLE_128B K-major operands, the 3xTF32 operand pattern over a ring of
// stages (hi.hi, hi.lo, lo.hi per K8 step), with and without epilogue warps
// reading the other TMEM accumulator concurrently (tcgen05.ld 32x32b.x16).
// Operands are zeroed shared memory; only the tensor pipe's rate is measured.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_shapes tc_shapes.cu && ./tc_shapes
#include <cstdint>
#include <cstdio>

constexpr int THREADS = 64 + 32 * 16;
__constant__ int g_random;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t a, int rowb) {
    return (uint64_t)((a & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)((8 * rowb) >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)(rowb == 128 ? 2 : 4) << 61);
}

__device__ __forceinline__ void wait_bar(uint32_t b, uint32_t ph) {
    uint32_t done;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(b), "r"(ph)
                     : "memory");
    } while (!done);
}

// pair: 1 = cta_group::2 (cluster of 2, M = 256), 0 = cta_group::1 (M = 128)
// rowb: 64 (SW64, K-chunk 16) or 128 (SW128, K-chunk 32)
// pattern: 0 = one MMA per K8 step on one stage (probe), 1 = 3xTF32 (3 MMAs per K8)
// epi: epilogue warps read the other accumulator in a loop
template <int PAIR>
__global__ void __launch_bounds__(THREADS, 1) k_tc(int rounds, int rowb, int pattern, int epi, int stages,
                                                   int N, uint32_t* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* base = sm + ((1024 - (sa(sm) & 1023)) & 1023);
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t s_tmem;
    __shared__ volatile int s_stop;
    const int warp = threadIdx.x >> 5;
    uint32_t rank = 0;
    if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    // per-CTA stage: A hi / lo (128 rows) + B hi / lo (N rows held by this CTA)
    const int kchunk = rowb / 4;                     // tf32 per row
    const int nrows_b = PAIR ? N / 2 : N;            // B rows held in this CTA's smem
    const int a_bytes = 128 * rowb, b_bytes = nrows_b * rowb;
    const int stage_bytes = 2 * a_bytes + 2 * b_bytes;
    for (int i = threadIdx.x; i < stages * stage_bytes / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 40503u;
        h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
        reinterpret_cast<float*>(base)[i] = g_random ? ((float)(h >> 8) * (1.0f / 8388608.0f) - 1.0f) : 0.f;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_stop = 0;
    }
    if (warp == 1) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&s_tmem)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&s_tmem)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (PAIR) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    if (warp == 1 && threadIdx.x == 32 && rank == 0) {
        const uint32_t s0 = sa(base);
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)((PAIR ? 256 : 128) >> 4) << 24);
        uint32_t ph[2] = {0, 0};
        int s = 0;
        int issued = 0, ngrp = 0;
        for (int r = 0; r < rounds; ++r) {
            // one "stage" worth of MMAs
            const uint32_t st = s0 + s * stage_bytes;
            const int ksteps = kchunk / 8;
            for (int kk = 0; kk < ksteps; ++kk) {
                const uint64_t ah = desc(st + kk * 32, rowb), al = desc(st + a_bytes + kk * 32, rowb);
                const uint64_t bh = desc(st + 2 * a_bytes + kk * 32, rowb);
                const uint64_t bl = desc(st + 2 * a_bytes + b_bytes + kk * 32, rowb);
                if (PAIR) {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                 "l"(ah), "l"(bh), "r"(idesc), "r"(1u)
                                 : "memory");
                    if (pattern) {
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                     "l"(ah), "l"(bl), "r"(idesc), "r"(1u)
                                     : "memory");
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                     "l"(al), "l"(bh), "r"(idesc), "r"(1u)
                                     : "memory");
                    }
                } else {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                 "l"(ah), "l"(bh), "r"(idesc), "r"(1u)
                                 : "memory");
                    if (pattern) {
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                     "l"(ah), "l"(bl), "r"(idesc), "r"(1u)
                                     : "memory");
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                     "l"(al), "l"(bh), "r"(idesc), "r"(1u)
                                     : "memory");
                    }
                }
                issued += pattern ? 3 : 1;
            }
            if (++s == stages) s = 0;
            if (issued >= 48 || r + 1 == rounds) {  // commit this group; wait for the group before the previous one
                issued = 0;
                const int g = ngrp & 1;
                if (ngrp >= 2) { wait_bar(sa(&bar[g]), ph[g]); ph[g] ^= 1; }
                if (PAIR)
                    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(sa(&bar[g])), "h"((uint16_t)3) : "memory");
                else
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar[g])) : "memory");
                ++ngrp;
            }
        }
        for (int i = ngrp >= 2 ? ngrp - 2 : 0; i < ngrp; ++i) { wait_bar(sa(&bar[i & 1]), ph[i & 1]); ph[i & 1] ^= 1; }
        s_stop = 1;
        if (PAIR) {  // the peer's epilogue warps stop too
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(remote) : "r"(sa((const void*)&s_stop)));
            asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(remote), "r"(1) : "memory");
        }
    }
    if (warp >= 2 && epi) {
        // read the other accumulator (columns 256..511) until the MMA thread is done
        const int q = warp & 3, h = (warp - 2) >> 2;
        float acc = 0.f;
        while (!s_stop) {
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t r[16];
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + 256u + (uint32_t)(h * 64 + ch * 16);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15])
                    : "r"(ta));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 16; ++i) acc = __fmaf_rn(__uint_as_float(r[i]), __uint_as_float(r[i]), acc);
            }
        }
        if (acc == 1.2345f) sink[1] = 1;
    }
    __syncthreads();
    // wait for every committed MMA group (the drain commit arrives on bar[0] after all groups)
    if (threadIdx.x == 0) {
        // count arrivals on bar[0]: we only know the last phase completes eventually; poll both phases
        // (each commit flips bar[g]'s phase; simply wait for quiescence by spinning on a fence)
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (PAIR) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
        __syncthreads();
    }
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
    if (threadIdx.x == 0 && rounds < 0) sink[0] = tmem;
}

template <int PAIR>
float run(int sms, int rounds, int rowb, int pattern, int epi, int stages, int N, uint32_t* sink, int smem) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(PAIR ? (sms / 2) * 2 : sms);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PAIR ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, k_tc<PAIR>, 2, rowb, pattern, epi, stages, N, sink);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, k_tc<PAIR>, rounds, rowb, pattern, epi, stages, N, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* sink;
    cudaMalloc(&sink, 8);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k_tc<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_tc<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int rnd = 1;
    cudaMemcpyToSymbol(g_random, &rnd, sizeof(int));
    const int cases[4][2] = {{0, 256}, {0, 128}, {1, 256}, {1, 128}};  // (pair, N)
    for (const auto& cs : cases)
        for (int epi : {0, 1}) {
            const int pair = cs[0], N = cs[1], rowb = 64, pattern = 1;
            const int stage_bytes = 2 * 128 * rowb + 2 * (pair ? N / 2 : N) * rowb;
            int stages = (192 * 1024) / stage_bytes;
            if (stages > 4) stages = 4;
            const int rounds = 4000;
            float ms = pair ? run<1>(sms, rounds, rowb, pattern, epi, stages, N, sink, smem)
                            : run<0>(sms, rounds, rowb, pattern, epi, stages, N, sink, smem);
            const int ctas = pair ? (sms / 2) * 2 : sms;
            const double per_round = (double)(rowb / 4 / 8) * 3;  // MMAs per round
            // flops per CTA per MMA: 2 * 128 * N * 8 (pair: M = 256 over two CTAs)
            const double flops = (double)ctas * rounds * per_round * 2.0 * 128 * N * 8;
            printf("{\"random\": 1, \"pair\": %d, \"N\": %d, \"rowb\": %d, \"epi\": %d, \"stages\": %d, "
                   "\"tflops\": %.1f, \"err\": \"%s\"}\n",
                   pair, N, rowb, epi, stages, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
            fflush(stdout);
        }
    return 0;
}
