// tcgen05.mma kind::i8 (s8 x s8 -> s32) throughput vs N, one CTA per SM,
// M = 128, K = 32 per instruction, operands from (zeroed) shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_mma i8_mma.cu && ./i8_mma
#include <cstdint>
#include <cstdio>

__global__ void __launch_bounds__(128, 1) k_i8(int rounds, int n, int kind_i8, uint32_t* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* base = sm + ((1024 - ((uint32_t)__cvta_generic_to_shared(sm) & 1023)) & 1023);
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t s_tmem;
    for (int i = threadIdx.x; i < 48 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    if (threadIdx.x == 0) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(base), sb = sa + 16384;
        auto desc = [](uint32_t a) {
            return (uint64_t)((a & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
                   ((uint64_t)2 << 61);
        };
        // i8: c S32 (2), a/b signed (1); tf32 reference: c F32 (1), a/b TF32 (2)
        const uint32_t idesc = kind_i8 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24))
                                       : ((1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24));
        uint32_t ph = 0;
        for (int r = 0; r < rounds; ++r) {
            for (int i = 0; i < 64; ++i) {
                const uint64_t ad = desc(sa + (i & 3) * 32), bd = desc(sb + (i & 3) * 32);
                if (kind_i8)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                 "l"(ad), "l"(bd), "r"(idesc), "r"(1u)
                                 : "memory");
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                 "l"(ad), "l"(bd), "r"(idesc), "r"(1u)
                                 : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
            uint32_t done;
            do {
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(done)
                             : "r"(b), "r"(ph)
                             : "memory");
            } while (!done);
            ph ^= 1;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
    if (threadIdx.x == 0 && rounds < 0) sink[0] = tmem;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 48 * 1024 + 1024;
    cudaFuncSetAttribute(k_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    uint32_t* sink;
    cudaMalloc(&sink, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int kind = 0; kind < 2; ++kind)
        for (int n : {16, 32, 64, 128, 256}) {
            k_i8<<<sms, 128, smem>>>(4, n, kind, sink);
            cudaDeviceSynchronize();
            const int rounds = 400;
            float best = 1e30f;
            for (int r = 0; r < 3; ++r) {
                cudaEventRecord(e0);
                k_i8<<<sms, 128, smem>>>(rounds, n, kind, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            const int K = kind ? 32 : 8;
            const double ops = (double)sms * rounds * 64 * 2.0 * 128 * n * K;
            printf("{\"kind\": \"%s\", \"M\": 128, \"N\": %d, \"K\": %d, \"tops\": %.1f, \"err\": \"%s\"}\n",
                   kind ? "i8" : "tf32", n, K, ops / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
