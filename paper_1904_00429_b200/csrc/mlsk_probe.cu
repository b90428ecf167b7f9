// mlsk_probe.cu -- per-kernel event timing (mlsk_profile_*) and the in-run
// fp64 tensor-pipe peak measurement used as the roofline denominator.
#include <algorithm>
#include <cstdio>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "mlsk_internal.h"

namespace mlsk {

namespace {

struct Pending {
    std::string name;
    cudaEvent_t e0, e1;
};

std::mutex g_mu;
bool g_on = false;
std::vector<Pending> g_pending;
std::map<std::string, std::pair<int64_t, double>> g_acc;  // launches, ms
cudaEvent_t g_base = nullptr;                              // timeline origin
struct Span {
    std::string name;
    double t0, t1;
};
std::vector<Span> g_timeline;

void drain() {
    for (auto& p : g_pending) {
        float ms = 0.f;
        cudaEventSynchronize(p.e1);
        cudaEventElapsedTime(&ms, p.e0, p.e1);
        auto& a = g_acc[p.name];
        a.first += 1;
        a.second += ms;
        if (g_base && g_timeline.size() < 100000) {
            float t0 = 0.f, t1 = 0.f;
            cudaEventElapsedTime(&t0, g_base, p.e0);
            cudaEventElapsedTime(&t1, g_base, p.e1);
            g_timeline.push_back({p.name, t0, t1});
        }
        cudaEventDestroy(p.e0);
        cudaEventDestroy(p.e1);
    }
    g_pending.clear();
}

// DMMA throughput loop: 8 independent m8n8k4 accumulators per warp
__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
    double c[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[j][0]), "+d"(c[j][1])
                         : "d"(a), "d"(b));
    }
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += c[j][0] + c[j][1];
    if (acc == 12345.678) out[0] = acc;
}

// TF32 tcgen05 throughput loop: one CTA per SM, M=128 N=256 K=8 MMAs from
// (zeroed) shared memory into TMEM, committed to an mbarrier every 64 MMAs.
__global__ void __launch_bounds__(128, 1) k_tf32_peak(int rounds, int n, uint32_t* sink) {
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
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
        uint32_t ph = 0;
        for (int r = 0; r < rounds; ++r) {
            for (int i = 0; i < 64; ++i) {
                const uint64_t ad = desc(sa + (i & 3) * 32), bd = desc(sb + (i & 3) * 32);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                             "l"(ad), "l"(bd), "r"(idesc), "r"(1u)
                             : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b)
                         : "memory");
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

}  // namespace

Prof::Prof(const char* n, cudaStream_t s) : name(n), stream(s) {
    if (!g_on) return;
    cudaEventCreate(&e0);
    cudaEventRecord(e0, stream);
}

Prof::~Prof() {
    if (!e0) return;
    cudaEvent_t e1;
    cudaEventCreate(&e1);
    cudaEventRecord(e1, stream);
    std::lock_guard<std::mutex> lk(g_mu);
    g_pending.push_back({name, e0, e1});
}

int run_guarded(const std::function<void()>& body);

}  // namespace mlsk

using namespace mlsk;

extern "C" {

int mlsk_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_on = on != 0;
    return 0;
}

int mlsk_profile_reset(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    drain();
    g_acc.clear();
    g_timeline.clear();
    if (!g_base) cudaEventCreate(&g_base);
    cudaEventRecord(g_base, 0);
    cudaEventSynchronize(g_base);
    return 0;
}

// Timeline entry i (launch order of completion draining): returns the count.
int mlsk_profile_timeline(int i, char* name, int name_len, double* t0, double* t1) {
    std::lock_guard<std::mutex> lk(g_mu);
    drain();
    if (i >= 0 && i < (int)g_timeline.size()) {
        if (name && name_len > 0) snprintf(name, name_len, "%s", g_timeline[i].name.c_str());
        if (t0) *t0 = g_timeline[i].t0;
        if (t1) *t1 = g_timeline[i].t1;
    }
    return (int)g_timeline.size();
}

// Entries in name order; returns the number of entries, fills entry `i`.
int mlsk_profile_read(int i, char* name, int name_len, int64_t* launches, double* ms) {
    std::lock_guard<std::mutex> lk(g_mu);
    drain();
    int k = 0;
    for (auto& kv : g_acc) {
        if (k == i) {
            if (name && name_len > 0) {
                snprintf(name, name_len, "%s", kv.first.c_str());
            }
            if (launches) *launches = kv.second.first;
            if (ms) *ms = kv.second.second;
        }
        ++k;
    }
    return (int)g_acc.size();
}

// Measured fp64 tensor (DMMA) peak in TFLOP/s on `device` (-1 = current).
double mlsk_measure_fp64_peak(int device) {
    double result = -1.0;
    run_guarded([&] {
        if (device >= 0) MLSK_CUDA(cudaSetDevice(device));
        int dev = 0, sms = 0;
        MLSK_CUDA(cudaGetDevice(&dev));
        MLSK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        DevArray<double> out(1);
        const int grid = sms * 4, iters = 4096;
        k_dmma_peak<<<grid, 256>>>(out.p, 64);
        launched();
        MLSK_CUDA(cudaDeviceSynchronize());
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            k_dmma_peak<<<grid, 256>>>(out.p, iters);
            cudaEventRecord(e1);
            launched();
            MLSK_CUDA(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        const double flops = (double)grid * 8 /*warps*/ * iters * 8 /*mma*/ * 512.0;
        result = flops / (best * 1e-3) / 1e12;
    });
    return result;
}

// Dense TF32 tcgen05 throughput measured on the device (M=128, N=n, K=8 per
// instruction, one CTA per SM), TFLOP/s.  The 3xTF32 fp32 engine's peak is a third.
double mlsk_measure_tf32_peak(int device, int n) {
    double result = -1.0;
    run_guarded([&] {
        if (device >= 0) MLSK_CUDA(cudaSetDevice(device));
        int dev = 0, sms = 0;
        MLSK_CUDA(cudaGetDevice(&dev));
        MLSK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        if (n <= 0 || n > 256 || n % 16) n = 256;
        const int smem = 48 * 1024 + 1024;
        MLSK_CUDA(cudaFuncSetAttribute(k_tf32_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        DevArray<uint32_t> sink(1);
        k_tf32_peak<<<sms, 128, smem>>>(4, n, sink.p);
        launched();
        MLSK_CUDA(cudaDeviceSynchronize());
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e30f;
        const int rounds = 400;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            k_tf32_peak<<<sms, 128, smem>>>(rounds, n, sink.p);
            cudaEventRecord(e1);
            launched();
            MLSK_CUDA(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        const double flops = (double)sms * rounds * 64 * 2.0 * 128 * n * 8;
        result = flops / (best * 1e-3) / 1e12;
    });
    return result;
}

// Config-1 RNG roofline: index-samples / s of the fused inner kernel's
// per-index work alone (k_index_rate).
double mlsk_measure_index_rate(int device) {
    double result = -1.0;
    run_guarded([&] { result = measure_index_rate(device); });
    return result;
}

}  // extern "C"
