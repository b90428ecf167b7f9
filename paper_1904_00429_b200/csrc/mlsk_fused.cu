// mlsk_fused.cu -- the fused fp64 engine (throughput path, philox stream,
// identity target).
//
// Fused formulation: for a level-sample with c
// indices and coarse prefix cc = c/M,
//     Y = f(fine) - f(coarse) = sum_t w_t a_t b_t^T,
//     w_t = n/c for t >= cc,   w_t = n/c - n/cc for t < cc   (level 0: n/c),
// one signed contraction with K = c instead of the reference's two passes
// (estimators.cpp:137-147).  Per level the work is split in two kernels:
//
//  k_gen_panels_f64  draws each level-sample's indices and generates ONLY the
//                    sampled columns A[:, S] and rows B[S, :] (mean gather +
//                    Philox/Box-Muller noise, w_t folded into B) straight into
//                    16-wide K-chunks laid out for the MMA (k-permuted,
//                    16-byte XOR swizzle), each element generated exactly once.
//  k_gemm_f64        persistent CTAs, one 128 x 64 output tile per CTA over a
//                    strided set of samples; a producer warp streams the K-chunks
//                    with cp.async.bulk (TMA bulk copies) into a 4-stage mbarrier
//                    ring; 8 consumer warps run DMMA (mma.sync m8n8k4 f64) into
//                    register accumulators; at each sample boundary the epilogue
//                    adds Y into a register-resident running sum S and Y^2 into
//                    a scalar -- the per-sample output never touches memory.
//  k_reduce_tiles    deterministic (fixed-order) sum of the per-CTA partials
//                    into the level accumulators.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "mlsk_internal.h"

namespace mlsk {

namespace {

#ifndef MLSK_F64_PANEL_HINT
#define MLSK_F64_PANEL_HINT 1  // measured +0.2% on the config-2 step (1.5756 vs 1.5722 M)
#endif
constexpr int KC = 16;        // K-chunk (indices per smem stage)
constexpr int BM = 128;       // tile rows
#ifndef MLSK_F64_BN
#define MLSK_F64_BN 64
#endif
constexpr int BN = MLSK_F64_BN;  // tile cols (64: running sum in registers; 128: in tensor memory)
constexpr int STAGES = 6;
#ifndef MLSK_GEMM_WN
#define MLSK_GEMM_WN (BN / 2)
#endif
constexpr int WN = MLSK_GEMM_WN;          // warp tile: 32 rows x WN columns
constexpr int WARPS_N = BN / WN;
constexpr int NJ = WN / 8;                // 8-column DMMA tiles per warp
constexpr int CONSUMERS = (BM / 32) * WARPS_N;  // consumer warps
constexpr int GEMM_THREADS = CONSUMERS * 32;  // lane 0 of warp 0 also produces
constexpr int GEMM_MAXNREG = CONSUMERS == 8 ? 192 : 128;
// 32 x 64 warp tiles (BN = 128): the 64 accumulator doubles take 128 registers,
// so the running sum moves to tensor memory and the fragments load in halves
constexpr bool S_TMEM = NJ == 8;
constexpr uint32_t S_TMEM_COLS = 256;  // 2 warps per lane quadrant x 64 doubles x 2 words
constexpr int A_STAGE_BYTES = BM * KC * 8;
constexpr int B_STAGE_BYTES = BN * KC * 8;
constexpr int GEN_THREADS = 256;

// ---------------------------------------------------------------- layout

// Element (r, k) of a K-chunk tile, 16 doubles per row: k permuted so that
// lane (g, t) finds k = t, t+4, t+8, t+12 in two 16-byte granules, granules
// XOR-swizzled by r & 7 (conflict-free LDS.128 fragment loads).
__device__ __forceinline__ int tile_slot(int r, int k) {
    const int pos = (k & 3) * 4 + (k >> 2);
    const int g = pos >> 1;
    return r * KC + (((g ^ (r & 7)) << 1) | (pos & 1));
}

__device__ __forceinline__ void load_tables(double2* s_sc, double2* s_lg, const Tables& T) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_sc[i] = reinterpret_cast<const double2*>(T.sincos_d)[i];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) s_lg[i] = reinterpret_cast<const double2*>(T.log_d)[i];
}

// full-circle (1024-entry) sincos table, see sincos_iv_full
__device__ __forceinline__ void load_tables_full(double2* s_sc1024, double2* s_lg, const Tables& T) {
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_sc1024[i] = full_circle_entry(i, T.sincos_d);
    for (int i = threadIdx.x; i < 128; i += blockDim.x) s_lg[i] = reinterpret_cast<const double2*>(T.log_d)[i];
}

// --------------------------------------------------------- panel generator

// grid-stride over work items (b, kc); each item produces the A chunk
// (MP x 16) and the weighted B chunk (PP x 16) of sample b in phases of 128
// rows / columns, double-buffered in shared memory: 256 threads generate one
// phase (row pairs share one Philox block) while the previous phase's tile is
// streamed out with coalesced 16-byte stores.
constexpr int GROWS = 128;
constexpr int GEN_DYN_SMEM = 2 * GROWS * KC * 8;  // the two staging tiles

// One phase: 128 rows of A (IS_A) or 128 columns of B, 16 sampled columns.
// Thread (rp = tid % 64, tq = tid / 64) owns row pair rp of chunk columns
// tq, tq+4, tq+8, tq+12 (lanes span row pairs: coalesced mean loads); the four
// items are unrolled so their mean loads issue up front and four independent
// Philox / Box-Muller chains interleave.
template <bool IS_A>
__device__ __forceinline__ void gen_phase(const DevModel& M, const Tables& T, uint64_t key, int64_t rb,
                                          const int* s_j, const double* s_w, double* tl, int tid) {
    constexpr int U = KC / (GEN_THREADS / (GROWS / 2));  // items per thread (4)
    const int rp = tid & (GROWS / 2 - 1), tq = tid / (GROWS / 2);
    const int r0 = 2 * rp;
    const int64_t dim = IS_A ? M.m : M.p;
    const int64_t lim = dim - rb;                      // valid rows / cols of this phase
    const double* mrow = (IS_A ? M.mean_at : M.mean_b) + rb + r0;
    const uint32_t rowpair = (uint32_t)((rb + r0) >> 1);
    const double sd = M.sd;
    if (r0 + 1 < lim && (dim & 1) == 0) {
        // full aligned pair: vector mean loads first, then the generators
        double2 mv[U];
        int jj[U];
        double v0[U], v1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            jj[u] = s_j[tq + 4 * u];  // padding columns carry j = 0 (and B weight 0)
            mv[u] = __ldg(reinterpret_cast<const double2*>(mrow + (uint64_t)(uint32_t)jj[u] * (uint32_t)dim));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            // one Philox block per chain, interleaved by the scheduler with the
            // previous chain's fp64 Box-Muller (integer and fp64 pipes overlap)
            const u32x4 r = philox((uint32_t)jj[u], rowpair, 0, IS_A ? MLSK_CTR_A : MLSK_CTR_B, key);
            double z0, z1;
            box_muller<true>(lo64(r), hi64(r), z0, z1, T);
            double a = __dadd_rn(mv[u].x, __dmul_rn(sd, z0));
            double b = __dadd_rn(mv[u].y, __dmul_rn(sd, z1));
            if (!IS_A) {
                // padding columns (only when KC does not divide c): A holds a finite
                // draw of column 0, B is 0 * x = 0 (s_w = 0), so the product is 0
                const double w = s_w[tq + 4 * u];
                a = __dmul_rn(w, a);
                b = __dmul_rn(w, b);
            }
            v0[u] = a;
            v1[u] = b;
        }
        // chunk columns k and k + 4 share one 16-byte granule: 128-bit stores
#pragma unroll
        for (int u = 0; u < U; u += 2) {
            *reinterpret_cast<double2*>(tl + tile_slot(r0, tq + 4 * u)) = make_double2(v0[u], v0[u + 1]);
            *reinterpret_cast<double2*>(tl + tile_slot(r0 + 1, tq + 4 * u)) = make_double2(v1[u], v1[u + 1]);
        }
    } else {
        // ragged edge (odd dimension or the last rows of the phase)
#pragma unroll 1
        for (int u = 0; u < U; ++u) {
            const int j = s_j[tq + 4 * u];
            double a = 0.0, b = 0.0;
            if (r0 < lim) {
                const double* mp = mrow + (int64_t)j * dim;
                const bool pair = r0 + 1 < lim;
                const double m0 = __ldg(mp), m1 = pair ? __ldg(mp + 1) : 0.0;
                const u32x4 r = philox((uint32_t)j, rowpair, 0, IS_A ? MLSK_CTR_A : MLSK_CTR_B, key);
                double z0, z1;
                box_muller<true>(lo64(r), hi64(r), z0, z1, T);
                a = __dadd_rn(m0, __dmul_rn(sd, z0));
                if (pair) b = __dadd_rn(m1, __dmul_rn(sd, z1));
                if (!IS_A) {
                    const double w = s_w[tq + 4 * u];
                    a = __dmul_rn(w, a);
                    b = __dmul_rn(w, b);
                }
            }
            tl[tile_slot(r0, tq + 4 * u)] = a;
            tl[tile_slot(r0 + 1, tq + 4 * u)] = b;
        }
    }
}

__global__ void __launch_bounds__(GEN_THREADS, 4)
k_gen_panels_f64(DevModel M, uint64_t seed, uint64_t tag, const int64_t* __restrict__ ks, int nb, int64_t c,
                 int64_t cc, double w_fine, double w_coarse, int64_t MP, int64_t PP, int64_t nkc, int64_t kc0,
                 double* __restrict__ Apan, double* __restrict__ Bpan, uint32_t* __restrict__ idx_out, int64_t pcc,
                 const MkEntry* __restrict__ mk, int64_t mk_stride, const MkInfo* __restrict__ mk_info) {
    // pcc >= cc: K slots [0, pcc) hold the coarse prefix t < cc (zero padding
    // up to pcc), slots [pcc, ...) the suffix t >= cc.  pcc = cc (identity
    // target) is the plain layout; a nonlinear target pads the prefix to whole
    // K-chunks so the GEMM can read the coarse sum at a chunk boundary.
    __shared__ __align__(16) double2 s_sc[1024];
    __shared__ __align__(16) double2 s_lg[128];
    extern __shared__ __align__(16) double gen_dyn[];  // 2 x GROWS x KC tiles (past the 48 KB static limit)
    __shared__ int s_j[KC];
    __shared__ double s_w[KC];
    load_tables_full(s_sc, s_lg, M.tab);
    Tables T = M.tab;
    T.sincos_d = reinterpret_cast<const double*>(s_sc);
    T.log_d = reinterpret_cast<const double*>(s_lg);
    const int tid = threadIdx.x;
    const int64_t items = (int64_t)nb * nkc;
    const int a_phases = (int)((MP + GROWS - 1) / GROWS), b_phases = (int)((PP + GROWS - 1) / GROWS);
    int buf = 0;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int b = (int)(it / nkc);
        const int64_t kc = it - (int64_t)b * nkc;
        const uint64_t key = derive_seed(seed, tag, (uint64_t)ks[b]);
        __syncthreads();  // previous item's readers of s_j are done
        if (tid < KC) {
            const int64_t sl = (kc0 + kc) * KC + tid;  // K slot (kc0: first chunk of this K-range)
            const int64_t t = sl < pcc ? sl : sl - pcc + cc;  // column of the sample
            int j = 0;  // padding slots: column 0 with weight 0
            double w = 0.0;
            if (mk) {
                // merged sampled columns: slot sl of the sample's (j, W_j) list
                if (sl < mk_info[b].len) {
                    const MkEntry e = mk[(int64_t)b * mk_stride + sl];
                    if (e.j >= 0) {
                        j = e.j;
                        w = e.w;
                    }
                }
            } else if (sl < pcc ? t < cc : t < c) {
                const u32x4 r = philox((uint32_t)(t >> 1), 0, 0, MLSK_CTR_INDEX, key);
                const uint32_t ix = index_from_u64((t & 1) ? hi64(r) : lo64(r), M.n, M.log2n, M.cum);
                j = (int)(ix - 1);
                w = t < cc ? w_coarse : w_fine;
                if (idx_out) idx_out[(int64_t)b * c + t] = ix;
            }
            s_j[tid] = j;
            s_w[tid] = w;
        }
        __syncthreads();
        double* const baseA = Apan + ((int64_t)b * nkc + kc) * MP * KC;
        double* const baseB = Bpan + ((int64_t)b * nkc + kc) * PP * KC;
        for (int ph = 0; ph < a_phases + b_phases; ++ph) {
            const bool isA = ph < a_phases;
            const int rb = (isA ? ph : ph - a_phases) * GROWS;
            const int span = (int)(isA ? MP : PP) - rb;  // rows / cols in the panel
            double* tl = gen_dyn + buf * (GROWS * KC);
            if (isA) gen_phase<true>(M, T, key, rb, s_j, s_w, tl, tid);
            else gen_phase<false>(M, T, key, rb, s_j, s_w, tl, tid);
            // the tile leaves by one bulk copy (TMA engine), not by the threads
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                double* dst = (isA ? baseA : baseB) + (int64_t)rb * KC;
                const uint32_t bytes = (uint32_t)((span < GROWS ? span : GROWS) * KC * 8);
#if MLSK_F64_PANEL_HINT
                uint64_t pol;  // panels stream through L2 once: evict them first
                asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                             "r"((uint32_t)__cvta_generic_to_shared(tl)), "r"(bytes), "l"(pol)
                             : "memory");
#else
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                             "r"((uint32_t)__cvta_generic_to_shared(tl)), "r"(bytes)
                             : "memory");
#endif
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                // the other tile's copy (previous phase) has finished reading
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            }
            __syncthreads();
            buf ^= 1;
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------- mbarriers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ double2 lds128(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}


__device__ __forceinline__ void tm_ld32(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_st32(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// ------------------------------------------------------------------ GEMM

struct GemmShape {
    int nb;        // samples in the batch
    int64_t nkc;   // K-chunks per sample
    int64_t MP, PP;
    int T;         // output tiles
    int Gs;        // sample groups (CTAs per tile)
    int tiles_n;   // tiles along the columns
};

// 192-register cap (no spills; 218 uncapped): 192 x 256 leaves the SM room for
// one generator CTA beside the GEMM CTA (measured +2% on the config-2 step).
// SPLIT: one sample split along K per launch (split_part 1 first, 2 middle,
// 3 last); a separate instantiation keeps the common path's registers intact.
// NL: nonlinear target.  The panels hold the coarse prefix in K-chunks
// [0, pre_kc) (uniform weights n / c); after chunk pre_kc - 1 every thread
// stores f(cscale * acc) (the coarse estimate, cscale = c / cc) of its
// fragments to `nl_scratch` (coalesced, L2-resident), and the sample's
// epilogue forms Y = f(acc) - f(coarse) (estimators.cpp:137-147).
struct NlArgs {
    int target;
    double tparam;
    int64_t pre_kc;  // 0: level 0 (no coarse term)
    double cscale;
    double* scratch;
};
// Y of one fragment entry at the sample's end: f(fine) - f(coarse)
__device__ __forceinline__ double nl_y(const NlArgs& a, int g, int i, int j, int e, double fine) {
    double y = apply_target(a.target, a.tparam, fine);
    if (a.pre_kc > 0) {
        const double* sc = a.scratch + (int64_t)g * (4 * NJ * 2) * GEMM_THREADS + threadIdx.x;
        y = __dsub_rn(y, sc[(int64_t)((i * NJ + j) * 2 + e) * GEMM_THREADS]);
    }
    return y;
}
template <bool SPLIT, bool NL>
__global__ void __maxnreg__(GEMM_MAXNREG)
k_gemm_f64(const double* __restrict__ Apan, const double* __restrict__ Bpan, GemmShape sh,
           double* __restrict__ part, double* __restrict__ part_sq, int split_part, double* __restrict__ ypart,
           NlArgs nla) {
    extern __shared__ __align__(1024) unsigned char smem[];
    double* sA = reinterpret_cast<double*>(smem);
    double* sB = reinterpret_cast<double*>(smem + STAGES * A_STAGE_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * (A_STAGE_BYTES + B_STAGE_BYTES));
    __shared__ double s_sq[CONSUMERS];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x;
    const int tile = g % sh.T, grp = g / sh.T;
    const int tm = tile / sh.tiles_n, tn = tile % sh.tiles_n;
    const int my_samples = grp < sh.nb ? (sh.nb - 1 - grp) / sh.Gs + 1 : 0;
    const int64_t iters = (int64_t)my_samples * sh.nkc;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&bars[s]), 1);                     // full: producer arrive + tx
            mbar_init(smem_u32(&bars[STAGES + s]), CONSUMERS);    // empty: one per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __shared__ uint32_t s_tmem;
    if (S_TMEM && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(S_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (S_TMEM) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (S_TMEM) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // producer state (lane 0 of warp 0): next (sample, chunk) to load
    const bool producer = threadIdx.x == 0;
    int p_s = 0;
    uint32_t p_ph = 0;
    int64_t p_b = grp, p_kc = 0, p_it = 0;
    auto produce = [&]() {
        // load iteration p_it into slot p_s once every warp has released it
        mbar_wait(smem_u32(&bars[STAGES + p_s]), p_ph ^ 1);
        const uint32_t full = smem_u32(&bars[p_s]);
        mbar_expect_tx(full, A_STAGE_BYTES + B_STAGE_BYTES);
        MLSK_DCHECK(p_b < sh.nb && p_kc < sh.nkc && (int64_t)tm * BM < sh.MP && (int64_t)tn * BN < sh.PP);
        const double* srcA = Apan + ((p_b * sh.nkc + p_kc) * sh.MP + (int64_t)tm * BM) * KC;
        const double* srcB = Bpan + ((p_b * sh.nkc + p_kc) * sh.PP + (int64_t)tn * BN) * KC;
        bulk_g2s(smem_u32(sA + p_s * (BM * KC)), srcA, A_STAGE_BYTES, full);
        bulk_g2s(smem_u32(sB + p_s * (BN * KC)), srcB, B_STAGE_BYTES, full);
        if (++p_s == STAGES) {
            p_s = 0;
            p_ph ^= 1u;
        }
        if (++p_kc == sh.nkc) {
            p_kc = 0;
            p_b += sh.Gs;
        }
        ++p_it;
    };
    if (producer)
        while (p_it < iters && p_it < STAGES - 1) produce();

    // ---------------------------------------------------- consumer warps
    const int wi = warp / WARPS_N, wj = warp % WARPS_N;
    const int gid = lane >> 2, tig = lane & 3;
    double acc[4][NJ][2], S[4][NJ][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            acc[i][j][0] = acc[i][j][1] = 0.0;
            if (!S_TMEM) S[i][j][0] = S[i][j][1] = 0.0;
        }
    double sq = 0.0;
    // S_TMEM: this thread's running sums at TMEM lane (warp % 4) * 32 + lane,
    // columns (warp / 4) * 128 + 32 i + [0, 32) for accumulator row block i
    const uint32_t s_t = S_TMEM ? s_tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128) : 0u;
    if (S_TMEM) {
        uint32_t z[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) z[e] = 0u;
#pragma unroll
        for (int i = 0; i < 4; ++i) tm_st32(s_t + 32 * i, z);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }

    const uint32_t full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[STAGES]);
    const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
    // per-lane fragment offsets (bytes) inside a stage: rows wi*32 + 8i + gid,
    // cols wj*32 + 8j + gid, granules (2 tig + h) ^ gid
    const uint32_t a_off = (uint32_t)((wi * 32 + gid) * KC * 8), b_off = (uint32_t)((wj * WN + gid) * KC * 8);
    const uint32_t g0 = (uint32_t)((((2 * tig) ^ gid) << 4)), g1 = (uint32_t)((((2 * tig + 1) ^ gid) << 4));
    int s = 0;
    uint32_t ph = 0;
    int64_t kc = 0;
    for (int64_t it = 0; it < iters; ++it) {
        mbar_wait(full0 + 8 * s, ph);
        const uint32_t a_st = a_base + s * A_STAGE_BYTES + a_off;
        const uint32_t b_st = b_base + s * B_STAGE_BYTES + b_off;
        if (S_TMEM) {
            // fragments in two halves (granules g0, g1): 32 + 32 DMMA-pairs' worth per half
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const uint32_t gg = hf ? g1 : g0;
                double2 af[4], bf[NJ];
#pragma unroll
                for (int i = 0; i < 4; ++i) af[i] = lds128(a_st + i * (8 * KC * 8) + gg);
#pragma unroll
                for (int j = 0; j < NJ; ++j) bf[j] = lds128(b_st + j * (8 * KC * 8) + gg);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i].x, bf[j].x);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i].y, bf[j].y);
            }
        } else {
        // all fragments of the stage first (16 x LDS.128), then 64 DMMAs
            double2 af0[4], bf0[NJ], af1[4], bf1[NJ];
    #pragma unroll
            for (int i = 0; i < 4; ++i) {
                af0[i] = lds128(a_st + i * (8 * KC * 8) + g0);
                af1[i] = lds128(a_st + i * (8 * KC * 8) + g1);
            }
    #pragma unroll
            for (int j = 0; j < NJ; ++j) {
                bf0[j] = lds128(b_st + j * (8 * KC * 8) + g0);
                bf1[j] = lds128(b_st + j * (8 * KC * 8) + g1);
            }
    #pragma unroll
            for (int i = 0; i < 4; ++i)
    #pragma unroll
                for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], af0[i].x, bf0[j].x);
    #pragma unroll
            for (int i = 0; i < 4; ++i)
    #pragma unroll
                for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], af0[i].y, bf0[j].y);
    #pragma unroll
            for (int i = 0; i < 4; ++i)
    #pragma unroll
                for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], af1[i].x, bf1[j].x);
    #pragma unroll
            for (int i = 0; i < 4; ++i)
    #pragma unroll
                for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], af1[i].y, bf1[j].y);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * s);
        if (producer && p_it < iters) produce();
        if (++s == STAGES) {
            s = 0;
            ph ^= 1u;
        }
        if (NL && kc + 1 == nla.pre_kc) {
            // the coarse prefix is complete: f(coarse) of this thread's fragments
            double* sc = nla.scratch + (int64_t)g * (4 * NJ * 2) * GEMM_THREADS + threadIdx.x;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        sc[(int64_t)((i * NJ + j) * 2 + e) * GEMM_THREADS] =
                            apply_target(nla.target, nla.tparam, __dmul_rn(nla.cscale, acc[i][j][e]));
        }
        if (++kc == sh.nkc) {
            kc = 0;
            if (SPLIT) {
                // one sample split along K (one sample per launch): carry the partial Y
                double* yp = ypart + (int64_t)tile * (BM * BN);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NJ; ++j) {
                        double2* q2 = reinterpret_cast<double2*>(yp + (wi * 32 + 8 * i + gid) * BN + wj * WN + 8 * j +
                                                                 2 * tig);
                        if (split_part >= 2) {
                            const double2 pv = *q2;
                            acc[i][j][0] = __dadd_rn(pv.x, acc[i][j][0]);
                            acc[i][j][1] = __dadd_rn(pv.y, acc[i][j][1]);
                        }
                        if (split_part <= 2) {
                            *q2 = make_double2(acc[i][j][0], acc[i][j][1]);
                            acc[i][j][0] = acc[i][j][1] = 0.0;
                        }
                    }
                if (split_part <= 2) continue;  // not the last segment: no epilogue yet
            }
            // sample boundary: fused level epilogue (Y^2 and running sum)
            if (S_TMEM) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    uint32_t r[32];
                    tm_ld32(s_t + 32 * i, r);
#pragma unroll
                    for (int j = 0; j < NJ; ++j)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const double y = NL ? nl_y(nla, g, i, j, e, acc[i][j][e]) : acc[i][j][e];
                            sq = __fma_rn(y, y, sq);
                            const int w = 2 * (2 * j + e);
                            const double v = __dadd_rn(__hiloint2double((int)r[w + 1], (int)r[w]), y);
                            r[w] = (uint32_t)__double2loint(v);
                            r[w + 1] = (uint32_t)__double2hiint(v);
                            acc[i][j][e] = 0.0;
                        }
                    tm_st32(s_t + 32 * i, r);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NJ; ++j)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const double y = NL ? nl_y(nla, g, i, j, e, acc[i][j][e]) : acc[i][j][e];
                            sq = __fma_rn(y, y, sq);
                            S[i][j][e] = __dadd_rn(S[i][j][e], y);
                            acc[i][j][e] = 0.0;
                        }
            }
        }
    }

    // partial outputs of this CTA (deterministic layout / order)
    double* out = part + (int64_t)g * (BM * BN);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint32_t r32[32];
        if (S_TMEM) tm_ld32(s_t + 32 * i, r32);
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int r = wi * 32 + 8 * i + gid;
            const int q = wj * WN + 8 * j + 2 * tig;
            const double v0 = S_TMEM ? __hiloint2double((int)r32[4 * j + 1], (int)r32[4 * j]) : S[i][j][0];
            const double v1 = S_TMEM ? __hiloint2double((int)r32[4 * j + 3], (int)r32[4 * j + 2]) : S[i][j][1];
            *reinterpret_cast<double2*>(out + r * BN + q) = make_double2(v0, v1);
        }
    }
    sq = warp_sum(sq);
    if (lane == 0) s_sq[warp] = sq;
    if (S_TMEM) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < CONSUMERS; ++w) t += s_sq[w];
        part_sq[g] = t;
    }
    if (S_TMEM && warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(S_TMEM_COLS));
    }
}

// total[cell] += sum over groups (fixed order) of the tile partials
template <int RBM, int RBN>
__global__ void k_reduce_tiles(const double* __restrict__ part, const double* __restrict__ part_sq, GemmShape sh,
                               int64_t rows, int64_t cols, double* __restrict__ total, double* __restrict__ total_sq) {
    const int64_t cells = rows * cols;
    for (int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cell < cells;
         cell += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = cell / cols, q = cell - r * cols;
        const int tile = (int)((r / RBM) * sh.tiles_n + q / RBN);
        const int64_t off = (r % RBM) * RBN + (q % RBN);
        double acc = 0.0;
        for (int grp = 0; grp < sh.Gs; ++grp) acc += part[(int64_t)(grp * sh.T + tile) * (RBM * RBN) + off];
        total[cell] += acc;
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        const double acc = warp_sum_array(part_sq, sh.T * sh.Gs, threadIdx.x);
        if (threadIdx.x == 0) *total_sq += acc;
    }
}

// ----------------------------------------------------- vector (config 1)

// one warp per sample: Y = sum_t w_t a_t b_t with a_t, b_t drawn at the
// sampled index from one Philox block (a takes z0, b takes z1)
__global__ void __launch_bounds__(256)
k_fused_inner(DevModel M, uint64_t seed, uint64_t tag, const int64_t* __restrict__ ks, int nb, int64_t c,
              int64_t cc, double w_fine, double w_coarse, double* __restrict__ y_out,
              uint32_t* __restrict__ idx_out, int target, double tparam) {
    const bool nl = target != MLSK_TARGET_IDENTITY;  // prefix / suffix apart (k_fused_inner_multi<true>)
    __shared__ __align__(16) double2 s_sc[256];
    __shared__ __align__(16) double2 s_lg[128];
    load_tables(s_sc, s_lg, M.tab);
    __syncthreads();
    Tables T = M.tab;
    T.sincos_d = reinterpret_cast<const double*>(s_sc);
    T.log_d = reinterpret_cast<const double*>(s_lg);
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nb; b += warps) {
        const uint64_t key = derive_seed(seed, tag, (uint64_t)ks[b]);
        double acc = 0.0, pre = 0.0;
        for (int64_t tp = lane; 2 * tp < c; tp += 32) {
            const u32x4 ri = philox((uint32_t)tp, 0, 0, MLSK_CTR_INDEX, key);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t t = 2 * tp + h;
                if (t >= c) break;
                const uint32_t ix = index_from_u64(h ? hi64(ri) : lo64(ri), M.n, M.log2n, M.cum);
                if (idx_out) idx_out[(int64_t)b * c + t] = ix;
                const int64_t j = (int64_t)ix - 1;
                const u32x4 r = philox((uint32_t)j, 0, 0, MLSK_CTR_A, key);
                double z0, z1;
                box_muller(lo64(r), hi64(r), z0, z1, T);
                const double a = __dadd_rn(M.mean_a[j], __dmul_rn(M.sd, z0));
                const double bb = __dadd_rn(M.mean_b[j], __dmul_rn(M.sd, z1));
                if (nl && t < cc) pre = __fma_rn(__dmul_rn(a, bb), w_fine, pre);
                else acc = __fma_rn(__dmul_rn(a, bb), t < cc ? w_coarse : w_fine, acc);
            }
        }
        acc = warp_sum(acc);
        if (nl) {
            pre = warp_sum(pre);
            double y = apply_target(target, tparam, __dadd_rn(pre, acc));
            if (cc > 0) y = __dsub_rn(y, apply_target(target, tparam, __dmul_rn((double)c / (double)cc, pre)));
            acc = y;
        }
        if (lane == 0) y_out[b] = acc;
    }
}

// single block: total += sum_b y_b, total_sq += sum_b y_b^2 (fixed order)
__global__ void k_reduce_inner(const double* __restrict__ y, int nb, double* total, double* total_sq) {
    __shared__ double s1[256], s2[256];
    double a = 0.0, q = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        a += y[b];
        q = __fma_rn(y[b], y[b], q);
    }
    s1[threadIdx.x] = a;
    s2[threadIdx.x] = q;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            s1[threadIdx.x] += s1[threadIdx.x + s];
            s2[threadIdx.x] += s2[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *total += s1[0];
        *total_sq += s2[0];
    }
}

// All levels of a round in one launch (config 1 is launch-bound: c = 8 .. 256).
// A part = one level's slice of the round.  A warp task is 32 / g
// replications of one part, g = the part's threads per replication (up to
// INNER_G, no more than its index pairs: level 0 of config 1 has c = 8, i.e. 4
// pairs, and 8 threads left half of them idle), lanes over index pairs,
// reduced within the g-lane group.
constexpr int INNER_MAX_PARTS = 16;
constexpr int INNER_G = 8;
struct InnerPart {
    uint64_t tag;
    int64_t c, cc;
    double w_fine, w_coarse;  // nonlinear targets: both n / c (prefix and suffix kept apart)
    int64_t ks_off;    // into the round's replication list
    int64_t y_off;     // first output slot (parts are contiguous)
    int64_t nb;
    int64_t task_off;  // first warp task
    int64_t k0;        // >= 0: the part's replications are k0, k0 + 1, ... (no index list read)
    uint64_t key_prefix;  // derive_prefix(seed, tag): one mix per replication instead of three
    int g;             // threads per replication (power of two <= INNER_G)
    double* total;
    double* total_sq;
};
struct InnerParts {
    int n;
    int64_t tasks;
    InnerPart p[INNER_MAX_PARTS];
};

inline int inner_group(int64_t c) {
    int g = 1;
    while (g < INNER_G && 2 * g < c) g *= 2;  // g <= ceil(c / 2) index pairs
    return g;
}

// NL (nonlinear target f1 / f2, models.cpp:99-117): the prefix and suffix
// sums are kept apart, Y = f((n/c)(S_pre + S_suf)) - f((n/cc) S_pre) per
// replication (estimators.cpp:78-80), instead of one signed sum.
// (256, 3): <= 80 registers, three CTAs per SM (uncapped: 118 registers, two
// CTAs per SM, "wait" 35% of the stall samples at 24% warps active).  Measured
// per step: 1 / 3 / 4 / 5 CTAs per SM 0.351 / 0.340 / 0.349 / 0.359 ms.
#ifndef MLSK_INNER_MINB
#define MLSK_INNER_MINB 3
#endif
template <bool NL>
__global__ void __launch_bounds__(256, MLSK_INNER_MINB)
k_fused_inner_multi(DevModel M, uint64_t seed, const int64_t* __restrict__ ks, InnerParts P,
                    double* __restrict__ y_out, int target, double tparam) {
    __shared__ __align__(16) double2 s_sc[256];
    __shared__ __align__(16) double2 s_lg[128];
    load_tables(s_sc, s_lg, M.tab);
    __syncthreads();
    Tables T = M.tab;
    T.sincos_d = reinterpret_cast<const double*>(s_sc);
    T.log_d = reinterpret_cast<const double*>(s_lg);
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t task = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; task < P.tasks; task += warps) {
        int pi = 0;  // warp-uniform
        while (pi + 1 < P.n && task >= P.p[pi + 1].task_off) ++pi;
        const InnerPart q = P.p[pi];  // a register copy (a reference re-read the param bank per use)
        MLSK_DCHECK(task >= q.task_off && q.g >= 1 && q.g <= INNER_G);
        const int g = q.g, gl = lane & (g - 1);
        const int64_t b = (task - q.task_off) * (32 / g) + lane / g;
        const bool live = b < q.nb;
        double acc = 0.0, pre = 0.0;
        if (live) {
            const int64_t k = q.k0 >= 0 ? q.k0 + b : ks[q.ks_off + b];
            const uint64_t key = derive_from_prefix(q.key_prefix, (uint64_t)k);  // = derive_seed(seed, tag, k)
            for (int64_t tp = gl; 2 * tp < q.c; tp += g) {
                const u32x4 ri = philox((uint32_t)tp, 0, 0, MLSK_CTR_INDEX, key);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t t = 2 * tp + h;
                    if (t >= q.c) break;
                    const uint32_t ix = index_from_u64(h ? hi64(ri) : lo64(ri), M.n, M.log2n, M.cum);
                    const int64_t j = (int64_t)ix - 1;
                    const u32x4 r = philox((uint32_t)j, 0, 0, MLSK_CTR_A, key);
                    double z0, z1;
                    box_muller(lo64(r), hi64(r), z0, z1, T);
                    const double a = __dadd_rn(M.mean_a[j], __dmul_rn(M.sd, z0));
                    const double bb = __dadd_rn(M.mean_b[j], __dmul_rn(M.sd, z1));
                    if (NL && t < q.cc) pre = __fma_rn(__dmul_rn(a, bb), q.w_fine, pre);
                    else acc = __fma_rn(__dmul_rn(a, bb), t < q.cc ? q.w_coarse : q.w_fine, acc);
                }
            }
        }
        for (int o = g / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (NL) {
            for (int o = g / 2; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
            if (live && gl == 0) {
                // fine = (n/c)(S_pre + S_suf), coarse = (n/cc) S_pre = (c/cc) (n/c) S_pre
                double y = apply_target(target, tparam, __dadd_rn(pre, acc));
                if (q.cc > 0)
                    y = __dsub_rn(y, apply_target(target, tparam, __dmul_rn((double)q.c / (double)q.cc, pre)));
                acc = y;
            }
        }
        if (live && gl == 0) y_out[q.y_off + b] = acc;
    }
}

// INNER_RB blocks per part, each over a fixed contiguous range of the part's
// replications; the last block of a part to finish adds the INNER_RB partials
// in block order (fixed order: bit-identical reruns).  One block per part
// (the previous form) serialised 0.5 M replications of level 0 on one SM.
#ifndef MLSK_INNER_RB
#define MLSK_INNER_RB 64
#endif
constexpr int INNER_RB = MLSK_INNER_RB;
__global__ void __launch_bounds__(256)
k_reduce_inner_multi(const double* __restrict__ y, InnerParts P, double* __restrict__ part,
                     unsigned* __restrict__ done) {
    __shared__ double s1[256], s2[256];
    __shared__ bool last;
    const int pi = blockIdx.y;
    const InnerPart& q = P.p[pi];
    const int64_t b0 = q.nb * blockIdx.x / INNER_RB, b1 = q.nb * (blockIdx.x + 1) / INNER_RB;
    double a = 0.0, r = 0.0;
    for (int64_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
        const double v = y[q.y_off + b];
        a += v;
        r = __fma_rn(v, v, r);
    }
    s1[threadIdx.x] = a;
    s2[threadIdx.x] = r;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st) {
            s1[threadIdx.x] += s1[threadIdx.x + st];
            s2[threadIdx.x] += s2[threadIdx.x + st];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[(pi * INNER_RB + blockIdx.x) * 2] = s1[0];
        part[(pi * INNER_RB + blockIdx.x) * 2 + 1] = s2[0];
        __threadfence();
        last = atomicAdd(&done[pi], 1u) == INNER_RB - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        const volatile double* vp = part + pi * INNER_RB * 2;
        double t = 0.0, t2 = 0.0;
        for (int k = 0; k < INNER_RB; ++k) {
            t += vp[2 * k];
            t2 += vp[2 * k + 1];
        }
        *q.total += t;
        *q.total_sq += t2;
        done[pi] = 0;  // ready for the next launch (stream-ordered)
    }
}

int sm_count() {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}


// RNG roofline of the inner-product path (config 1): exactly the per-index
// work of k_fused_inner_multi -- half an index Philox block, the (a, b)
// Philox block, one Box-Muller pair, two mean gathers, one fma -- with no
// level bookkeeping, replication reduction or launch boundary.  Its
// index-samples / s is the ceiling the fused inner kernel is measured against.
__global__ void __launch_bounds__(256) k_index_rate(DevModel M, uint64_t seed, int64_t pairs, double* sink) {
    __shared__ __align__(16) double2 s_sc[256];
    __shared__ __align__(16) double2 s_lg[128];
    load_tables(s_sc, s_lg, M.tab);
    __syncthreads();
    Tables T = M.tab;
    T.sincos_d = reinterpret_cast<const double*>(s_sc);
    T.log_d = reinterpret_cast<const double*>(s_lg);
    const uint64_t key = derive_seed(seed, blockIdx.x, threadIdx.x);
    double acc = 0.0;
    for (int64_t tp = 0; tp < pairs; ++tp) {
        const u32x4 ri = philox((uint32_t)tp, 0, 0, MLSK_CTR_INDEX, key);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t ix = index_from_u64(h ? hi64(ri) : lo64(ri), M.n, M.log2n, M.cum);
            const int64_t j = (int64_t)ix - 1;
            const u32x4 r = philox((uint32_t)j, 0, 0, MLSK_CTR_A, key);
            double z0, z1;
            box_muller(lo64(r), hi64(r), z0, z1, T);
            const double a = __dadd_rn(M.mean_a[j], __dmul_rn(M.sd, z0));
            const double bb = __dadd_rn(M.mean_b[j], __dmul_rn(M.sd, z1));
            acc = __fma_rn(__dmul_rn(a, bb), 0.5, acc);
        }
    }
    if (acc == 1234.5678) sink[0] = acc;  // keeps the loop
}

}  // namespace

bool tc_supported(const Model& M, int target);                                   // mlsk_tc.cu

// fp64 gauss models (configs 1-2) take any target: identity as one signed
// contraction, f1 / f2 with the prefix and suffix kept apart (k_fused_inner*
// and k_gemm_f64<NL>); the fp32 engine is identity-only (tc_supported).
bool fused_supported(const Model& M, int target) {
    return (M.dm.stream == MLSK_STREAM_PHILOX && M.dm.kind == MLSK_MODEL_GAUSS_MEAN && M.dm.dtype == MLSK_F64) ||
           tc_supported(M, target);
}

namespace {

class F64Engine final : public PanelEngine {
   public:
    F64Engine(const Model& M, Workspace& ws, int target, double tparam)
        : M_(M), ws_(ws), target_(target), tparam_(tparam), nl_(target != MLSK_TARGET_IDENTITY) {
        nsm_ = sm_count();
        MP_ = (M.rows + BM - 1) / BM * BM;
        PP_ = (M.cols + BN - 1) / BN * BN;
        tiles_n_ = (int)(PP_ / BN);
        T_ = (int)(MP_ / BM) * tiles_n_;
        Gs_ = std::max(1, nsm_ / T_);
        smem_ = STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + 2 * STAGES * 8;
        const int smem = smem_;
        once_per_device((const void*)&k_gemm_f64<false, false>, [smem] {
            for (auto f : {k_gemm_f64<false, false>, k_gemm_f64<true, false>, k_gemm_f64<false, true>})
                MLSK_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            MLSK_CUDA(cudaFuncSetAttribute(k_gen_panels_f64, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           GEN_DYN_SMEM));
        });
        ws_.partial.ensure((size_t)T_ * Gs_ * (BM * BN) + (size_t)T_ * Gs_);
        int gen_occ = 0;
        MLSK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&gen_occ, k_gen_panels_f64, GEN_THREADS, GEN_DYN_SMEM));
        gen_occ = std::max(gen_occ, 1);
        gen_ctas_ = nsm_ * gen_occ;  // one full wave of the grid-stride generator
        if (const char* e = getenv("MLSK_GEN_CTAS_PER_SM")) gen_ctas_ = nsm_ * std::max(1, atoi(e));  // experiments
    }
    int64_t chunk_cols() const override { return KC; }
    int64_t chunk_bytes() const override { return (MP_ + PP_) * KC * 8; }
    bool splits_k() const override { return true; }
    int64_t group_size() const override { return Gs_; }
    void gen(cudaStream_t s, uint64_t seed, uint64_t tag, const int64_t* ks, int nb, int64_t c, int64_t cc,
             double w_fine, double w_coarse, void* panels, uint32_t* idx, const KRange& kr) override {
        const int64_t k = kr.nkc >= 0 ? kr.nkc : nchunks(c, cc);
        double* Apan = static_cast<double*>(panels);
        double* Bpan = Apan + (size_t)nb * k * MP_ * KC;
        Prof p("gen_panels_f64", s);
        k_gen_panels_f64<<<(int)std::min<int64_t>((int64_t)nb * k, (int64_t)gen_ctas_), GEN_THREADS, GEN_DYN_SMEM, s>>>(
            M_.dm, seed, tag, ks, nb, c, cc, w_fine, w_coarse, MP_, PP_, k, kr.kc0, Apan, Bpan, idx, pcc(cc), kr.mk,
            kr.mk_stride, kr.mk_info);
        launched();
    }
    void gemm(cudaStream_t s, const void* panels, int nb, int64_t c, int64_t cc, double, double, LevelState& st,
              const KRange& kr) override {
        const int64_t k = kr.nkc >= 0 ? kr.nkc : nchunks(c, cc);
        const double* Apan = static_cast<const double*>(panels);
        const double* Bpan = Apan + (size_t)nb * k * MP_ * KC;
        double* part = ws_.partial.p;
        double* part_sq = part + (size_t)T_ * Gs_ * (BM * BN);
        double* ypart = nullptr;
        if (kr.part != 0) {
            ws_.ypart64.ensure((size_t)T_ * BM * BN);  // the carried partial Y of a split sample
            ypart = ws_.ypart64.p;
        }
        GemmShape sh{nb, k, MP_, PP_, T_, Gs_, tiles_n_};
        {
            Prof p("gemm_f64", s);
            NlArgs nla{target_, tparam_, 0, 1.0, nullptr};
            if (nl_) {
                if (kr.part != 0) throw Error(MLSK_EINVAL, "fused engine: nonlinear targets need whole level-samples");
                nla.pre_kc = cc > 0 ? (cc + KC - 1) / KC : 0;
                nla.cscale = cc > 0 ? (double)c / (double)cc : 1.0;
                ws_.nl_scratch.ensure((size_t)T_ * Gs_ * (4 * NJ * 2) * GEMM_THREADS);
                nla.scratch = ws_.nl_scratch.p;
                k_gemm_f64<false, true><<<T_ * Gs_, GEMM_THREADS, smem_, s>>>(Apan, Bpan, sh, part, part_sq, 0,
                                                                              nullptr, nla);
            } else if (kr.part == 0)
                k_gemm_f64<false, false><<<T_ * Gs_, GEMM_THREADS, smem_, s>>>(Apan, Bpan, sh, part, part_sq, 0,
                                                                               nullptr, nla);
            else
                k_gemm_f64<true, false><<<T_ * Gs_, GEMM_THREADS, smem_, s>>>(Apan, Bpan, sh, part, part_sq, kr.part,
                                                                              ypart, nla);
        }
        if (kr.part == 1 || kr.part == 2) {  // the sample completes in a later launch
            launched();
            return;
        }
        const int64_t cells = M_.rows * M_.cols;
        {
            Prof p("reduce_tiles", s);
            k_reduce_tiles<BM, BN><<<(int)std::min<int64_t>((cells + 255) / 256, (int64_t)nsm_ * 8), 256, 0, s>>>(
                part, part_sq, sh, M_.rows, M_.cols, st.total(), st.total_sq());
        }
        launched(2);
    }

    // merged sampled columns: summed weights folded into B (identity target)
    int merge_mode(int64_t, int64_t, double, double) const override { return nl_ ? 0 : 1; }

    // nonlinear targets: the coarse prefix padded to whole K-chunks
    int64_t nchunks(int64_t c, int64_t cc) const override {
        return nl_ ? (cc + KC - 1) / KC + (c - cc + KC - 1) / KC : (c + KC - 1) / KC;
    }

   private:
    int64_t pcc(int64_t cc) const { return nl_ ? (cc + KC - 1) / KC * KC : cc; }
    const Model& M_;
    Workspace& ws_;
    int target_;
    double tparam_;
    bool nl_;
    int nsm_, T_, Gs_, tiles_n_, smem_, gen_ctas_;
    int64_t MP_, PP_;
};

std::unique_ptr<PanelEngine> make_f64_engine(const Model& M, Workspace& ws, int target, double tparam) {
    return std::unique_ptr<PanelEngine>(new F64Engine(M, ws, target, tparam));
}

// ks[dst + i] = k0 + i for i < count, runs sorted by dst and covering [0, total)
struct KsRun {
    int64_t k0, count, dst;
};
__global__ void k_expand_ks(const KsRun* __restrict__ runs, int nruns, int64_t total, int64_t* __restrict__ ks) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nruns - 1;  // last run with dst <= e
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (runs[mid].dst <= e) lo = mid;
            else hi = mid - 1;
        }
        MLSK_DCHECK(runs[lo].dst <= e && e < runs[lo].dst + runs[lo].count);
        ks[e] = runs[lo].k0 + (e - runs[lo].dst);
    }
}

// ------------------------------------------- merged sampled columns pre-pass
//
// (KRange, mlsk_internal.h.)  k_mk_count draws every index of a group of
// samples and counts, per sample and column j, how often j falls in the coarse
// prefix (high word) and in the suffix (low word): integer atomics, so the
// counts -- and everything derived from them -- are the same in every run.
// k_mk_tiles / k_mk_scan / k_mk_write turn a sample's counts into its list,
// ordered by j (tiles of 4096 columns: counts, exclusive scan, ordered writes):
//   mode 1: one entry per column with W_j = cnt_f w_fine + cnt_c w_coarse != 0;
//   mode 2: one entry per column with cnt_f != cnt_c carrying the column
//           scale sqrt(|cnt_f - cnt_c|) (Y = sum_j sign_j (s_j z_j)(s_j z_j)^T |w|),
//           the negative ones (cnt_f < cnt_c) first, padded to whole K-chunks.
// The write pass clears the counts it read; the scan raises the job's maximum
// chunk count, which the host reads once per round to size the launches.
constexpr int MK_T = 256, MK_ITEMS = 16, MK_TILE = MK_T * MK_ITEMS;
constexpr int MK_MAX_JOBS = 64;  // merged levels per round

__global__ void __launch_bounds__(256)
k_mk_count(DevModel M, uint64_t seed, uint64_t tag, const int64_t* __restrict__ ks, int64_t nb, int64_t c, int64_t cc,
           unsigned long long* __restrict__ cnt) {
    const int64_t hp = (c + 1) / 2;  // index pairs per sample (one Philox block each)
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nb * hp;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / hp, tp = e - b * hp;
        const uint64_t key = derive_seed(seed, tag, (uint64_t)ks[b]);
        const u32x4 r = philox((uint32_t)tp, 0, 0, MLSK_CTR_INDEX, key);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t t = 2 * tp + h;
            if (t < c) {
                const uint32_t ix = index_from_u64(h ? hi64(r) : lo64(r), M.n, M.log2n, M.cum);
                atomicAdd(cnt + b * M.n + (ix - 1), t < cc ? (1ull << 32) : 1ull);
            }
        }
    }
}

// entries column j contributes and whether they belong to the negative group
__device__ __forceinline__ int mk_entries(unsigned long long v, int mode, double w_fine, double w_coarse, bool& neg) {
    const int64_t cf = (int64_t)(v & 0xffffffffull), ccn = (int64_t)(v >> 32);
    neg = false;
    if (v == 0) return 0;
    if (mode == 2) {  // |w_coarse| == |w_fine|, w_coarse < 0 (shared_panel)
        neg = cf < ccn;
        return cf != ccn ? 1 : 0;
    }
    if (w_coarse == -w_fine) return cf != ccn ? 1 : 0;  // exact cancellation (M = 2)
    return __fma_rn((double)cf, w_fine, __dmul_rn((double)ccn, w_coarse)) != 0.0 ? 1 : 0;
}

// (neg, pos) entry counts of this thread's MK_ITEMS consecutive columns
__device__ __forceinline__ void mk_thread_counts(const unsigned long long* __restrict__ my, int64_t n, int64_t j0,
                                                 int mode, double w_fine, double w_coarse,
                                                 unsigned long long (&v)[MK_ITEMS], int (&en)[MK_ITEMS],
                                                 bool (&ng)[MK_ITEMS], int& tn, int& tp) {
    tn = tp = 0;
    if (j0 + MK_ITEMS <= n) {
#pragma unroll
        for (int i = 0; i < MK_ITEMS; i += 2) {
            const ulonglong2 q = *reinterpret_cast<const ulonglong2*>(my + j0 + i);
            v[i] = q.x;
            v[i + 1] = q.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < MK_ITEMS; ++i) v[i] = j0 + i < n ? my[j0 + i] : 0ull;
    }
#pragma unroll
    for (int i = 0; i < MK_ITEMS; ++i) {
        en[i] = mk_entries(v[i], mode, w_fine, w_coarse, ng[i]);
        if (ng[i]) tn += en[i];
        else tp += en[i];
    }
}

// per (tile of MK_TILE columns, sample): entry counts of the tile
__global__ void __launch_bounds__(MK_T)
k_mk_tiles(const unsigned long long* __restrict__ cnt, int64_t n, int mode, double w_fine, double w_coarse,
           int2* __restrict__ tile_cnt) {
    __shared__ int s_neg[MK_T / 32], s_pos[MK_T / 32];
    const int tile = blockIdx.x, b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long v[MK_ITEMS];
    int en[MK_ITEMS];
    bool ng[MK_ITEMS];
    int tn, tp;
    mk_thread_counts(cnt + (int64_t)b * n, n, (int64_t)tile * MK_TILE + (int64_t)tid * MK_ITEMS, mode, w_fine,
                     w_coarse, v, en, ng, tn, tp);
    for (int o = 16; o > 0; o >>= 1) {
        tn += __shfl_xor_sync(0xffffffffu, tn, o);
        tp += __shfl_xor_sync(0xffffffffu, tp, o);
    }
    if (lane == 0) {
        s_neg[warp] = tn;
        s_pos[warp] = tp;
    }
    __syncthreads();
    if (tid == 0) {
        int a = 0, q = 0;
        for (int w = 0; w < MK_T / 32; ++w) {
            a += s_neg[w];
            q += s_pos[w];
        }
        tile_cnt[(int64_t)b * gridDim.x + tile] = make_int2(a, q);
    }
}

// per sample: exclusive scan of its tiles' counts (in place), its (len, neg_kc),
// the padding of the negative group and the job's maximum chunk count
__global__ void __launch_bounds__(MK_T)
k_mk_scan(int2* __restrict__ tile_cnt, int tiles, int kcols, MkEntry* __restrict__ list, int64_t stride,
          MkInfo* __restrict__ info, int32_t* __restrict__ job_max) {
    __shared__ int s_neg[MK_T / 32], s_pos[MK_T / 32];
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int2* my = tile_cnt + (int64_t)b * tiles;
    int base_n = 0, base_p = 0;
    for (int t0 = 0; t0 < tiles; t0 += MK_T) {
        const int t = t0 + tid;
        const int2 cv = t < tiles ? my[t] : make_int2(0, 0);
        int xn = cv.x, xp = cv.y;
        for (int o = 1; o < 32; o <<= 1) {
            const int yn = __shfl_up_sync(0xffffffffu, xn, o), yp = __shfl_up_sync(0xffffffffu, xp, o);
            if (lane >= o) {
                xn += yn;
                xp += yp;
            }
        }
        __syncthreads();
        if (lane == 31) {
            s_neg[warp] = xn;
            s_pos[warp] = xp;
        }
        __syncthreads();
        int wn = 0, wp = 0, alln = 0, allp = 0;
        for (int w = 0; w < MK_T / 32; ++w) {
            if (w < warp) {
                wn += s_neg[w];
                wp += s_pos[w];
            }
            alln += s_neg[w];
            allp += s_pos[w];
        }
        if (t < tiles) my[t] = make_int2(base_n + wn + xn - cv.x, base_p + wp + xp - cv.y);
        base_n += alln;
        base_p += allp;
    }
    const int negpad = (base_n + kcols - 1) / kcols * kcols;
    const int len = negpad + base_p;
    MLSK_DCHECK((int64_t)len <= stride);
    if (tid == 0) {
        info[b] = MkInfo{len, negpad / kcols};
        atomicMax(job_max, (len + kcols - 1) / kcols);
    }
    MkEntry* out = list + (int64_t)b * stride;
    for (int q = base_n + tid; q < negpad; q += MK_T) out[q] = MkEntry{-1, 0, 0.0};
}

// per (tile, sample): the tile's entries, ordered by column, at their offsets;
// the counts it read are cleared for the next group
__global__ void __launch_bounds__(MK_T)
k_mk_write(unsigned long long* __restrict__ cnt, int64_t n, int mode, double w_fine, double w_coarse, int kcols,
           const int2* __restrict__ tile_off, const MkInfo* __restrict__ info, MkEntry* __restrict__ list,
           int64_t stride) {
    __shared__ int s_neg[MK_T / 32], s_pos[MK_T / 32];
    const int tile = blockIdx.x, b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long* my = cnt + (int64_t)b * n;
    MkEntry* out = list + (int64_t)b * stride;
    const int64_t j0 = (int64_t)tile * MK_TILE + (int64_t)tid * MK_ITEMS;
    unsigned long long v[MK_ITEMS];
    int en[MK_ITEMS];
    bool ng[MK_ITEMS];
    int tn, tp;
    mk_thread_counts(my, n, j0, mode, w_fine, w_coarse, v, en, ng, tn, tp);
#pragma unroll
    for (int i = 0; i < MK_ITEMS; ++i)
        if (v[i]) my[j0 + i] = 0ull;
    int xn = tn, xp = tp;
    for (int o = 1; o < 32; o <<= 1) {
        const int yn = __shfl_up_sync(0xffffffffu, xn, o), yp = __shfl_up_sync(0xffffffffu, xp, o);
        if (lane >= o) {
            xn += yn;
            xp += yp;
        }
    }
    if (lane == 31) {
        s_neg[warp] = xn;
        s_pos[warp] = xp;
    }
    __syncthreads();
    int wn = 0, wp = 0;
    for (int w = 0; w < warp; ++w) {
        wn += s_neg[w];
        wp += s_pos[w];
    }
    const int2 off = tile_off[(int64_t)b * gridDim.x + tile];
    int on = off.x + wn + xn - tn, op = info[b].neg_kc * kcols + off.y + wp + xp - tp;
#pragma unroll
    for (int i = 0; i < MK_ITEMS; ++i) {
        if (en[i] == 0) continue;
        const int64_t cf = (int64_t)(v[i] & 0xffffffffull), ccn = (int64_t)(v[i] >> 32);
        MkEntry e;
        e.j = (int32_t)(j0 + i);
        e.reps = (int32_t)(cf > ccn ? cf - ccn : ccn - cf);
        // mode 2: the signed column scale sqrt(|cnt_f - cnt_c|) (the panel column is
        // scaled, the sign is the chunk's negate bit); mode 1: the summed weight
        e.w = mode == 2 ? (ng[i] ? -sqrt((double)e.reps) : sqrt((double)e.reps))
                        : __fma_rn((double)cf, w_fine, __dmul_rn((double)ccn, w_coarse));
        int& o = ng[i] ? on : op;
        out[o++] = e;
    }
}

constexpr int NBUF = 3;  // panel buffers in flight (gen i+1, i+2 while GEMM i)

// Engine-private pipeline state kept in the Workspace across rounds.
struct Pipe {
    cudaStream_t s_gen = nullptr, s_mm = nullptr;
    cudaEvent_t start = nullptr, end = nullptr, staged = nullptr;
    cudaEvent_t gen_done[NBUF] = {}, mm_done[NBUF] = {};
    bool used[NBUF] = {};
    DevArray<double> panels[NBUF];
    DevArray<uint32_t> idx[NBUF];
    DevArray<int64_t> ks;      // all replication indices of the round (expanded on the device)
    DevArray<KsRun> runs;      // the round's replication runs
    KsRun* runs_host = nullptr;  // pinned staging
    size_t runs_cap = 0;
    DevArray<double> part;
    DevArray<double> red_part;    // k_reduce_inner_multi: per-block partials
    DevArray<unsigned> red_done;  // per-part finished-block counters (self-resetting)
    bool staged_pending = false;
    // merged sampled columns (pre-pass state)
    DevArray<unsigned long long> mk_cnt;  // [group sample][n] packed counts, all zero between uses
    DevArray<int2> mk_tile;               // [group sample][tile] entry counts, then offsets
    DevArray<MkEntry> mk_list;
    DevArray<MkInfo> mk_info[2];          // by round parity: the last round's GEMMs may still read theirs
    int mk_parity = 0;
    cudaEvent_t mk_info_done[2] = {};     // end of the last round that used mk_info[parity]
    bool mk_info_used[2] = {};
    uint64_t last_serial = 0;             // model of the last matrix round (cross-round overlap)
    DevArray<int32_t> mk_max;             // per merged job: maximum K-chunks over its samples
    int32_t* mk_max_host = nullptr;       // pinned
    cudaEvent_t mk_done = nullptr;
    bool ran = false;                     // a round's end event has been recorded
    uint64_t batch_seq = 0;               // batches launched so far (panel buffer rotation)

    void ensure_inner_red() {
        if (red_done.p) return;
        red_part.ensure((size_t)INNER_MAX_PARTS * INNER_RB * 2);
        red_done.ensure(INNER_MAX_PARTS);
        MLSK_CUDA(cudaMemsetAsync(red_done.p, 0, INNER_MAX_PARTS * sizeof(unsigned), s_gen));
    }

    Pipe() {
        int lo = 0, hi = 0;
        MLSK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        MLSK_CUDA(cudaStreamCreateWithPriority(&s_mm, cudaStreamNonBlocking, hi));   // GEMM: highest
        MLSK_CUDA(cudaStreamCreateWithPriority(&s_gen, cudaStreamNonBlocking, lo));  // generator: lowest
        MLSK_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
        MLSK_CUDA(cudaEventCreateWithFlags(&end, cudaEventDisableTiming));
        MLSK_CUDA(cudaEventCreateWithFlags(&staged, cudaEventDisableTiming));
        MLSK_CUDA(cudaEventCreateWithFlags(&mk_done, cudaEventDisableTiming));
        for (int i = 0; i < 2; ++i) MLSK_CUDA(cudaEventCreateWithFlags(&mk_info_done[i], cudaEventDisableTiming));
        MLSK_CUDA(cudaMallocHost(&mk_max_host, MK_MAX_JOBS * sizeof(int32_t)));
        for (int i = 0; i < NBUF; ++i) {
            MLSK_CUDA(cudaEventCreateWithFlags(&gen_done[i], cudaEventDisableTiming));
            MLSK_CUDA(cudaEventCreateWithFlags(&mm_done[i], cudaEventDisableTiming));
        }
    }
    ~Pipe() {
        if (s_gen) cudaStreamSynchronize(s_gen);
        if (s_mm) cudaStreamSynchronize(s_mm);
        for (int i = 0; i < NBUF; ++i) {
            cudaEventDestroy(gen_done[i]);
            cudaEventDestroy(mm_done[i]);
        }
        cudaEventDestroy(start);
        cudaEventDestroy(end);
        cudaEventDestroy(staged);
        cudaEventDestroy(mk_done);
        for (int i = 0; i < 2; ++i) cudaEventDestroy(mk_info_done[i]);
        if (mk_max_host) cudaFreeHost(mk_max_host);
        if (runs_host) cudaFreeHost(runs_host);
        if (s_gen) cudaStreamDestroy(s_gen);
        if (s_mm) cudaStreamDestroy(s_mm);
    }
    // Replication lists go to the device as runs of consecutive k (one run per
    // level at world = 1, one per owned 64-chunk when sharded) and are expanded
    // there: a config-1 round of 1 M level-samples otherwise spent ~4 ms of host
    // time building and copying 8 MB of indices per step.
    void stage_ks(const std::vector<KsRun>& h, int64_t total, cudaStream_t s) {
        if (staged_pending) MLSK_CUDA(cudaEventSynchronize(staged));  // previous round's copy done
        if (h.size() > runs_cap) {
            if (runs_host) cudaFreeHost(runs_host);
            runs_cap = std::max<size_t>(h.size(), 1 << 10);
            MLSK_CUDA(cudaMallocHost(&runs_host, runs_cap * sizeof(KsRun)));
        }
        std::memcpy(runs_host, h.data(), h.size() * sizeof(KsRun));
        runs.ensure(h.size());
        ks.ensure((size_t)total);
        MLSK_CUDA(cudaMemcpyAsync(runs.p, runs_host, h.size() * sizeof(KsRun), cudaMemcpyHostToDevice, s));
        MLSK_CUDA(cudaEventRecord(staged, s));
        staged_pending = true;
        const int64_t grid = std::min<int64_t>((total + 255) / 256, 4096);
        k_expand_ks<<<(int)grid, 256, 0, s>>>(runs.p, (int)h.size(), total, ks.p);
        launched();
    }
};

Pipe& pipe_of(Workspace& ws) {
    if (!ws.fused) ws.fused = std::shared_ptr<void>(new Pipe(), [](void* p) { delete static_cast<Pipe*>(p); });
    return *static_cast<Pipe*>(ws.fused.get());
}

// MLSK_SERIAL=1 serialises generator and GEMM (diagnostics: per-kernel
// standalone durations).
bool serial_mode() {
    static const bool v = [] {
        const char* e = getenv("MLSK_SERIAL");
        return e && e[0] == '1';
    }();
    return v;
}

struct Batch {
    size_t job;
    int64_t off;  // into the job's replication list
    int nb;
    int64_t ks_off;  // into the round's device ks array
    KRange kr;       // K-chunk range (split samples)
};

// A level of the round that runs on merged sampled columns.
struct MergeJob {
    int mode;
    int64_t stride;      // list entries per sample
    size_t list_off;     // into Pipe::mk_list / mk_info (entries / samples)
    size_t info_off;
    int64_t nk;          // merged K-chunks (maximum over the job's samples), from the pre-pass
};

// MLSK_MERGE=0 turns merged sampled columns off; MLSK_MERGE_MIN_DEN=d merges
// the levels with c >= n / d instead of the levels where it pays (merge_pays)
// (read every round: tests switch them in-process)
bool merge_enabled() {
    const char* e = getenv("MLSK_MERGE");
    return !(e && e[0] == '0');
}
int64_t merge_min_den() {
    const char* e = getenv("MLSK_MERGE_MIN_DEN");
    return e ? std::max<int64_t>(1, atoll(e)) : int64_t(16);
}
// Is merging worth its pre-pass for a level of c draws (coarse prefix cc) from n
// columns, K-chunks of kcols?  The expected number of surviving columns is
// n (1 - e^{-l} I_0(l)), l = c / n, when the prefix is half the draws with the
// opposite weight (Skellam(l/2, l/2) multiplicity != 0), n (1 - e^{-l}) when
// only duplicates merge; the launches are sized by the maximum over the level's
// samples (~ mean + 3 sigma, sigma^2 <= the merged-away count) in whole chunks
// (+ one chunk of padding per sign group).  Merge when that saves at least 3%
// of the chunks: at config 2's c = 256 (16 chunks, 244.5 expected columns) it
// saves none and the pre-pass is a net loss.  MLSK_MERGE_MIN_DEN set: the plain
// c >= n / d rule (tests force merging with a large d).
bool merge_pays(int64_t c, int64_t cc, int64_t n, int64_t kcols, bool cancels, int groups) {
    if (getenv("MLSK_MERGE_MIN_DEN")) return c * merge_min_den() >= n;
    if (c * 64 < n) return false;
    const double l = (double)c / (double)n;
    double keep;
    if (cc > 0 && cancels && 2 * cc == c) {
        double i0 = 0.0, term = 1.0;  // I_0(l) = sum (l/2)^{2k} / (k!)^2
        for (int k = 1; k < 40; ++k) {
            i0 += term;
            term *= (l / 2) * (l / 2) / ((double)k * (double)k);
        }
        keep = (double)n * (1.0 - std::exp(-l) * i0);
    } else {
        keep = (double)n * (1.0 - std::exp(-l));  // distinct columns
    }
    const double away = std::max(0.0, (double)c - keep);
    const double worst = keep + 3.0 * std::sqrt(away);
    const double chunks = std::ceil(worst / (double)kcols) + (groups - 1);
    const double full = (double)((c + kcols - 1) / kcols);
    return chunks <= 0.97 * full && chunks <= full - 1.0;
}

}  // namespace

void fused_run_round(const RunArgs& a, std::vector<FusedJob>& jobs) {
    const Model& M = *a.model;
    Workspace& ws = *a.ws;
    Pipe& P = pipe_of(ws);
    const int sms = sm_count();
    const double n = (double)M.desc.n;
    // nonlinear target: fine and coarse kept apart (uniform weights n / c)
    const bool nl = a.target != MLSK_TARGET_IDENTITY;

    // replication lists of all jobs as runs of consecutive k, expanded on the
    // device once per round (job j's list starts at job_off[j])
    std::vector<KsRun> runs;
    std::vector<int64_t> job_off(jobs.size()), job_cnt(jobs.size(), 0);
    int64_t all = 0;
    for (size_t j = 0; j < jobs.size(); ++j) {
        job_off[j] = all;
        for (const auto& sg : jobs[j].segs) {
            if (sg.count <= 0) continue;
            if (!runs.empty() && job_cnt[j] > 0 && runs.back().k0 + runs.back().count == sg.k0)
                runs.back().count += sg.count;
            else
                runs.push_back({sg.k0, sg.count, all});
            all += sg.count;
            job_cnt[j] += sg.count;
        }
    }
    if (all == 0) return;
    bool any_probe = false;
    for (const auto& job : jobs) any_probe = any_probe || job.probe_host;
    // host copies of the lists only for the coupling probe (which k is < probe_k)
    std::vector<std::vector<int64_t>> jks(any_probe ? jobs.size() : 0);
    if (any_probe)
        for (size_t j = 0; j < jobs.size(); ++j)
            for (const auto& sg : jobs[j].segs)
                for (int64_t k = 0; k < sg.count; ++k) jks[j].push_back(sg.k0 + k);
    MLSK_CUDA(cudaEventRecord(P.start, a.stream));
    // Cross-round overlap (matrix path): the generator stream reads only the
    // model and its own scratch (replication lists, merged-column lists, panel
    // buffers guarded by the GEMMs' events), so when the last round on this
    // pipeline ran the same model -- which waited for the caller's stream
    // after the model was built -- it need not wait for the caller's stream
    // again: the pre-pass and first generators of this round then run under the
    // last round's GEMM tail (config 2: 0.7 ms of a 19.7 ms round, config 3:
    // 0.7 of 14.5).  The GEMM stream (level accumulators) always waits.
    // MLSK_ROUND_OVERLAP=0 restores the full dependency.
    const char* ov_env = getenv("MLSK_ROUND_OVERLAP");
    const bool overlap_rounds = !M.vector && P.ran && P.last_serial == M.serial && !(ov_env && ov_env[0] == '0');
    if (!overlap_rounds) MLSK_CUDA(cudaStreamWaitEvent(P.s_gen, P.start, 0));
    MLSK_CUDA(cudaStreamWaitEvent(P.s_mm, P.start, 0));
    P.last_serial = M.vector ? 0 : M.serial;
    P.stage_ks(runs, all, P.s_gen);
    if (M.vector && !any_probe) {
        // config-1 shape: every level of the round in one launch (+ one reduction
        // launch), in slices of at most 4M replications / INNER_MAX_PARTS parts
        const int64_t max_slice = int64_t(1) << 22;
        InnerParts parts{};
        int64_t filled = 0;
        auto flush = [&]() {
            if (parts.n == 0) return;
            ws.v.ensure((size_t)filled);
            // many more CTAs than fit at once: the block scheduler then balances
            // the tasks dynamically (a one-wave grid-stride grid was 5% slower)
            const int64_t grid = std::min<int64_t>((parts.tasks * 32 + 255) / 256, (int64_t)sms * 16);
            {
                Prof p("fused_inner_f64", P.s_gen);
                if (nl)
                    k_fused_inner_multi<true><<<(int)std::max<int64_t>(grid, 1), 256, 0, P.s_gen>>>(
                        M.dm, a.seed, P.ks.p, parts, ws.v.p, a.target, a.target_param);
                else
                    k_fused_inner_multi<false><<<(int)std::max<int64_t>(grid, 1), 256, 0, P.s_gen>>>(
                        M.dm, a.seed, P.ks.p, parts, ws.v.p, a.target, a.target_param);
            }
            {
                Prof p("reduce_inner", P.s_gen);
                P.ensure_inner_red();
                k_reduce_inner_multi<<<dim3(INNER_RB, parts.n), 256, 0, P.s_gen>>>(ws.v.p, parts, P.red_part.p,
                                                                                   P.red_done.p);
            }
            launched(2);
            parts = InnerParts{};
            filled = 0;
        };
        // longest replications (largest c) first: the grid-stride loop hands out
        // replications in list order, so the deep levels' long chains start at
        // once instead of forming the kernel's tail
        std::vector<size_t> order(jobs.size());
        for (size_t j = 0; j < jobs.size(); ++j) order[j] = j;
        std::stable_sort(order.begin(), order.end(),
                         [&](size_t x, size_t y) { return jobs[x].lv.c > jobs[y].lv.c; });
        for (size_t j : order) {
            FusedJob& job = jobs[j];
            const int64_t c = job.lv.c, cc = job.lv.cc;
            const double w_fine = n / (double)c * kRescalePerturb;
            const double w_coarse = cc > 0 && !nl ? w_fine - n / (double)cc : w_fine;
            const int64_t total = job_cnt[j];
            for (int64_t off = 0; off < total;) {
                if (parts.n == INNER_MAX_PARTS || filled == max_slice) flush();
                const int64_t take = std::min(total - off, max_slice - filled);
                const int g = inner_group(c);
                // contiguous replications (one run covers the part): k = k0 + b
                int64_t k0 = -1;
                const int64_t pos = job_off[j] + off;
                // the run holding pos (runs are sorted by dst; one per owned chunk when sharded)
                auto rit = std::upper_bound(runs.begin(), runs.end(), pos,
                                            [](int64_t v, const KsRun& r) { return v < r.dst; });
                if (rit != runs.begin()) {
                    const KsRun& r = *(rit - 1);
                    if (r.dst <= pos && pos + take <= r.dst + r.count) k0 = r.k0 + (pos - r.dst);
                }
                parts.p[parts.n++] = InnerPart{job.lv.tag, c,
                                               cc,         w_fine,
                                               w_coarse,   job_off[j] + off,
                                               filled,     take,
                                               parts.tasks, k0,
                                               derive_prefix(a.seed, job.lv.tag), g,
                                               job.st->total(), job.st->total_sq()};
                parts.tasks += (take * g + 31) / 32;
                filled += take;
                off += take;
            }
            job.st->count += total;
        }
        flush();
        MLSK_CUDA(cudaEventRecord(P.end, P.s_gen));
        MLSK_CUDA(cudaStreamWaitEvent(a.stream, P.end, 0));
        return;
    }
    if (M.vector) {
        // config-1 shape with the coupling probe: one warp per replication, per level
        for (size_t j = 0; j < jobs.size(); ++j) {
            FusedJob& job = jobs[j];
            const int64_t c = job.lv.c, cc = job.lv.cc;
            const double w_fine = n / (double)c * kRescalePerturb;
            const double w_coarse = cc > 0 && !nl ? w_fine - n / (double)cc : w_fine;
            const int64_t total = job_cnt[j];
            const int64_t max_batch = 1 << 20;
            for (int64_t off = 0; off < total; off += max_batch) {
                const int nb = (int)std::min<int64_t>(max_batch, total - off);
                ws.v.ensure(nb);
                uint32_t* idx = nullptr;
                if (job.probe_host) {
                    ws.idx.ensure((size_t)nb * c);
                    idx = ws.idx.p;
                }
                const int grid = (int)std::min<int64_t>((nb + 7) / 8, (int64_t)sms * 8);
                {
                    Prof p("fused_inner_f64", P.s_gen);
                    k_fused_inner<<<grid, 256, 0, P.s_gen>>>(M.dm, a.seed, job.lv.tag, P.ks.p + job_off[j] + off, nb,
                                                             c, cc, w_fine, w_coarse, ws.v.p, idx, a.target,
                                                             a.target_param);
                }
                {
                    Prof p("reduce_inner", P.s_gen);
                    k_reduce_inner<<<1, 256, 0, P.s_gen>>>(ws.v.p, nb, job.st->total(), job.st->total_sq());
                }
                launched(2);
                if (idx) {
                    MLSK_CUDA(cudaStreamSynchronize(P.s_gen));
                    for (int b = 0; b < nb; ++b)
                        if (jks[j][off + b] < a.probe_k)
                            MLSK_CUDA(cudaMemcpy(job.probe_host + jks[j][off + b] * c, idx + (int64_t)b * c,
                                                 sizeof(uint32_t) * c, cudaMemcpyDeviceToHost));
                }
            }
            job.st->count += total;
        }
        MLSK_CUDA(cudaEventRecord(P.end, P.s_gen));
        MLSK_CUDA(cudaStreamWaitEvent(a.stream, P.end, 0));
        return;
    }


    // ---- matrix path: batches of replications, software-pipelined over a
    // panel engine (fp64 DMMA or the tcgen05 3xTF32 engine for fp32 models)
    // geometry-only object, rebuilt per round (the workspace may be shared by models)
    std::unique_ptr<PanelEngine> engine =
        tc_supported(M, a.target) ? make_tc_engine(M, ws) : make_f64_engine(M, ws, a.target, a.target_param);
    PanelEngine& E = *engine;
    const int64_t Gs = E.group_size();
    int64_t budget = int64_t(768) << 20;  // panel bytes per batch (x NBUF in flight; 384 MiB measured 1% slower)
    if (const char* e = getenv("MLSK_PANEL_BUDGET_MB")) budget = std::max<int64_t>(1, atoll(e)) << 20;
    // samples up to split_limit take one batch of their own (a K-split costs the
    // partial-Y traffic and shorter launches); larger ones run as K-segments
    int64_t split_limit = int64_t(8) << 30;
    if (const char* e = getenv("MLSK_SPLIT_MB"))  // tests: force K-split samples at small shapes
        split_limit = std::max<int64_t>(1, atoll(e)) << 20;

    // ---- passes.  The merged-column lists of a round (16 bytes per sampled
    // index) must fit their budget (1 GiB; MLSK_MERGE_LIST_MB): a round with more
    // (the adaptive driver's large rounds: millions of samples per level) runs
    // as several passes over slices of every level's samples, each with its own
    // pre-pass and synchronisation.
    const int64_t KCOLS = E.chunk_cols();
    auto merge_stride = [&](int64_t c) { return (c + KCOLS - 1) / KCOLS * KCOLS + KCOLS; };
    auto merge_mode_of = [&](size_t j) {
        const int64_t c = jobs[j].lv.c, cc = jobs[j].lv.cc;
        if (nl || !merge_enabled() || jobs[j].probe_host || jobs[j].lv.full || c < 4 * KCOLS ||
            M.desc.n > (int64_t(1) << 31) - 2)
            return 0;
        const double w_fine = n / (double)c * kRescalePerturb;
        const double w_coarse = cc > 0 ? w_fine - n / (double)cc : w_fine;
        const int mode = E.merge_mode(c, cc, w_fine, w_coarse);
        if (!mode || !merge_pays(c, cc, M.desc.n, KCOLS, w_coarse == -w_fine, mode == 2 ? 2 : 1)) return 0;
        return mode;
    };
    int64_t list_mb = 1024;
    if (const char* e = getenv("MLSK_MERGE_LIST_MB")) list_mb = std::max<int64_t>(1, atoll(e));  // tests
    const size_t list_budget = (size_t)(list_mb << 20) / sizeof(MkEntry);
    int64_t npass = 1;
    {
        double entries = 0;
        for (size_t j = 0; j < jobs.size(); ++j)
            if (job_cnt[j] > 0 && merge_mode_of(j)) entries += (double)job_cnt[j] * (double)merge_stride(jobs[j].lv.c);
        npass = std::max<int64_t>(1, (int64_t)std::ceil(entries / (0.95 * (double)list_budget)));
    }
    std::vector<int64_t> plo(jobs.size(), 0), pcnt(jobs.size(), 0);
    for (int64_t pass = 0; pass < npass; ++pass) {
        for (size_t j = 0; j < jobs.size(); ++j) {
            // slice boundaries on multiples of the engine's sample group
            auto cut = [&](int64_t q) {
                if (q >= npass) return job_cnt[j];
                const int64_t v = (int64_t)((double)job_cnt[j] * (double)q / (double)npass);
                return std::min(job_cnt[j], v / Gs * Gs);
            };
            plo[j] = cut(pass);
            pcnt[j] = cut(pass + 1) - plo[j];
        }
        // ---- merged sampled columns: the pre-pass of every level that qualifies
        // (deepest first, within the pass's budget of list memory), then ONE host
        // synchronisation for the merged chunk counts that size the launches
        std::vector<int> mj_of(jobs.size(), -1);
        std::vector<MergeJob> mjs;
        if (!nl && merge_enabled()) {
            std::vector<size_t> order(jobs.size());
            for (size_t j = 0; j < jobs.size(); ++j) order[j] = j;
            std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) { return jobs[x].lv.c > jobs[y].lv.c; });
            size_t list_used = 0, info_used = 0;
            for (size_t j : order) {
                if (pcnt[j] == 0 || (int)mjs.size() == MK_MAX_JOBS) continue;
                const int mode = merge_mode_of(j);
                if (!mode) continue;
                const int64_t stride = merge_stride(jobs[j].lv.c);
                const size_t need = (size_t)pcnt[j] * (size_t)stride;
                if (list_used + need > list_budget) continue;
                mj_of[j] = (int)mjs.size();
                mjs.push_back({mode, stride, list_used, info_used, 0});
                list_used += need;
                info_used += (size_t)pcnt[j];
            }
            if (!mjs.empty()) {
                // (the lists are read by the generators only, in order on this stream;
                // the per-sample info also by the GEMMs: double-buffered by round)
                P.mk_parity ^= 1;
                if (P.mk_info_used[P.mk_parity])
                    MLSK_CUDA(cudaStreamWaitEvent(P.s_gen, P.mk_info_done[P.mk_parity], 0));
                P.mk_list.ensure(list_used);
                P.mk_info[P.mk_parity].ensure(info_used);
                P.mk_max.ensure(MK_MAX_JOBS);
                MLSK_CUDA(cudaMemsetAsync(P.mk_max.p, 0, MK_MAX_JOBS * sizeof(int32_t), P.s_gen));
                // count scratch: groups of samples within 256 MiB
                int64_t cnt_mb = 256;
                if (const char* e = getenv("MLSK_MERGE_GROUP_MB")) cnt_mb = std::max<int64_t>(1, atoll(e));  // tests
                const int64_t mk_tiles = (M.desc.n + MK_TILE - 1) / MK_TILE;
                // (a launch's grid.y: at most 65535 samples per group)
                const int64_t grp_cap = std::min<int64_t>(65535, std::max<int64_t>(1, (cnt_mb << 20) / (8 * M.desc.n)));
                int64_t max_grp = 0;
                for (size_t j = 0; j < jobs.size(); ++j)
                    if (mj_of[j] >= 0) max_grp = std::max(max_grp, std::min(grp_cap, pcnt[j]));
                const size_t cnt_need = (size_t)max_grp * (size_t)M.desc.n;
                if (cnt_need > P.mk_cnt.n) {
                    P.mk_cnt.ensure(cnt_need);
                    P.mk_cnt.zero(P.s_gen);
                }
                P.mk_tile.ensure((size_t)max_grp * (size_t)mk_tiles);
                Prof p("merge_columns", P.s_gen);
                for (size_t j = 0; j < jobs.size(); ++j) {
                    if (mj_of[j] < 0) continue;
                    const MergeJob& mj = mjs[mj_of[j]];
                    const int64_t c = jobs[j].lv.c, cc = jobs[j].lv.cc;
                    const double w_fine = n / (double)c * kRescalePerturb;
                    const double w_coarse = cc > 0 ? w_fine - n / (double)cc : w_fine;
                    for (int64_t off = 0; off < pcnt[j]; off += grp_cap) {
                        const int64_t g = std::min(grp_cap, pcnt[j] - off);
                        const int64_t work = g * ((c + 1) / 2);
                        k_mk_count<<<(int)std::min<int64_t>((work + 255) / 256, (int64_t)sms * 16), 256, 0, P.s_gen>>>(
                            M.dm, a.seed, jobs[j].lv.tag, P.ks.p + job_off[j] + plo[j] + off, g, c, cc, P.mk_cnt.p);
                        MkEntry* list = P.mk_list.p + mj.list_off + (size_t)off * mj.stride;
                        MkInfo* info = P.mk_info[P.mk_parity].p + mj.info_off + off;
                        const dim3 tg((unsigned)mk_tiles, (unsigned)g);
                        k_mk_tiles<<<tg, MK_T, 0, P.s_gen>>>(P.mk_cnt.p, M.desc.n, mj.mode, w_fine, w_coarse, P.mk_tile.p);
                        k_mk_scan<<<(int)g, MK_T, 0, P.s_gen>>>(P.mk_tile.p, (int)mk_tiles, (int)KCOLS, list, mj.stride,
                                                               info, P.mk_max.p + mj_of[j]);
                        k_mk_write<<<tg, MK_T, 0, P.s_gen>>>(P.mk_cnt.p, M.desc.n, mj.mode, w_fine, w_coarse, (int)KCOLS,
                                                             P.mk_tile.p, info, list, mj.stride);
                        launched(4);
                    }
                }
                MLSK_CUDA(cudaMemcpyAsync(P.mk_max_host, P.mk_max.p, mjs.size() * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                          P.s_gen));
                MLSK_CUDA(cudaEventRecord(P.mk_done, P.s_gen));
                MLSK_CUDA(cudaEventSynchronize(P.mk_done));
                for (size_t q = 0; q < mjs.size(); ++q) mjs[q].nk = std::max<int64_t>(1, P.mk_max_host[q]);
            }
        }
        auto job_chunks = [&](size_t j) {
            return mj_of[j] >= 0 ? mjs[mj_of[j]].nk : E.nchunks(jobs[j].lv.c, jobs[j].lv.cc);
        };
        auto with_merge = [&](KRange kr, size_t j, int64_t off) {
            if (mj_of[j] >= 0) {
                const MergeJob& mj = mjs[mj_of[j]];
                if (kr.nkc < 0) kr.nkc = mj.nk;
                kr.mk = P.mk_list.p + mj.list_off + (size_t)off * mj.stride;
                kr.mk_stride = mj.stride;
                kr.mk_info = P.mk_info[P.mk_parity].p + mj.info_off + off;
            }
            return kr;
        };

        // panel bytes a batch of nb samples needs in its buffer.  Merged chunk
        // counts vary a little from round to round (they follow the draws), and a
        // buffer that grew with every new maximum would be reallocated for many
        // rounds: merged batches reserve 3% + 64 MiB of headroom, capped at the
        // unmerged size.
        auto reserve_bytes = [&](size_t j, int64_t nb, int64_t chunks) {
            const int64_t need = nb * chunks * E.chunk_bytes();
            if (mj_of[j] < 0) return need;
            const int64_t ub = nb * E.nchunks(jobs[j].lv.c, jobs[j].lv.cc) * E.chunk_bytes();
            const int64_t q = int64_t(64) << 20;
            return std::min(ub, (need + need / 32 + q - 1) / q * q);
        };
        // Level order (each level has its own accumulators, so the order changes no
        // result): the pipeline's tail is the last batch's GEMM with no generator
        // left to overlap, its head the first batch's generator alone.  When one
        // sample's panels exceed a batch (configs 4 / 5: long single-sample GEMMs at
        // the deep levels) the levels run deepest first, so that those GEMMs run
        // over the other levels' generators instead of ending the round alone
        // (config 4: 13.2 -> 12.75 ms per step, config 5: 345 -> 341); with many
        // samples per batch at every level (configs 2 / 3) the order is neutral to
        // slightly worse (19.73 -> 19.90 ms) and stays ascending.
        // MLSK_LEVEL_ORDER=asc|desc overrides.
        std::vector<size_t> level_order(jobs.size());
        for (size_t j = 0; j < jobs.size(); ++j) level_order[j] = j;
        {
            bool desc = false;
            for (size_t j = 0; j < jobs.size(); ++j)
                if (pcnt[j] > 0 && job_chunks(j) * E.chunk_bytes() > budget) desc = true;
            if (const char* e = getenv("MLSK_LEVEL_ORDER")) desc = e[0] == 'd';
            if (desc)
                std::stable_sort(level_order.begin(), level_order.end(),
                                 [&](size_t x, size_t y) { return jobs[x].lv.c > jobs[y].lv.c; });
        }
        std::vector<Batch> batches;
        int64_t max_panel = 0;
        for (size_t j : level_order) {
            const int64_t per = job_chunks(j) * E.chunk_bytes();
            const int64_t total = pcnt[j];  // this pass's samples of the level: [plo, plo + total)
            if (per > split_limit && E.splits_k()) {
                if (nl)
                    throw Error(MLSK_EINVAL, "fused engine: nonlinear targets need a level-sample's panels within one "
                                             "batch (" + std::to_string(split_limit >> 20) + " MiB)");
                // one sample's panels exceed a batch: K-segments of one sample each,
                // the partial Y carried between them
                if (jobs[j].probe_host)
                    throw Error(MLSK_EINVAL, "probe: not available for level-samples split along K (panels > " + std::to_string(split_limit >> 20) + " MiB)");
                const int64_t nk = job_chunks(j);
                const int64_t seg = std::max<int64_t>(1, split_limit / E.chunk_bytes());  // few, large segments
                for (int64_t off = 0; off < total; ++off)
                    for (int64_t k0 = 0; k0 < nk; k0 += seg) {
                        KRange kr;
                        kr.kc0 = k0;
                        kr.nkc = std::min(seg, nk - k0);
                        kr.part = nk <= seg ? 0 : (k0 == 0 ? 1 : (k0 + kr.nkc == nk ? 3 : 2));
                        batches.push_back({j, plo[j] + off, 1, job_off[j] + plo[j] + off, with_merge(kr, j, off)});
                        max_panel = std::max(max_panel, reserve_bytes(j, 1, kr.nkc));
                    }
                continue;
            }
            int64_t max_nb = std::max<int64_t>(1, budget / per);
            // every CTA group needs a sample: stretch the batch (up to 4x the budget)
            // rather than leave groups idle (config 3's deepest level: 268 MB samples)
            if (max_nb < Gs && Gs * per <= 4 * budget) max_nb = Gs;
            if (max_nb > Gs) max_nb = max_nb / Gs * Gs;
            for (int64_t off = 0; off < total; off += max_nb) {
                const int nb = (int)std::min<int64_t>(max_nb, total - off);
                batches.push_back({j, plo[j] + off, nb, job_off[j] + plo[j] + off, with_merge(KRange{}, j, off)});
                max_panel = std::max(max_panel, reserve_bytes(j, nb, job_chunks(j)));
            }
        }
        if ((size_t)(max_panel + 7) / 8 > P.panels[0].n) {
            // the buffers must grow: one level-sample's panels must fit a buffer;
            // fail with a clear message instead of an opaque allocation error
            // (queried only when growing: cudaMemGetInfo on every round stalled
            // the launching thread for milliseconds now and then)
            size_t free_b = 0, total_b = 0;
            MLSK_CUDA(cudaMemGetInfo(&free_b, &total_b));
            size_t held = 0;
            for (int i = 0; i < NBUF; ++i) held += P.panels[i].n * sizeof(double);
            if ((double)NBUF * (double)max_panel > (double)(free_b + held))
                throw Error(MLSK_ERUNTIME, "fused engine: the sampled panels of one batch (" +
                                               std::to_string(max_panel >> 20) + " MiB x " + std::to_string(NBUF) +
                                               " buffers) exceed free device memory; use a smaller c_l or m, p");
        }
        for (int i = 0; i < NBUF; ++i) P.panels[i].ensure((size_t)(max_panel + 7) / 8);
        {
            // KRange::finish: only a level's last batch of the pass
            std::vector<char> seen(jobs.size(), 0);
            for (size_t q = batches.size(); q-- > 0;) {
                batches[q].kr.finish = !seen[batches[q].job];
                seen[batches[q].job] = 1;
            }
        }

        for (size_t bi = 0; bi < batches.size(); ++bi, ++P.batch_seq) {
            const size_t i = (size_t)P.batch_seq;  // buffers rotate across passes and rounds
            const Batch& bt = batches[bi];
            FusedJob& job = jobs[bt.job];
            const int64_t c = job.lv.c, cc = job.lv.cc;
            const double w_fine = n / (double)c * kRescalePerturb;                                        // n/c
            const double w_coarse = cc > 0 && !nl ? w_fine - n / (double)cc : w_fine;  // n/c - n/cc on the prefix
            const int buf = (int)(i % NBUF);
            void* panels = P.panels[buf].p;
            uint32_t* idx = nullptr;
            if (job.probe_host) {
                P.idx[buf].ensure((size_t)bt.nb * c);
                idx = P.idx[buf].p;
            }
            // generator: wait until the GEMM that last used this buffer is done
            if (P.used[buf]) MLSK_CUDA(cudaStreamWaitEvent(P.s_gen, P.mm_done[buf], 0));
            if (serial_mode() && P.used[(i + NBUF - 1) % NBUF])
                MLSK_CUDA(cudaStreamWaitEvent(P.s_gen, P.mm_done[(i + NBUF - 1) % NBUF], 0));
            E.gen(P.s_gen, a.seed, job.lv.tag, P.ks.p + bt.ks_off, bt.nb, c, cc, w_fine, w_coarse, panels, idx, bt.kr);
            MLSK_CUDA(cudaEventRecord(P.gen_done[buf], P.s_gen));
            // GEMM + fused level epilogue + fixed-order reduction
            MLSK_CUDA(cudaStreamWaitEvent(P.s_mm, P.gen_done[buf], 0));
            E.gemm(P.s_mm, panels, bt.nb, c, cc, w_fine, w_coarse, *job.st, bt.kr);
            {
                const int64_t full = E.nchunks(c, cc);
                const int64_t k = bt.kr.nkc >= 0 ? bt.kr.nkc : full;
                g_columns[0] += (int64_t)bt.nb * k * E.chunk_cols();
                // (a K-split sample's segments add up to its merged chunks; its c indices count once)
                g_columns[1] += bt.kr.part == 0 || bt.kr.part == 1 ? (int64_t)bt.nb * c : 0;
            }
            MLSK_CUDA(cudaEventRecord(P.mm_done[buf], P.s_mm));
            P.used[buf] = true;
            if (idx) {
                MLSK_CUDA(cudaStreamSynchronize(P.s_gen));
                for (int b = 0; b < bt.nb; ++b) {
                    const int64_t k = jks[bt.job][bt.off + b];
                    if (k < a.probe_k)
                        MLSK_CUDA(cudaMemcpy(job.probe_host + k * c, idx + (int64_t)b * c, sizeof(uint32_t) * c,
                                             cudaMemcpyDeviceToHost));
                }
            }
        }
        if (!mjs.empty()) {
            MLSK_CUDA(cudaEventRecord(P.mk_info_done[P.mk_parity], P.s_mm));
            P.mk_info_used[P.mk_parity] = true;
        }
    }  // passes
    for (auto& job : jobs) {
        int64_t cnt = 0;
        for (const auto& sg : job.segs) cnt += sg.count;
        job.st->count += cnt;
    }
    MLSK_CUDA(cudaEventRecord(P.end, P.s_mm));
    P.ran = true;
    MLSK_CUDA(cudaStreamWaitEvent(a.stream, P.end, 0));
}


double measure_index_rate(int device) {
    if (device >= 0) MLSK_CUDA(cudaSetDevice(device));
    mlsk_model_desc d{};
    d.kind = MLSK_MODEL_GAUSS_MEAN;
    d.dtype = MLSK_F64;
    d.stream_mode = MLSK_STREAM_PHILOX;
    d.n = 4096;  // config 1
    d.sd = 1.0;
    d.mean_lo = 0.0;
    d.mean_hi = 1.0;
    d.data_seed = 1;
    Model M;
    build_model(M, &d, 0);
    DevArray<double> sink(1);
    const int grid = sm_count() * 8;
    const int64_t pairs = 256;
    k_index_rate<<<grid, 256>>>(M.dm, 7, 4, sink.p);
    launched();
    MLSK_CUDA(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_index_rate<<<grid, 256>>>(M.dm, 7 + r, pairs, sink.p);
        cudaEventRecord(e1);
        launched();
        MLSK_CUDA(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return (double)grid * 256 * pairs * 2 / (best * 1e-3);
}

}  // namespace mlsk
