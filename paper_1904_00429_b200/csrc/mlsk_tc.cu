// mlsk_tc.cu -- the fp32 configurations (BASELINE configs 3-5) on the 5th-gen
// tensor cores: 3xTF32 sampled GEMM with tcgen05.mma, TMEM accumulators and the
// level epilogue (Y^2, running sum) fused into dedicated epilogue warps.
//
// Same fused formulation as the fp64 engine (mlsk_fused.cu): per level-sample
// Y = sum_t w_t a_t b_t^T with signed weights, K = c.  fp32 accuracy from TF32
// tensor cores by the 3xTF32 split  a b ~= a_hi b_hi + a_hi b_lo + a_lo b_hi,
// a_hi = a (the MMA reads the fp32 word and uses its TF32 part), a_lo = a -
// tf32(a) (exact in fp32) -- three MMAs per K-step into one fp32 accumulator.
//
// The two cross terms run as BF16 MMAs (kind::f16, K = 16) over BF16
// copies of the values and of their lo parts -- see "BF16 cross terms" below:
// 2 TF32 + 2 BF16 MMAs per 16-column K-chunk instead of 6 TF32 ones, the same
// fp32-level accuracy (the cross terms are 2^-11 of the product).
//
//  k_gen_panels_tf32  sampled indices + the sampled columns of A / rows of B
//                     (gauss f32, Student-t or random-Fourier features,
//                     generated on the fly), written as hi / lo K-chunks in the
//                     UMMA canonical K-major SWIZZLE_64B layout (16 tf32 = 64 B
//                     per row of a K-chunk).
//  k_gemm_tf32x3      one 128 x 256 output tile per CTA over a strided set of
//                     samples (tile groups: Gs CTAs per tile when the grid is
//                     smaller than the SM count), 20 warps in two register
//                     classes (setmaxnreg): warpgroup 0 = warp 0 the
//                     cp.async.bulk producer (4-stage mbarrier ring, 48 KB per
//                     stage: A_hi, A_lo, B_hi, B_lo of one K-chunk), warp 1
//                     TMEM allocation + single-thread tcgen05.mma (M128 N256 K8,
//                     3 MMAs per K-step) into two 256-column TMEM accumulators
//                     (all 512 columns, double-buffered across samples and
//                     accumulation segments), warps 2-3 idle; warps 4-19 the
//                     epilogue, four per TMEM lane quadrant taking 64 columns
//                     each (tcgen05.ld.32x32b.x16, ||Y||^2 in fp64, the running
//                     sum in 64 fp32 registers per thread, flushed every 32
//                     samples by red.global.add into an fp64 CTA partial, or
//                     -- samples longer than TC_SEG K-chunks -- each sample's Y,
//                     summed over its segments in registers with round-to-
//                     nearest, by red.add.f32 into an fp32 partial).  Tiles are
//                     rasterised in groups of 16 tile rows.  N = 256 cuts the
//                     operand bytes per flop that cross L2 -> SMEM by a quarter
//                     vs 128 x 128 tiles.  When the tile rows pair up (every
//                     BASELINE config) the CTAs run as clusters of two on tiles
//                     (tm, tn), (tm + 1, tn): the leader issues
//                     tcgen05.mma.cta_group::2 (M = 256) over both CTAs' shared
//                     memory, each CTA staging its A rows and half of the B
//                     columns (32 KB stages, seven of them) -- a third less
//                     shared-memory traffic per SM, 3-9% faster per level.
//  k_reduce_tiles_tc  level total += the group partials (fixed order);
//  k_kpar_combine     one-sample levels split over two CTA groups along K;
//  k_mirror_lower     symmetric (RFF Gram) outputs: lower blocks mirrored.

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "mlsk_internal.h"

namespace mlsk {

namespace {

#ifndef MLSK_PANEL_HINT
#define MLSK_PANEL_HINT 1  // measured: config 5 -2.6%, config 3 neutral; 2 (loads too): +7% / +10% slower
#endif
constexpr int TBM = 128, TBN = 256, TBK = 16;       // TBK tf32 = 64 bytes per row (SWIZZLE_64B)
constexpr int ROWB = TBK * 4;                       // bytes per K-chunk row
#ifndef MLSK_TC_STAGES
#define MLSK_TC_STAGES 4
#endif
constexpr int TSTAGES = MLSK_TC_STAGES;             // 4 x 48 KB (3 stages: 6% slower GEMM, no gain from a co-resident generator CTA)
constexpr int TTILE = TBM * TBK * 4;                // 8 KB: one 128-row K-chunk (A tile, half a B tile)
constexpr int TA_BYTES = TTILE, TB_BYTES = 2 * TTILE;
constexpr int TSTAGE_BYTES = 2 * TA_BYTES + 2 * TB_BYTES;  // A_hi, A_lo, B_hi, B_lo: 48 KB
constexpr int EPI_WARPS = 16;                       // four per TMEM lane quadrant (64-column quarters)
// CTA pair (cta_group::2, M = 256 over two SMs of a TPC): each CTA stages its
// own 128 A rows and HALF of the 256 B columns, 32 KB per stage, six stages
#ifndef MLSK_TC_PSTAGES
#define MLSK_TC_PSTAGES 7  // 224 KB: measured 1.5% faster than 6 at config 3, configs 4 / 5 unchanged
#endif
constexpr int PSTAGES = MLSK_TC_PSTAGES;
constexpr int PB_BYTES = TTILE;                             // half a B tile (128 columns)
constexpr int PSTAGE_BYTES = 2 * TA_BYTES + 2 * PB_BYTES;  // 32 KB
static_assert(PSTAGES * PSTAGE_BYTES + 1024 <= 226 * 1024, "pair ring exceeds the shared memory of a CTA");
// warpgroup 0: producer (warp 0), TMEM allocation + MMA issue (warp 1), two
// idle warps; warpgroups 1-4: epilogue.  setmaxnreg moves registers from the
// control warpgroup to the epilogue (32 / 112 per thread) for its 64-entry
// running sum / sample Y plus a 16-column TMEM load.  The budget is the
// launch's own allocation (640 threads x 96 = 61440; a launch of 18 warps
// or more is capped at 96 registers: five warps share one SMSP's 16 K):
// 4 x 32 x 32 + 16 x 32 x 112 = 61440 <= 61440, so setmaxnreg.inc cannot
// wait forever for registers no warp will release.
constexpr int CTRL_WARPS = 4;
constexpr int TC_THREADS = 32 * (CTRL_WARPS + EPI_WARPS);
constexpr int CTRL_REGS = 32, EPI_REGS = 112;
static_assert(32 * (CTRL_WARPS * CTRL_REGS + EPI_WARPS * EPI_REGS) <= TC_THREADS * 96,
              "setmaxnreg budget exceeds the launch allocation: the epilogue's inc would block forever");
#ifndef MLSK_TC_FLUSH
#define MLSK_TC_FLUSH 32
#endif
constexpr int FLUSH = MLSK_TC_FLUSH;                // samples per fp32 running-sum flush
constexpr uint32_t TMEM_COLS = 2 * TBN;             // two accumulators: all 512 columns
constexpr int TC_SEG = 32;                          // K-chunks (K = 512) per TMEM accumulation segment
constexpr int GEN_T = 256;

// ----------------------------------------------------------------- PTX

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
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
__device__ __forceinline__ void bar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
#if MLSK_PANEL_HINT >= 2
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
#else
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
#endif
}
// panel tile out of shared memory by the TMA engine; MLSK_PANEL_HINT >= 1: with
// an L2 evict_first policy (panels stream through L2 once; the model's means
// and the CTA partials are what should stay)
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
#if MLSK_PANEL_HINT >= 1
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"((uint32_t)__cvta_generic_to_shared(src)), "r"(bytes), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"((uint32_t)__cvta_generic_to_shared(src)), "r"(bytes)
                 : "memory");
#endif
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// CTA pair: the MMA completion arrives on the barrier at the same offset in both CTAs
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
        "h"((uint16_t)3)
        : "memory");
}
// this CTA's shared address `a` as seen in cluster CTA `rank`
__device__ __forceinline__ uint32_t cluster_addr(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
// (relaxed: a release arrive compiles to MEMBAR.ALL.GPU -- microseconds per
// stage on the relay's critical path; the data it reports is already complete:
// the stage's bulk copies have landed (observed on this CTA's barrier), the
// TMEM reads have returned (tcgen05.wait::ld))
__device__ __forceinline__ void bar_arrive_remote(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void bar_wait_cluster(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tc_mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// BF16 cross terms (TcShape::bfx): kind::f16 MMAs with BF16 operands, K = 16
__device__ __forceinline__ void tc_mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tc_mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// 32 lanes x 16 consecutive 32-bit columns: lane i of the warp gets row
// (quadrant*32 + i), columns [col, col + 16)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// fire-and-forget fp32 add in L2 (no load round trip in the epilogue); the
// reductions of one thread to one address apply in program order, so the
// partial's bits do not depend on timing
__device__ __forceinline__ void red_add_f32(float* p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add_f64(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_64B (ROWB = 64) or
// SWIZZLE_128B (ROWB = 128): 8-row groups 8 * ROWB bytes apart (SBO), version
// 1 (sm_100), layout type 4 / 2.
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;                  // LBO (unused for swizzled K-major)
    d |= (uint64_t)((8 * ROWB) >> 4) << 32;  // SBO
    d |= (uint64_t)1 << 46;                  // descriptor version (sm_100)
    d |= (uint64_t)(ROWB == 128 ? 2 : 4) << 61;
    return d;
}

// kind::tf32 instruction descriptor: F32 accumulate, TF32 A / B, K-major, M x N
__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// byte offset of element (r, k) in a 128-row x TBK-tf32 swizzled K-major tile:
// the 16-byte chunk index XOR address bits [7, 7 + log2(ROWB / 16))
__device__ __forceinline__ int sw_off(int r, int k) {
    return r * ROWB + ((((k >> 2) ^ ((r * ROWB >> 7) & (ROWB / 16 - 1))) << 4) | ((k & 3) << 2));
}

// ---- BF16 cross terms (bfx).  a b ~= tf32(a) tf32(b) + a b_lo + a_lo b: the
// two cross terms are 2^-11 of the product, so BF16 operands (8 bits, rounded
// to nearest) leave them accurate to 2^-9 of themselves, 2^-20 of the product
// (1.3e-6 relative on a level-sample's Y, emulated on the CPU; the TF32 form
// leaves 3.5e-7, and the accumulation's own error is 2-5e-6).  A BF16 MMA is
// K = 16 at twice the TF32 rate: a K-chunk costs 2 TF32 + 2 BF16 MMAs instead
// of 6 TF32 ones (a third less tensor time) and reads 32 KB instead of 48 KB of
// operands from shared memory.  The lo tile of a 128-row K-chunk (8 KB) then
// holds ONE BF16 tile in the same K-major SWIZZLE_64B layout (64-byte rows):
// row r = [bf16(x)(r, 0..15) | bf16(x - tf32(x))(r, 0..15)], i.e. the values are
// BF16 columns 0..15 and their lo parts columns 16..31 of a 32-column tile, and
// the two K = 16 operands are the row halves (descriptor start + 0 / + 32 bytes,
// as the TF32 K = 8 steps of the hi tile).  The hi tile is unchanged, so panels,
// stages and bulk copies keep their sizes.  (Two separate 32-byte-row tiles in
// SWIZZLE_32B were measured first: correct, but their MMAs ran ~1.6x slower than
// the 64-byte-row form.)  MLSK_TC_BF16X=0 keeps the three TF32 MMAs.
static_assert(TBK * 2 * 2 == ROWB, "values and lo parts as BF16 fill a 64-byte row");
// byte offset of BF16 element (r, k) of the values (which = 0) or the lo parts (1)
__device__ __forceinline__ int sw_off_b(int r, int k, int which) {
    const int kp = k + TBK * which;
    return r * ROWB + ((((kp >> 3) ^ ((r * ROWB >> 7) & (ROWB / 16 - 1))) << 4) | ((kp & 7) << 1));
}
// kind::f16 instruction descriptor: F32 accumulate, BF16 A / B, K-major, M x N
__host__ __device__ constexpr uint32_t bf16_idesc(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// two floats -> packed BF16 pair (round to nearest even), x0 in the low half
__device__ __forceinline__ uint32_t bf16x2_rn(float x0, float x1) {
    uint32_t d;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(x1), "f"(x0));
    return d;
}
// two floats -> packed FP16 pair (round to nearest even, saturating), x0 in the low half
__device__ __forceinline__ uint32_t f16x2_rn(float x0, float x1) {
    uint32_t d;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(x1), "f"(x0));
    return d;
}

// ---- FP16 pairs (TcShape::bfx == 2, models whose entries are bounded: fp32
// Gaussian draws -- the 24-bit Box-Muller radius is at most 5.77 -- and random
// Fourier features).  An entry is stored as TWO halves, hi = fp16(x) (11 bits,
// round to nearest) and lo = fp16(x - hi): 4 bytes per entry instead of 8, in
// ONE K-major SWIZZLE_64B tile per 128 rows of a K-chunk whose 64-byte rows are
// hi(r, 0..15) | lo(r, 0..15), and a K-chunk is three FP16 MMAs (K = 16): hi x
// hi, hi x lo, lo x hi over the row halves.  Half the panel bytes for the
// generators to write and the GEMM to read, three MMAs instead of four.
// (Mixed FP16 x BF16 operands in one MMA are an illegal instruction, so
// unbounded models -- Student-t: fp16 would saturate in the tails -- keep the
// TF32 + BF16 form.)  Entries below 2^-14 keep an absolute accuracy of 2^-25 in
// each half; the models' panel scale (a power of two, undone exactly in the
// epilogue) keeps typical entries near 1.
__device__ __forceinline__ void f16x2_unpack(uint32_t h, float& x0, float& x1) {
    asm("{\n\t.reg .b16 l, u;\n\tmov.b32 {l, u}, %2;\n\tcvt.f32.f16 %0, l;\n\tcvt.f32.f16 %1, u;\n\t}"
        : "=f"(x0), "=f"(x1)
        : "r"(h));
}
// chunk columns k, k + 1 (k even) of row r into the (only) tile of FP16 pairs
__device__ __forceinline__ void store_h16_pair(unsigned char* t, int r, int k, float v0, float v1) {
    const uint32_t h = f16x2_rn(v0, v1);
    float h0, h1;
    f16x2_unpack(h, h0, h1);
    *reinterpret_cast<uint32_t*>(t + sw_off_b(r, k, 0)) = h;
    *reinterpret_cast<uint32_t*>(t + sw_off_b(r, k, 1)) = f16x2_rn(__fsub_rn(v0, h0), __fsub_rn(v1, h1));
}
// ---- FP16 hi + BF16 cross terms (TcShape::bfx == 3, unbounded fp32 models:
// Student-t).  hi = fp16(x) saturating, and the cross terms as in the BF16 form
// over bf16(x) and bf16(x - hi): whatever hi cannot hold -- the excess of a tail
// draw beyond 65504, the low bits of a tiny entry -- lands in the BF16 lo part,
// which has fp32's exponent range.  6 bytes per entry: the first tile's 64-byte
// rows are hi(r, 0..15) | bf16(x)(r, 0..15), a second tile of 32-byte rows
// (K-major SWIZZLE_32B, 4 KB per 128 rows) holds bf16(x - hi); a K-chunk is one
// FP16 MMA (hi x hi) + two BF16 MMAs (x b_lo: A from the first tile's second row
// half, B from the second tile; a_lo b the other way round).
constexpr int LROWB = TBK * 2;        // bytes per row of the BF16 lo tile
constexpr int LTILE = TBM * LROWB;    // 4 KB per 128 rows
__device__ __forceinline__ int sw32_off(int r, int k) {  // BF16 element (r, k), SWIZZLE_32B
    return r * LROWB + ((((k >> 3) ^ ((r * LROWB >> 7) & 1)) << 4) | ((k & 7) << 1));
}
__device__ __forceinline__ uint64_t sw32_desc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;                   // LBO (unused for swizzled K-major)
    d |= (uint64_t)((8 * LROWB) >> 4) << 32;  // SBO: 8-row groups
    d |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
    d |= (uint64_t)6 << 61;                   // SWIZZLE_32B
    return d;
}
// chunk columns k, k + 1 (k even) of row r: t1 = the hi | bf16(x) tile, t2 = the bf16 lo tile
__device__ __forceinline__ void store_h16b_pair(unsigned char* t1, unsigned char* t2, int r, int k, float v0, float v1) {
    const uint32_t h = f16x2_rn(v0, v1);
    float h0, h1;
    f16x2_unpack(h, h0, h1);
    *reinterpret_cast<uint32_t*>(t1 + sw_off_b(r, k, 0)) = h;
    *reinterpret_cast<uint32_t*>(t1 + sw_off_b(r, k, 1)) = bf16x2_rn(v0, v1);
    *reinterpret_cast<uint32_t*>(t2 + sw32_off(r, k)) = bf16x2_rn(__fsub_rn(v0, h0), __fsub_rn(v1, h1));
}
// kind::f16 instruction descriptor: F32 accumulate, FP16 A / B, K-major, M x N
__host__ __device__ constexpr uint32_t f16_idesc(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ---------------------------------------------------------------- entries

__device__ __forceinline__ float tf32_lo(float x) {
    return __fsub_rn(x, __uint_as_float(__float_as_uint(x) & 0xFFFFE000u));
}
// chunk columns k, k + 1 (k even) of row r into the lo tile: TF32 lo words, or
// (bfx) the BF16 pair of the values and of their lo parts
__device__ __forceinline__ void store_lo_pair(unsigned char* tlo, int r, int k, float v0, float v1, bool bfx) {
    if (bfx) {
        *reinterpret_cast<uint32_t*>(tlo + sw_off_b(r, k, 0)) = bf16x2_rn(v0, v1);
        *reinterpret_cast<uint32_t*>(tlo + sw_off_b(r, k, 1)) = bf16x2_rn(tf32_lo(v0), tf32_lo(v1));
    } else {
        *reinterpret_cast<float2*>(tlo + sw_off(r, k)) = make_float2(tf32_lo(v0), tf32_lo(v1));
    }
}

struct TcModel {
    DevModel M;
};

// Student-t(3) draw t of A[row][col] (which = 0) or B[col][row] (which = 1)
__device__ __forceinline__ float student_t_draw(uint64_t key, int64_t col, int64_t rq, int which, const Tables& T) {
    const u32x4 r = philox((uint32_t)col, (uint32_t)rq, (uint32_t)which, MLSK_CTR_T, key);
    float z[4];
    box_muller_f<true>(r.x, r.y, z[0], z[1], T);
    box_muller_f<true>(r.z, r.w, z[2], z[3], T);
    const float v = __fadd_rn(__fadd_rn(__fmul_rn(z[1], z[1]), __fmul_rn(z[2], z[2])), __fmul_rn(z[3], z[3]));
    return __fdiv_rn(z[0], __fsqrt_rn(__fdiv_rn(v, 3.0f)));
}
// the entry with its on-the-fly mean (one row at a time: the generic path)
__device__ __forceinline__ float student_t_entry(const TcModel& S, uint64_t key, int64_t col, int64_t rq, int which,
                                                 const Tables& T) {
    const float mean = st_mean(which == 0 ? S.M.st_key_a : S.M.st_key_b, col, rq, S.M.st_lo, S.M.st_w);
    return __fadd_rn(mean, student_t_draw(key, col, rq, which, T));
}

// RFF feature sqrt(2/n) cos(w_col . x_row + b_col) (fp32 dot, accurate cosf)
__device__ __forceinline__ float rff_entry(const DevModel& M, int64_t col, int64_t row) {
    float acc = 0.f;
    const float* x = M.rff_x + row * M.rff_dim;
    for (int64_t t = 0; t < M.rff_dim; ++t) acc = __fmaf_rn(x[t], M.rff_w[t * M.n + col], acc);
    return (float)M.rff_scale * cosf(acc + M.rff_b[col]);
}

// ------------------------------------------------------------ generator

// Gauss fp32 phase: 128 rows of A (IS_A) or 128 columns of B for the 16 chunk
// columns.  Thread = (row quad qq, column pair cp): one float4 mean load and
// one Philox block (4 normals) per column, 64-bit stores of the column pair
// per row (hi and lo tiles).  Padding columns carry j = 0 and B weight 0.
static_assert(GEN_T == 256 && TBK == 16 && TBM == 128, "gauss_phase_f32 thread map: 8 column pairs x 32 row quads");
template <bool IS_A>
__device__ __forceinline__ void gauss_phase_f32(const DevModel& M, const Tables& T, uint64_t key, int64_t rb,
                                                const int* s_j, const float* s_w, unsigned char* thi,
                                                unsigned char* tlo, int tid, int bfx) {
    const int cp = tid & 7, qq = tid >> 3;
    const int r0 = 4 * qq;
    const int64_t dim = IS_A ? M.m : M.p;
    const int64_t lim = dim - rb;
    const float* mbase = (IS_A ? M.mean_at_f : M.mean_b_f) + rb + r0;
    const uint32_t rowq = (uint32_t)((rb + r0) >> 2);
    const float sd = (float)M.sd;
    float v[2][4];
    if (r0 + 3 < lim && (dim & 3) == 0) {
        int jj[2];
        float4 mv[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            jj[u] = s_j[2 * cp + u];
            mv[u] = __ldg(reinterpret_cast<const float4*>(mbase + (uint64_t)(uint32_t)jj[u] * (uint32_t)dim));
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const u32x4 r = philox((uint32_t)jj[u], rowq, 0, IS_A ? MLSK_CTR_A : MLSK_CTR_B, key);
            float z[4];
            box_muller_f<true>(r.x, r.y, z[0], z[1], T);
            box_muller_f<true>(r.z, r.w, z[2], z[3], T);
            const float m4[4] = {mv[u].x, mv[u].y, mv[u].z, mv[u].w};
            const float w = IS_A ? 1.0f : s_w[2 * cp + u];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float x = __fadd_rn(m4[e], __fmul_rn(sd, z[e]));
                v[u][e] = IS_A ? x : __fmul_rn(w, x);
            }
        }
    } else {
        // ragged edge: rows past the matrix are zero
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int j = s_j[2 * cp + u];
#pragma unroll
            for (int e = 0; e < 4; ++e) v[u][e] = 0.f;
            if (r0 < lim) {
                const float* mp = mbase + (int64_t)j * dim;
                float mv[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) mv[e] = r0 + e < lim ? __ldg(mp + e) : 0.f;
                const u32x4 r = philox((uint32_t)j, rowq, 0, IS_A ? MLSK_CTR_A : MLSK_CTR_B, key);
                float z[4];
                box_muller_f<true>(r.x, r.y, z[0], z[1], T);
                box_muller_f<true>(r.z, r.w, z[2], z[3], T);
                const float w = IS_A ? 1.0f : s_w[2 * cp + u];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (r0 + e < lim) {
                        const float x = __fadd_rn(mv[e], __fmul_rn(sd, z[e]));
                        v[u][e] = IS_A ? x : __fmul_rn(w, x);
                    }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (bfx == 2) {  // FP16 pairs: one tile
            store_h16_pair(thi, r0 + e, 2 * cp, v[0][e], v[1][e]);
            continue;
        }
        if (bfx == 3) {  // FP16 hi | BF16 values, BF16 lo
            store_h16b_pair(thi, tlo, r0 + e, 2 * cp, v[0][e], v[1][e]);
            continue;
        }
        const int off = sw_off(r0 + e, 2 * cp);  // chunk columns 2cp, 2cp+1: adjacent words
        *reinterpret_cast<float2*>(thi + off) = make_float2(v[0][e], v[1][e]);
        store_lo_pair(tlo, r0 + e, 2 * cp, v[0][e], v[1][e], bfx != 0);
    }
}

// Student-t(3) phase (config 5): same thread map as the gauss phase (a row
// quad x a chunk-column pair per thread, 64-bit stores of the pair per row);
// per column one Philox block gives the on-the-fly means of the row quad and
// each entry one block its t draw (1.25 blocks per entry; a block per mean
// doubled the generator's integer work), independent chains in flight.
template <bool IS_A>
__device__ __forceinline__ void student_t_phase_f32(const TcModel& S, const Tables& T, uint64_t key, int64_t rb,
                                                    const int* s_j, const float* s_w, unsigned char* thi,
                                                    unsigned char* tlo, int tid, int bfx, float ascale) {
    const int cp = tid & 7, qq = tid >> 3;
    const int r0 = 4 * qq;
    const int64_t lim = (IS_A ? S.M.m : S.M.p) - rb;
    float v[2][4];
    const uint64_t mkey = IS_A ? S.M.st_key_a : S.M.st_key_b;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int j = s_j[2 * cp + u];
        const float w = IS_A ? 1.0f : s_w[2 * cp + u];
        // the means of the thread's row quad: one Philox block (r0 is a multiple of 4)
        const u32x4 mr = philox((uint32_t)j, (uint32_t)((rb + r0) >> 2), 0, MLSK_CTR_SMEAN, mkey);
        const uint32_t mw[4] = {mr.x, mr.y, mr.z, mr.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float x = 0.f;
            if (r0 + e < lim) {
                x = __fadd_rn(st_mean_of(mw[e], S.M.st_lo, S.M.st_w),
                              student_t_draw(key, j, rb + r0 + e, IS_A ? 0 : 1, T));
                x = __fmul_rn(IS_A ? ascale : w, x);
            }
            v[u][e] = x;
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (bfx == 2) {
            store_h16_pair(thi, r0 + e, 2 * cp, v[0][e], v[1][e]);
            continue;
        }
        if (bfx == 3) {
            store_h16b_pair(thi, tlo, r0 + e, 2 * cp, v[0][e], v[1][e]);
            continue;
        }
        const int off = sw_off(r0 + e, 2 * cp);
        *reinterpret_cast<float2*>(thi + off) = make_float2(v[0][e], v[1][e]);
        store_lo_pair(tlo, r0 + e, 2 * cp, v[0][e], v[1][e], bfx != 0);
    }
}

// work item (b, kc): 16 sampled columns; phases of 128 rows of A / cols of B;
// hi and lo tiles staged in shared memory in the SW64 layout, then copied out
// by the TMA engine.
// KIND: GK_GAUSS, GK_STUDENT_T, or GK_GENERIC (per-entry loop: RFF with D > 64)
constexpr int GK_GAUSS = 0, GK_STUDENT_T = 1, GK_GENERIC = 2;
#ifndef MLSK_TC_TWO
#define MLSK_TC_TWO 1
#endif
#ifndef MLSK_TC_CPS
// K-chunks per stage with FP16 pairs (16 KB of operands per chunk and CTA of a pair): 2 / 3 / 4 / 6 / 7
// chunks -> config 3 10.90 / 10.40 / 10.12 / 10.64 / 10.82, config 4 9.19 / 8.60 / 8.33 / 8.62 / 8.61 ms per step
#define MLSK_TC_CPS 4
#endif
#ifndef MLSK_TC_CPS3
#define MLSK_TC_CPS3 3  // the same with FP16 hi + BF16 (24 KB per chunk): 2 / 3 / 4 -> config 5 243.5 / 232.8 / 245.7 ms per step
#endif
#ifndef MLSK_GEN_CHUNK_MAJOR
#define MLSK_GEN_CHUNK_MAJOR 1
#endif
template <int KIND>
#ifndef MLSK_GAUSS_MINB
#define MLSK_GAUSS_MINB 5  // gauss: 4 / 5 / 6 CTAs per SM -> config 3 16.1 / 15.6 / 16.1 ms per step
#endif
#ifndef MLSK_ST_MINB
#define MLSK_ST_MINB 2  // Student-t: 2 / 3 / 4 CTAs per SM -> config 5 367 / 370 / 381 ms per step
#endif
__global__ void __launch_bounds__(GEN_T, KIND == GK_GAUSS ? MLSK_GAUSS_MINB : KIND == GK_STUDENT_T ? MLSK_ST_MINB : 1)
k_gen_panels_tf32(TcModel S, uint64_t seed, uint64_t tag, const int64_t* __restrict__ ks, int nb, int64_t c,
                  int64_t cc, float w_fine, float w_coarse, int64_t MP, int64_t PP, int64_t nkc, int64_t kc0,
                  float* __restrict__ Ahi, float* __restrict__ Alo, float* __restrict__ Bhi, float* __restrict__ Blo,
                  uint32_t* __restrict__ idx_out, const MkEntry* __restrict__ mk, int64_t mk_stride,
                  const MkInfo* __restrict__ mk_info, int bfx_i, float ascale, float wscale) {
    // ascale / wscale (FP16 hi + BF16, bfx == 3): powers of two on the A entries and on the B
    // weights that keep fp16(x) far from saturation (Student-t tails times weights up to
    // n / c); the GEMM's epilogue undoes them exactly
    const int bfx = bfx_i;  // 0: TF32 lo; 1: BF16 cross-term tiles; 2: FP16 pairs (one tile); 3: FP16 hi + BF16
    __shared__ __align__(1024) unsigned char tbuf[2][2][TTILE];  // [buffer][hi / lo], double-buffered
    __shared__ __align__(16) float2 s_sc[256];  // full-circle sincos table
    __shared__ __align__(16) float2 s_lg[64];
    __shared__ int s_j[TBK];
    __shared__ float s_w[TBK];
    const DevModel& M = S.M;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_sc[i] = full_circle_entry_f(i, M.tab.sincos_f);
    for (int i = threadIdx.x; i < 64; i += blockDim.x) s_lg[i] = reinterpret_cast<const float2*>(M.tab.log_f)[i];
    Tables T = M.tab;
    T.sincos_f = reinterpret_cast<const float*>(s_sc);
    T.log_f = reinterpret_cast<const float*>(s_lg);
    const int tid = threadIdx.x;
    const int64_t items = (int64_t)nb * nkc;
    const int a_ph = (int)(MP / TBM), b_ph = (int)(PP / TBM);  // 128-row phases (a B tile is two)
    int buf = 0;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        // merged lists are ordered by column, so chunk kc of every sample covers about
        // the same columns: chunk-major item order lets the CTAs running at one time
        // gather the same mean rows (L2 hits); draw-order lists run sample-major
        const int b = (int)(MLSK_GEN_CHUNK_MAJOR && mk ? it % nb : it / nkc);
        const int64_t kc = MLSK_GEN_CHUNK_MAJOR && mk ? it / nb : it - (int64_t)b * nkc;
        const uint64_t key = derive_seed(seed, tag, (uint64_t)ks[b]);
        __syncthreads();
        if (tid < TBK) {
            const int64_t t = (kc0 + kc) * TBK + tid;  // column of the sample (kc0: first chunk of this K-range)
            int j = 0;  // padding columns (t >= c): column 0 with weight 0 (B = 0)
            float w = 0.f;
            if (mk) {
                // merged sampled columns (KRange): slot t of the sample's (j, W_j) list
                if (t < mk_info[b].len) {
                    const MkEntry e = mk[(int64_t)b * mk_stride + t];
                    if (e.j >= 0) {
                        j = e.j;
                        w = (float)e.w;
                    }
                }
            } else if (t < c) {
                const u32x4 r = philox((uint32_t)(t >> 1), 0, 0, MLSK_CTR_INDEX, key);
                const uint32_t ix = index_from_u64((t & 1) ? hi64(r) : lo64(r), M.n, M.log2n, M.cum);
                j = (int)(ix - 1);
                w = t < cc ? w_coarse : w_fine;
                if (idx_out) idx_out[(int64_t)b * c + t] = ix;
            }
            s_j[tid] = j;
            s_w[tid] = __fmul_rn(w, wscale);
        }
        __syncthreads();
        for (int ph = 0; ph < a_ph + b_ph; ++ph) {
            const bool isA = ph < a_ph;
            const int64_t rb = (int64_t)(isA ? ph : ph - a_ph) * TBM;
            const int64_t lim = isA ? M.m - rb : M.p - rb;
            unsigned char* thi = tbuf[buf][0];
            unsigned char* tlo = tbuf[buf][1];
            if (KIND == GK_GAUSS) {
                if (isA) gauss_phase_f32<true>(M, T, key, rb, s_j, s_w, thi, tlo, tid, bfx);
                else gauss_phase_f32<false>(M, T, key, rb, s_j, s_w, thi, tlo, tid, bfx);
            } else if (KIND == GK_STUDENT_T) {
                if (isA) student_t_phase_f32<true>(S, T, key, rb, s_j, s_w, thi, tlo, tid, bfx, ascale);
                else student_t_phase_f32<false>(S, T, key, rb, s_j, s_w, thi, tlo, tid, bfx, ascale);
            } else {
                for (int item = tid; item < TBM * TBK; item += GEN_T) {
                    const int tt = item & (TBK - 1), rr = item / TBK;
                    const int j = s_j[tt];
                    float v = 0.f;
                    if (rr < lim) {
                        float x;
                        if (M.kind == MLSK_MODEL_STUDENT_T) x = student_t_entry(S, key, j, rb + rr, isA ? 0 : 1, T);
                        else x = rff_entry(M, j, rb + rr);  // RFF (D > 64): B = A^T
                        v = __fmul_rn(isA ? ascale : s_w[tt], x);
                    }
                    if (bfx == 2 || bfx == 3) {
                        const uint32_t h = f16x2_rn(v, 0.f);
                        float h0, h1;
                        f16x2_unpack(h, h0, h1);
                        *reinterpret_cast<unsigned short*>(thi + sw_off_b(rr, tt, 0)) = (unsigned short)(h & 0xffffu);
                        if (bfx == 2) {
                            *reinterpret_cast<unsigned short*>(thi + sw_off_b(rr, tt, 1)) =
                                (unsigned short)(f16x2_rn(__fsub_rn(v, h0), 0.f) & 0xffffu);
                        } else {
                            *reinterpret_cast<unsigned short*>(thi + sw_off_b(rr, tt, 1)) =
                                (unsigned short)(bf16x2_rn(v, 0.f) & 0xffffu);
                            *reinterpret_cast<unsigned short*>(tlo + sw32_off(rr, tt)) =
                                (unsigned short)(bf16x2_rn(__fsub_rn(v, h0), 0.f) & 0xffffu);
                        }
                        continue;
                    }
                    *reinterpret_cast<float*>(thi + sw_off(rr, tt)) = v;
                    if (bfx) {
                        *reinterpret_cast<unsigned short*>(tlo + sw_off_b(rr, tt, 0)) =
                            (unsigned short)(bf16x2_rn(v, 0.f) & 0xffffu);
                        *reinterpret_cast<unsigned short*>(tlo + sw_off_b(rr, tt, 1)) =
                            (unsigned short)(bf16x2_rn(tf32_lo(v), 0.f) & 0xffffu);
                    } else {
                        *reinterpret_cast<float*>(tlo + sw_off(rr, tt)) = tf32_lo(v);
                    }
                }
            }
            // both tiles leave by bulk copies (TMA engine), not by the threads
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                const int64_t off = (((int64_t)b * nkc + kc) * (isA ? MP : PP) + rb) * TBK;
                float* dh = (isA ? Ahi : Bhi) + off;
                bulk_store(dh, thi, TTILE);
                if (bfx == 3) bulk_store((isA ? Alo : Blo) + off / 2, tlo, LTILE);  // 32-byte rows: half the floats
                else if (bfx != 2) bulk_store((isA ? Alo : Blo) + off, tlo, TTILE);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // the other buffer is free
            }
            __syncthreads();
            buf ^= 1;
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// RFF features: Z[x][j] = sqrt(2/n) cos(w_j . x + b_j).  A_S = Z[:, S] and
// B_S = (w_t Z[:, j_t])^T, so the B chunk of columns [rb, rb+128) is the A
// chunk of rows [rb, rb+128) scaled by w_t: both come from one evaluation.
// The 128 x 32 dot products of a row block run from shared memory (X tile
// transposed for conflict-free reads, W columns broadcast).
constexpr int RFF_DMAX = 64;
constexpr int RFF_COLS = 32;               // sampled columns per work item (X tile reuse)
constexpr int RFF_CH = RFF_COLS / TBK;     // K-chunks per work item
constexpr int RFF_RSPLIT = 4;              // work items per column group (row-block ranges)
// 256 threads over 128-row X tiles (a 128-thread / 64-row variant small
// enough to sit beside a GEMM CTA was measured neutral in round 1: sharing the
// SM trades GEMM time for generator time one for one)
#ifndef MLSK_RFF_MINB
#define MLSK_RFF_MINB 3  // 79 registers, 3 CTAs per SM: config 4 16.70 -> 16.37 ms per step (4: 16.70)
#endif
constexpr int RFF_T = GEN_T, RFF_RB = TBM, RFF_MINB = MLSK_RFF_MINB;
// MLSK_RFF_MMA (default): the 128 x 32 x D phase products of a row block run on
// the tensor cores as 3xTF32 mma.sync (m16n8k8, one 16-row slab x four 8-column
// tiles per warp; hi x hi in one accumulator, the two cross terms in another,
// summed at the end: the large accumulator sees 8 MMAs, not 24) instead of 64
// FFMAs per entry: 0.38 k instead of 1.15 k instructions per thread and row
// block ahead of the cos / split / store epilogue.  The X and W tiles are
// padded by 8 floats per row so the fragment loads are conflict-free.
#ifndef MLSK_RFF_MMA
#define MLSK_RFF_MMA 1
#endif
constexpr int RFF_XS = MLSK_RFF_MMA ? RFF_RB + 8 : RFF_RB;      // X tile row stride (floats)
constexpr int RFF_WS = MLSK_RFF_MMA ? RFF_COLS + 8 : RFF_COLS;  // W tile row stride
constexpr int RFF_SMEM = (RFF_DMAX * RFF_XS + RFF_DMAX * RFF_WS) * 4;  // X tile + W columns (40 / 44 KB)

__device__ __forceinline__ void mma_tf32_16x8x8(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// work item (b, column group of 32 sampled columns, range of 128-row blocks):
// W columns and (per row block) the X tile in shared memory; each thread
// owns 4 consecutive columns x 4 consecutive rows and writes its 16-byte row
// pieces straight into the swizzled panels (no staging tiles: 40 KB of shared
// memory per CTA, five CTAs per SM).
__global__ void __launch_bounds__(RFF_T, RFF_MINB)
k_gen_panels_rff(TcModel S, uint64_t seed, uint64_t tag, const int64_t* __restrict__ ks, int nb, int64_t c,
                 int64_t cc, float w_fine, float w_coarse, int64_t MP, int64_t PP, int64_t nkc, int64_t kcg,
                 int write_b, float* __restrict__ Ahi,
                 float* __restrict__ Alo, float* __restrict__ Bhi, float* __restrict__ Blo,
                 uint32_t* __restrict__ idx_out, const MkEntry* __restrict__ mk, int64_t mk_stride,
                 const MkInfo* __restrict__ mk_info, int bfx_i, float pscale) {
    const int bfx = bfx_i;  // 0: TF32 lo tiles; 1: BF16 cross-term tiles; 2: FP16 pairs (one tile)
    extern __shared__ __align__(1024) unsigned char rsm[];
    float* xs = reinterpret_cast<float*>(rsm);  // [D][RFF_XS]
    float* wsm = xs + RFF_DMAX * RFF_XS;         // [D][RFF_WS]
    __shared__ int s_j[RFF_COLS];
    __shared__ float s_w[RFF_COLS], s_b[RFF_COLS];
    const DevModel& M = S.M;
    const int D = (int)M.rff_dim;
    const int D8 = MLSK_RFF_MMA ? (D + 7) & ~7 : D;
    const int tid = threadIdx.x;
    // (FP16 pairs: the features carry the model's power-of-two panel scale, undone in the GEMM's epilogue)
    const float scale = (float)M.rff_scale * pscale;
    const int64_t ngrp = (nkc + RFF_CH - 1) / RFF_CH;  // column groups of RFF_CH K-chunks
    const int64_t nrb = (MP > PP ? MP : PP) / RFF_RB;  // row blocks (A rows / B columns, m == p)
    const int64_t rb_per = (nrb + RFF_RSPLIT - 1) / RFF_RSPLIT;
    const int64_t items = (int64_t)nb * ngrp * RFF_RSPLIT;
    static_assert(RFF_COLS == 32 && RFF_T == 2 * RFF_RB && TBM % RFF_RB == 0, "4 x 4 thread tile map");
#if !MLSK_RFF_MMA
    const int t0 = 4 * (tid & 7), r0 = 4 * (tid >> 3);
    const int ch = t0 / TBK, tt = t0 % TBK;
#endif
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int64_t cgi = it / RFF_RSPLIT;
        const int rs = (int)(it - cgi * RFF_RSPLIT);
        const int b = (int)(cgi / ngrp);
        const int64_t kc0 = (cgi - (int64_t)b * ngrp) * RFF_CH;
        const uint64_t key = derive_seed(seed, tag, (uint64_t)ks[b]);
        __syncthreads();
        if (tid < RFF_COLS) {
            const int64_t t = (kcg + kc0) * TBK + tid;  // kcg: first chunk of this K-range
            int j = -1;
            float w = 0.f;
            if (mk) {
                // merged sampled columns (KRange); padding entries carry j = -1: a zero column
                if (t < mk_info[b].len) {
                    const MkEntry e = mk[(int64_t)b * mk_stride + t];
                    j = e.j;
                    w = (float)e.w;
                }
            } else if (t < c) {
                const u32x4 r = philox((uint32_t)(t >> 1), 0, 0, MLSK_CTR_INDEX, key);
                const uint32_t ix = index_from_u64((t & 1) ? hi64(r) : lo64(r), M.n, M.log2n, M.cum);
                j = (int)(ix - 1);
                w = t < cc ? w_coarse : w_fine;
                if (idx_out && rs == 0) idx_out[(int64_t)b * c + t] = ix;
            }
            s_j[tid] = j;
            s_w[tid] = w;
            s_b[tid] = j >= 0 ? M.rff_b[j] : 0.f;
        }
        __syncthreads();
        for (int e = tid; e < D8 * RFF_COLS; e += RFF_T) {  // (rows D .. D8: zero K padding of the MMAs)
            const int d = e / RFF_COLS, t = e - d * RFF_COLS;
            const int j = s_j[t];
            wsm[d * RFF_WS + t] = j >= 0 && d < D ? M.rff_w[(int64_t)d * M.n + j] : 0.f;
        }
        const bool colscale = mk != nullptr && !write_b;
#if !MLSK_RFF_MMA
        // this thread's columns: index, phase and weight are fixed over the item
        int jv[4];
        float bv[4], wv4[4];
#pragma unroll
        for (int cc4 = 0; cc4 < 4; ++cc4) {
            jv[cc4] = s_j[t0 + cc4];
            bv[cc4] = s_b[t0 + cc4];
            wv4[cc4] = s_w[t0 + cc4];
        }
        const int64_t kc = kc0 + ch;
        const bool col_ok = kc < nkc;
#endif
        const int64_t rb_end = nrb < (rs + 1) * rb_per ? nrb : (rs + 1) * rb_per;
        for (int64_t rbi = rs * rb_per; rbi < rb_end; ++rbi) {
            const int64_t rb = rbi * RFF_RB;
            const int64_t lim = M.m - rb;
            __syncthreads();  // previous X tile consumed
            // X tile from the transposed copy: rows contiguous per dimension, so
            // the global reads coalesce and the shared stores are conflict-free
            if (lim >= RFF_RB && (M.m & 3) == 0 && D8 == D) {
                for (int e = tid; e < RFF_RB / 4 * D; e += RFF_T) {
                    const int d = e / (RFF_RB / 4), r4 = e - d * (RFF_RB / 4);
                    reinterpret_cast<float4*>(xs + d * RFF_XS)[r4] =
                        __ldg(reinterpret_cast<const float4*>(M.rff_xt + (int64_t)d * M.m + rb) + r4);
                }
            } else {
                for (int e = tid; e < RFF_RB * D8; e += RFF_T) {
                    const int d = e / RFF_RB, r = e - d * RFF_RB;
                    xs[d * RFF_XS + r] = r < lim && d < D ? M.rff_xt[(int64_t)d * M.m + rb + r] : 0.f;
                }
            }
            __syncthreads();
#if MLSK_RFF_MMA
            // warp = rows 16 warp .. +15 of the block x the item's 32 columns
            const int lane = tid & 31, wrp = tid >> 5, g = lane >> 2, tq = lane & 3;
            float cm[4][4], cx[4][4];  // [n8 tile][fragment]: hi x hi, and the cross terms
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int q = 0; q < 4; ++q) cm[nt][q] = cx[nt][q] = 0.f;
            const float* xa = xs + 16 * wrp + g;
            const float* wb = wsm + g;
            for (int k0 = 0; k0 < D8; k0 += 8) {
                // A fragment (rows g, g + 8; k = tq, tq + 4): the mma reads the
                // TF32 part of the fp32 word (hi); lo = x - tf32(x)
                uint32_t ah[4], al[4];
                const float a0 = xa[(k0 + tq) * RFF_XS], a1 = xa[(k0 + tq) * RFF_XS + 8];
                const float a2 = xa[(k0 + tq + 4) * RFF_XS], a3 = xa[(k0 + tq + 4) * RFF_XS + 8];
                ah[0] = __float_as_uint(a0); ah[1] = __float_as_uint(a1);
                ah[2] = __float_as_uint(a2); ah[3] = __float_as_uint(a3);
                al[0] = __float_as_uint(tf32_lo(a0)); al[1] = __float_as_uint(tf32_lo(a1));
                al[2] = __float_as_uint(tf32_lo(a2)); al[3] = __float_as_uint(tf32_lo(a3));
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                    const float b0 = wb[(k0 + tq) * RFF_WS + 8 * nt], b1 = wb[(k0 + tq + 4) * RFF_WS + 8 * nt];
                    const uint32_t bh[2] = {__float_as_uint(b0), __float_as_uint(b1)};
                    const uint32_t bl[2] = {__float_as_uint(tf32_lo(b0)), __float_as_uint(tf32_lo(b1))};
                    mma_tf32_16x8x8(cm[nt], ah, bh);
                    mma_tf32_16x8x8(cx[nt], ah, bl);
                    mma_tf32_16x8x8(cx[nt], al, bh);
                }
            }
            const int64_t rt = rb & ~(int64_t)(TBM - 1);  // the 128-row panel tile holding this block
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const int cl = 8 * nt + 2 * tq;  // this thread's two adjacent columns of the item
                const int64_t kcn = kc0 + cl / TBK;
                if (kcn >= nkc) continue;
                const int ttn = cl % TBK;
                const int j0 = s_j[cl], j1 = s_j[cl + 1];
                const float b0 = s_b[cl], b1 = s_b[cl + 1], w0 = s_w[cl], w1 = s_w[cl + 1];
                const int64_t oa = ((b * nkc + kcn) * MP + rt) * TBK;
                const int64_t ob = ((b * nkc + kcn) * PP + rt) * TBK;  // B panels are padded to 256
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int rr = 16 * wrp + g + 8 * h;  // row within the block
                    float z0 = 0.f, z1 = 0.f;
                    if (rr < lim) {
                        if (j0 >= 0) z0 = scale * cosf(__fadd_rn(cm[nt][2 * h], cx[nt][2 * h]) + b0);
                        if (j1 >= 0) z1 = scale * cosf(__fadd_rn(cm[nt][2 * h + 1], cx[nt][2 * h + 1]) + b1);
                    }
                    // merged columns on the shared panel: |w| is the column scale sqrt(reps)
                    if (colscale) {
                        z0 = __fmul_rn(fabsf(w0), z0);
                        z1 = __fmul_rn(fabsf(w1), z1);
                    }
                    const int rti = (int)(rb - rt) + rr;  // row within the 128-row panel tile
                    const int off = sw_off(rti, ttn) / 4;  // floats
                    if (bfx == 2) {  // FP16 pairs: one tile per operand
                        if (rb < MP) store_h16_pair(reinterpret_cast<unsigned char*>(Ahi + oa), rti, ttn, z0, z1);
                        if (write_b && rb < PP)
                            store_h16_pair(reinterpret_cast<unsigned char*>(Bhi + ob), rti, ttn, __fmul_rn(w0, z0),
                                           __fmul_rn(w1, z1));
                        continue;
                    }
                    if (rb < MP) {
                        *reinterpret_cast<float2*>(Ahi + oa + off) = make_float2(z0, z1);
                        store_lo_pair(reinterpret_cast<unsigned char*>(Alo + oa), rti, ttn, z0, z1, bfx != 0);
                    }
                    if (write_b && rb < PP) {
                        const float v0 = __fmul_rn(w0, z0), v1 = __fmul_rn(w1, z1);
                        *reinterpret_cast<float2*>(Bhi + ob + off) = make_float2(v0, v1);
                        store_lo_pair(reinterpret_cast<unsigned char*>(Blo + ob), rti, ttn, v0, v1, bfx != 0);
                    }
                }
            }
#else
            // per dimension one 16-byte W read and one 16-byte X read (both
            // broadcast within the warp) feed 16 FMAs; each entry sums over d
            // in order (rff_entry)
            float acc[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;
#pragma unroll 4
            for (int d = 0; d < D; ++d) {
                const float4 wv = *reinterpret_cast<const float4*>(wsm + d * RFF_WS + t0);
                const float4 xv = *reinterpret_cast<const float4*>(xs + d * RFF_XS + r0);
                const float xa[4] = {xv.x, xv.y, xv.z, xv.w}, wa[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[i][q] = __fmaf_rn(xa[i], wa[q], acc[i][q]);
            }
            if (!col_ok) continue;
            const int64_t rt = rb & ~(int64_t)(TBM - 1);  // the 128-row panel tile holding this block
            const int64_t oa = (((int64_t)b * nkc + kc) * MP + rt) * TBK;
            const int64_t ob = (((int64_t)b * nkc + kc) * PP + rt) * TBK;  // B panels are padded to 256
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = (int)(rb - rt) + r0 + i;  // row within the 128-row tile
                float z[4], v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    z[q] = 0.f;
                    if (jv[q] >= 0 && r0 + i < lim) z[q] = scale * cosf(acc[i][q] + bv[q]);
                    // merged columns on the shared panel: |w| is the column scale sqrt(reps)
                    if (colscale) z[q] = __fmul_rn(fabsf(wv4[q]), z[q]);
                    v[q] = __fmul_rn(wv4[q], z[q]);
                }
                const int off = sw_off(r, tt) / 4;  // floats
                if (bfx == 2) {
                    if (rb < MP) {
                        store_h16_pair(reinterpret_cast<unsigned char*>(Ahi + oa), r, tt, z[0], z[1]);
                        store_h16_pair(reinterpret_cast<unsigned char*>(Ahi + oa), r, tt + 2, z[2], z[3]);
                    }
                    if (write_b && rb < PP) {
                        store_h16_pair(reinterpret_cast<unsigned char*>(Bhi + ob), r, tt, v[0], v[1]);
                        store_h16_pair(reinterpret_cast<unsigned char*>(Bhi + ob), r, tt + 2, v[2], v[3]);
                    }
                    continue;
                }
                if (rb < MP) {
                    *reinterpret_cast<float4*>(Ahi + oa + off) = make_float4(z[0], z[1], z[2], z[3]);
                    if (bfx) {
                        store_lo_pair(reinterpret_cast<unsigned char*>(Alo + oa), r, tt, z[0], z[1], true);
                        store_lo_pair(reinterpret_cast<unsigned char*>(Alo + oa), r, tt + 2, z[2], z[3], true);
                    } else {
                        *reinterpret_cast<float4*>(Alo + oa + off) =
                            make_float4(tf32_lo(z[0]), tf32_lo(z[1]), tf32_lo(z[2]), tf32_lo(z[3]));
                    }
                }
                if (write_b && rb < PP) {
                    *reinterpret_cast<float4*>(Bhi + ob + off) = make_float4(v[0], v[1], v[2], v[3]);
                    if (bfx) {
                        store_lo_pair(reinterpret_cast<unsigned char*>(Blo + ob), r, tt, v[0], v[1], true);
                        store_lo_pair(reinterpret_cast<unsigned char*>(Blo + ob), r, tt + 2, v[2], v[3], true);
                    } else {
                        *reinterpret_cast<float4*>(Blo + ob + off) =
                            make_float4(tf32_lo(v[0]), tf32_lo(v[1]), tf32_lo(v[2]), tf32_lo(v[3]));
                    }
                }
            }
#endif
        }
    }
}

// --------------------------------------------------------------- GEMM

struct TcShape {
    int nb;
    int64_t nkc;
    int64_t MP, PP;
    int T, Gs, tiles_n;
    // Gs == 1 (one CTA per tile): running sums go straight into the level
    // total (rows x cols, row-major) -- no partial buffer, no reduction pass
    double* direct;
    int64_t rows, cols;
    // kpar (SPLIT instantiation, one sample): group g of the T-CTA groups takes
    // K-chunks [g * ceil(nkc / 2), ...) and stores its partial Y into its own
    // ypart slot; k_kpar_combine forms Y, ||Y||^2 and the level total
    int kpar;
    // symmetric output (RFF Gram: B = diag(w) A^T, so Y = A_S D A_S^T): the
    // tiles cover only the 256 x 256 blocks (R, C) with R <= C, sym_nb blocks
    // per side (0 = full tile grid).  Off-diagonal blocks count twice in
    // ||Y||^2; k_mirror_lower fills the lower blocks of the level total.
    int sym_nb;
    // shared panel (RFF Gram, |w| a power of two on every column): B = A^T is
    // read from the A panel; the K-chunks below neg_kc (absolute index, kc0 =
    // first chunk of this launch's K-range) run with the B operand negated and
    // the epilogue scales Y by escale = |w| -- bit-identical to B = diag(w) A^T
    int64_t neg_kc, kc0;
    float escale;
    // merged sampled columns on the shared panel: the negated leading chunks
    // per sample (mk_info[b].neg_kc) instead of neg_kc
    const MkInfo* mk_info;
    // 1: BF16 cross terms (the lo tiles' rows hold bf16(x) | bf16(x - tf32(x)));
    // 2: FP16 pairs (one tile per operand, rows fp16(x) | fp16(x - fp16(x)));
    // 3: FP16 hi + BF16 cross terms (rows fp16(x) | bf16(x), and a tile of bf16(x - fp16(x)))
    int bfx;
    // K-chunks per TMEM accumulation segment (0: a CTA's whole K-range of a
    // sample is one segment).  tcgen05's fp32 accumulation rounds the running
    // sum toward zero, so its error grows with the number of MMAs folded into
    // one accumulator (measured: ~4e-8 relative per MMA, 1.3e-4 at K = 16384);
    // long samples restart the accumulator every `seg` K-chunks and the
    // epilogue adds the segments in registers with round-to-nearest.
    int seg = 0;
};

// tile index -> (tile row of 128, tile column of 256).  Full grids run in
// groups of RASTER_G tile rows, column by column inside a group: the CTAs
// resident at one time (148 of config 5's 2048 tiles) then cover about 8 x 18
// tiles instead of 4.6 rows x all 32 columns, so the panel chunks they share
// come from L2 and not once per wave from DRAM (config 5 at c = 512: 2.6 GB
// of DRAM reads per launch for 268 MB of panels before).  The group height
// must stay even (CTA pairs take tile rows 2u, 2u + 1).
#ifndef MLSK_TC_RASTER_G
#define MLSK_TC_RASTER_G 8  // config 5 (pairs): 4 / 8 / 16 / 32 rows: 382 / 369 / 381 / 400 ms per step
#endif
constexpr int RASTER_G = MLSK_TC_RASTER_G;
__device__ __forceinline__ void tile_coords(const TcShape& sh, int tile, int& tm, int& tn) {
    if (sh.sym_nb == 0) {
        const int rows_t = sh.T / sh.tiles_n;
        const int blk = tile / (RASTER_G * sh.tiles_n);
        const int r0 = blk * RASTER_G;
        const int rg = rows_t - r0 < RASTER_G ? rows_t - r0 : RASTER_G;  // rows in this group
        const int w = tile - blk * RASTER_G * sh.tiles_n;
        tm = r0 + w % rg;
        tn = w / rg;
        return;
    }
    // blocks (R, C >= R) in row-major order, two 128-row tiles per block
    const int u = tile >> 1;
    int R = 0, start = 0;
    while (u >= start + (sh.sym_nb - R)) {
        start += sh.sym_nb - R;
        ++R;
    }
    tm = 2 * R + (tile & 1);
    tn = R + (u - start);
}

// (tile row, tile column) -> tile index; -1 for a block below the diagonal
__device__ __forceinline__ int tile_index(const TcShape& sh, int tm, int tn) {
    if (sh.sym_nb == 0) {
        const int rows_t = sh.T / sh.tiles_n;
        const int r0 = tm / RASTER_G * RASTER_G;
        const int rg = rows_t - r0 < RASTER_G ? rows_t - r0 : RASTER_G;
        return r0 * sh.tiles_n + tn * rg + (tm - r0);
    }
    const int R = tm >> 1;
    if (R > tn) return -1;
    return 2 * (R * sh.sym_nb - R * (R - 1) / 2 + (tn - R)) + (tm & 1);
}

// SPLIT: one sample split along K per launch (split_part 1 first, 2 middle,
// 3 last, partial Y in ypart); a separate instantiation for the common path.
// SEGM: a sample's K-range runs as several TMEM accumulation segments of
// sh.seg K-chunks (TcShape::seg) summed in registers; else one segment.
// PAIR: clusters of two CTAs on tiles (tm, tn), (tm + 1, tn): the leader
// (rank 0) issues tcgen05.mma.cta_group::2 (M = 256) over both CTAs' shared
// memory, each CTA loading its A rows and half of the B columns (a third less
// shared-memory traffic per SM than the single-CTA tile, six stages); the
// peer relays its stage arrivals to the leader, both epilogues read their
// own TMEM lanes and release the accumulator to the leader.
template <bool SPLIT, bool SEGM, bool PAIR>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_gemm_tf32x3(const float* __restrict__ Ahi, const float* __restrict__ Alo, const float* __restrict__ Bhi,
              const float* __restrict__ Blo, TcShape sh, double* __restrict__ part, double* __restrict__ part_sq,
              int split_part, float* __restrict__ ypart) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    // 1024-byte aligned stage ring (SW128 atoms)
    unsigned char* ring = dsm + ((1024 - (smem_addr(dsm) & 1023)) & 1023);
    constexpr int NST = PAIR ? PSTAGES : TSTAGES;
    constexpr int STB = PAIR ? PSTAGE_BYTES : TSTAGE_BYTES;
    constexpr int BB = PAIR ? PB_BYTES : TB_BYTES;  // B bytes per stage held by this CTA
    // full[NST], empty[NST], tmem_full[2], tmem_empty[2], tmem_done, pair: peer_full[NST], pair_done
    __shared__ __align__(8) uint64_t bars[3 * PSTAGES + 6];
    __shared__ uint32_t s_tmem;
    __shared__ double s_sq[EPI_WARPS];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x;
    const int tile = g % sh.T, grp = g / sh.T;
    int tm, tn;
    tile_coords(sh, tile, tm, tn);
    const bool kpar = SPLIT && sh.kpar;
    const int my_samples = kpar ? 1 : grp < sh.nb ? (sh.nb - 1 - grp) / sh.Gs + 1 : 0;
    const int64_t kh = (sh.nkc + 1) / 2;
    const int64_t kb = kpar ? grp * kh : 0;                              // this CTA's K-chunk range
    const int64_t ke = kpar ? (kb + kh < sh.nkc ? kb + kh : sh.nkc) : sh.nkc;
    const int64_t iters = (int64_t)my_samples * (ke - kb);
    const int64_t seg = SEGM && sh.seg > 0 && sh.seg < ke - kb ? sh.seg : ke - kb;  // K-chunks per TMEM segment
    const int nseg = (int)((ke - kb + seg - 1) / seg);                             // segments per sample
    // FP16 pairs: a stage holds several K-chunks (MLSK_TC_CPS blocks of the chunk's
    // 16 KB of operands), so barrier round trips, commits and relays are paid per
    // 64 columns instead of per 16.  Chunks group inside a sample and a TMEM
    // segment only.
    // FP16 hi + BF16 (a chunk is 24 KB of operands per CTA of a pair): stages of
    // MLSK_TC_CPS3 chunk blocks.
    const bool two3 = MLSK_TC_TWO && PAIR && sh.bfx == 3;
    const bool two2 = MLSK_TC_TWO && sh.bfx == 2;
    constexpr int CH2 = TA_BYTES + BB;            // one chunk's operands, FP16 pairs: A | B
    constexpr int CH3 = (TA_BYTES + BB) * 3 / 2;  // FP16 hi + BF16: A1 | A2 | B1 | B2
    const int maxn = two2 ? MLSK_TC_CPS : two3 ? MLSK_TC_CPS3 : 1;  // K-chunks per stage
    const int stb = two2 ? MLSK_TC_CPS * CH2 : two3 ? MLSK_TC_CPS3 * CH3 : STB;  // stage stride
    const int nst = (NST * STB) / stb < NST ? (NST * STB) / stb : NST;  // stages in the ring
    auto step_n = [&](int64_t kc_, int64_t sgc_) {
        int64_t r = ke - kc_ < seg - sgc_ ? ke - kc_ : seg - sgc_;
        return (int)(r < maxn ? r : maxn);
    };

    const uint32_t full0 = smem_addr(&bars[0]), empty0 = smem_addr(&bars[NST]);
    const uint32_t tfull0 = smem_addr(&bars[2 * NST]), tempty0 = smem_addr(&bars[2 * NST + 2]);
    const uint32_t tdone = smem_addr(&bars[2 * NST + 4]);
    const uint32_t pfull0 = smem_addr(&bars[2 * NST + 5]), pdone = smem_addr(&bars[3 * NST + 5]);
    uint32_t rank = 0;
    if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            bar_init(full0 + 8 * s, 1);
            bar_init(empty0 + 8 * s, 1);
            if (PAIR) bar_init(pfull0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            bar_init(tfull0 + 8 * a, 1);
            bar_init(tempty0 + 8 * a, PAIR ? 2 * EPI_WARPS : EPI_WARPS);  // pair: both CTAs' epilogues (leader's)
        }
        bar_init(tdone, EPI_WARPS);  // every epilogue warp finished with TMEM
        if (PAIR) bar_init(pdone, 2);  // both CTAs done with the pair's TMEM
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&s_tmem)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&s_tmem)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR)  // both CTAs' barriers initialised before any remote arrive / multicast commit
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    // Role dispatch.  Each setmaxnreg dominates its role's code and the roles
    // do not join again (no common tail): ptxas then allocates each region
    // within its own register budget.
    if (warp < CTRL_WARPS) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(CTRL_REGS));
    if (warp == 0) {
        // --------------------------------------------------- producer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            int64_t b = kpar ? 0 : grp, kc = kb, sgc = 0;
            for (int64_t it = 0; it < iters;) {
                const int n = step_n(kc, sgc);  // K-chunks of this stage
                // (pair: freed by the leader's multicast commit)
                if (PAIR) bar_wait_cluster(empty0 + 8 * s, ph ^ 1);
                else bar_wait(empty0 + 8 * s, ph ^ 1);
                const uint32_t full = full0 + 8 * s;
#ifdef MLSK_TC_ABL_NOLD  // ablation (timing only, wrong results): no operand loads
                bar_arrive(full);
#else
                const bool h16 = sh.bfx == 2;  // FP16 pairs: one tile per operand (half the bytes)
                const bool h16b = sh.bfx == 3;  // FP16 hi | BF16 values + a BF16 lo tile of half the size
                bar_expect_tx(full, h16 ? n * (TA_BYTES + BB) : h16b ? n * CH3 : STB);
                MLSK_DCHECK(b < (kpar ? 1 : sh.nb) && kc + n <= sh.nkc && (int64_t)tm * TBM < sh.MP &&
                            (int64_t)tn * TBN < sh.PP);
                const int64_t oa = ((b * sh.nkc + kc) * sh.MP + (int64_t)tm * TBM) * TBK;
                // (pair: this CTA's half of the B tile, columns tn 256 + rank 128 ..)
                const int64_t ob = ((b * sh.nkc + kc) * sh.PP + (int64_t)tn * TBN + (PAIR ? rank * TBM : 0)) * TBK;
                const uint32_t st = smem_addr(ring + s * stb);
                if (h16b) {
                    // FP16 hi + BF16: per chunk a block A1 | A2 | B1 | B2 (A2, B2: the half-size lo tiles)
                    for (int q = 0; q < n; ++q) {
                        const uint32_t blk = st + q * CH3;
                        const int64_t qa = oa + q * sh.MP * TBK, qb = ob + q * sh.PP * TBK;
                        bulk_load(blk, Ahi + qa, TA_BYTES, full);
                        bulk_load(blk + TA_BYTES, Alo + qa / 2, TA_BYTES / 2, full);
                        bulk_load(blk + TA_BYTES * 3 / 2, Bhi + qb, BB, full);
                        bulk_load(blk + TA_BYTES * 3 / 2 + BB, Blo + qb / 2, BB / 2, full);
                    }
                } else if (h16) {
                    // FP16 pairs: per chunk a block A | B
                    for (int q = 0; q < n; ++q) {
                        const uint32_t blk = st + q * CH2;
                        bulk_load(blk, Ahi + oa + q * sh.MP * TBK, TA_BYTES, full);
                        bulk_load(blk + TA_BYTES, Bhi + ob + q * sh.PP * TBK, BB, full);
                    }
                } else {
                    bulk_load(st, Ahi + oa, TA_BYTES, full);
                    bulk_load(st + TA_BYTES, Alo + oa, TA_BYTES, full);
                    bulk_load(st + 2 * TA_BYTES, Bhi + ob, BB, full);
                    bulk_load(st + 2 * TA_BYTES + BB, Blo + ob, BB, full);
                }
#endif
                if (++s == nst) { s = 0; ph ^= 1; }
                it += n;
                kc += n;
                sgc += n;
                if (kc == ke) { kc = kb; b += sh.Gs; sgc = 0; }
                else if (sgc >= seg) sgc = 0;
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (PAIR && rank == 1) {
            // the peer's stage arrivals relayed to the leader, which issues the
            // pair's MMAs over both CTAs' shared memory
            if (lane == 0) {
                int s = 0;
                uint32_t ph = 0;
                const uint32_t lead_pfull0 = cluster_addr(pfull0, 0);
                int64_t kc = kb, sgc = 0;
                for (int64_t it = 0; it < iters;) {
                    const int n = step_n(kc, sgc);
                    bar_wait(full0 + 8 * s, ph);
                    bar_arrive_remote(lead_pfull0 + 8 * s);
                    if (++s == nst) { s = 0; ph ^= 1; }
                    it += n;
                    kc += n;
                    sgc += n;
                    if (kc == ke) { kc = kb; sgc = 0; }
                    else if (sgc >= seg) sgc = 0;
                }
            }
        } else if (lane == 0) {
            constexpr uint32_t idesc = tf32_idesc(PAIR ? 2 * TBM : TBM, TBN);
            int s = 0;
            uint32_t ph = 0;
            int64_t kc = kb;
            int64_t sgc = 0;  // K-chunks of the current accumulation segment so far
            int abuf = 0;
            uint32_t aph = 0;  // bit a = phase of accumulator a (no indexed local array)
            int sb = kpar ? 0 : grp;  // current sample (merged shared panel: its negated chunks)
            int64_t neg_kc = sh.mk_info ? (sb < sh.nb ? sh.mk_info[sb].neg_kc : 0) : sh.neg_kc;
            for (int64_t it = 0; it < iters;) {
                const int n = step_n(kc, sgc);  // K-chunks of this stage (FP16 pairs: up to two)
                if (sgc == 0) {  // first K-chunk of a segment (kpar: this CTA's range starts at kb > 0)
                    // the epilogue(s) released this accumulator
                    if (PAIR) bar_wait_cluster(tempty0 + 8 * abuf, ((aph >> abuf) & 1u) ^ 1u);
                    else bar_wait(tempty0 + 8 * abuf, ((aph >> abuf) & 1u) ^ 1u);
                    tc_fence_after();
                }
                bar_wait(full0 + 8 * s, ph);
                if (PAIR) bar_wait_cluster(pfull0 + 8 * s, ph);  // the peer's half of the stage
                tc_fence_after();
                const uint32_t st = smem_addr(ring + s * stb);
                const uint32_t dcol = tmem + (uint32_t)abuf * TBN;
                const uint32_t id = sh.kc0 + kc < neg_kc ? idesc | (1u << 14) : idesc;  // negate B
                if (sh.bfx == 2) {
                    // FP16 pairs: hi x hi, hi x lo, lo x hi over the row halves of the one tile,
                    // for each of the stage's chunks
                    constexpr uint32_t idh0 = f16_idesc(PAIR ? 2 * TBM : TBM, TBN);
#ifndef MLSK_TC_ABL_NOMMA
                    for (int q = 0; q < n; ++q) {
                        const uint32_t idh = sh.kc0 + kc + q < neg_kc ? idh0 | (1u << 14) : idh0;
                        const uint32_t sa = st + q * CH2, sbh = sa + TA_BYTES;  // the chunk's block A | B
                        const uint32_t acc0 = sgc + q > 0 ? 1u : 0u;
                        if (PAIR) {
                            tc_mma_bf16_pair(dcol, sw_desc(sa), sw_desc(sbh), idh, acc0);
                            tc_mma_bf16_pair(dcol, sw_desc(sa), sw_desc(sbh + 32), idh, 1u);
                            tc_mma_bf16_pair(dcol, sw_desc(sa + 32), sw_desc(sbh), idh, 1u);
                        } else {
                            tc_mma_bf16(dcol, sw_desc(sa), sw_desc(sbh), idh, acc0);
                            tc_mma_bf16(dcol, sw_desc(sa), sw_desc(sbh + 32), idh, 1u);
                            tc_mma_bf16(dcol, sw_desc(sa + 32), sw_desc(sbh), idh, 1u);
                        }
                    }
#endif
                } else if (sh.bfx == 3) {
                    // FP16 hi x hi; the cross terms as BF16 MMAs: bf16(x) is the second row half of
                    // the first tile, the lo parts are the SWIZZLE_32B tile
                    constexpr uint32_t idh0 = f16_idesc(PAIR ? 2 * TBM : TBM, TBN);
                    constexpr uint32_t idb0 = bf16_idesc(PAIR ? 2 * TBM : TBM, TBN);
#ifndef MLSK_TC_ABL_NOMMA
                    for (int q = 0; q < n; ++q) {
                        const uint32_t ng = sh.kc0 + kc + q < neg_kc ? (1u << 14) : 0u;
                        const uint32_t blk = st + q * CH3;  // A1 | A2 | B1 | B2
                        const uint32_t sal = blk + TA_BYTES, sbh = blk + TA_BYTES * 3 / 2, sbl = sbh + BB;
                        const uint32_t acc0 = sgc + q > 0 ? 1u : 0u;
                        if (PAIR) {
                            tc_mma_bf16_pair(dcol, sw_desc(blk), sw_desc(sbh), idh0 | ng, acc0);
                            tc_mma_bf16_pair(dcol, sw_desc(blk + 32), sw32_desc(sbl), idb0 | ng, 1u);   // x b_lo
                            tc_mma_bf16_pair(dcol, sw32_desc(sal), sw_desc(sbh + 32), idb0 | ng, 1u);  // a_lo x
                        } else {
                            tc_mma_bf16(dcol, sw_desc(blk), sw_desc(sbh), idh0 | ng, acc0);
                            tc_mma_bf16(dcol, sw_desc(blk + 32), sw32_desc(sbl), idb0 | ng, 1u);
                            tc_mma_bf16(dcol, sw32_desc(sal), sw_desc(sbh + 32), idb0 | ng, 1u);
                        }
                    }
#endif
                } else if (sh.bfx) {
                    // hi x hi as two TF32 MMAs (K = 8 each), the cross terms a b_lo and
                    // a_lo b as two BF16 MMAs (K = 16) over the row halves of the lo tiles
                    constexpr uint32_t idb0 = bf16_idesc(PAIR ? 2 * TBM : TBM, TBN);
                    const uint32_t idb = sh.kc0 + kc < neg_kc ? idb0 | (1u << 14) : idb0;
                    const uint32_t sal = st + TA_BYTES, sbh = st + 2 * TA_BYTES, sbl = sbh + BB;
#ifndef MLSK_TC_ABL_NOMMA
                    if (PAIR) {
                        tc_mma_tf32_pair(dcol, sw_desc(st), sw_desc(sbh), id, sgc > 0 ? 1u : 0u);
                        tc_mma_tf32_pair(dcol, sw_desc(st + 32), sw_desc(sbh + 32), id, 1u);
                        tc_mma_bf16_pair(dcol, sw_desc(sal), sw_desc(sbl + 32), idb, 1u);   // a b_lo
                        tc_mma_bf16_pair(dcol, sw_desc(sal + 32), sw_desc(sbl), idb, 1u);   // a_lo b
                    } else {
                        tc_mma_tf32(dcol, sw_desc(st), sw_desc(sbh), id, sgc > 0 ? 1u : 0u);
                        tc_mma_tf32(dcol, sw_desc(st + 32), sw_desc(sbh + 32), id, 1u);
                        tc_mma_bf16(dcol, sw_desc(sal), sw_desc(sbl + 32), idb, 1u);
                        tc_mma_bf16(dcol, sw_desc(sal + 32), sw_desc(sbl), idb, 1u);
                    }
#endif
                } else
#pragma unroll
                for (int kk = 0; kk < TBK / 8; ++kk) {
                    const uint64_t ah = sw_desc(st + kk * 32), al = sw_desc(st + TA_BYTES + kk * 32);
                    const uint64_t bh = sw_desc(st + 2 * TA_BYTES + kk * 32);
                    const uint64_t bl = sw_desc(st + 2 * TA_BYTES + BB + kk * 32);
#ifndef MLSK_TC_ABL_NOMMA  // ablation: no MMAs (commits only)
                    if (PAIR) {
                        tc_mma_tf32_pair(dcol, ah, bh, id, (sgc > 0 || kk > 0) ? 1u : 0u);
                        tc_mma_tf32_pair(dcol, ah, bl, id, 1u);
                        tc_mma_tf32_pair(dcol, al, bh, id, 1u);
                    } else {
                        tc_mma_tf32(dcol, ah, bh, id, (sgc > 0 || kk > 0) ? 1u : 0u);
                        tc_mma_tf32(dcol, ah, bl, id, 1u);
                        tc_mma_tf32(dcol, al, bh, id, 1u);
                    }
#endif
                }
                // smem stage free once these MMAs complete (pair: in both CTAs)
                if (PAIR) tc_commit_pair(empty0 + 8 * s);
                else tc_commit(empty0 + 8 * s);
                if (++s == nst) { s = 0; ph ^= 1; }
                it += n;
                sgc += n;
                kc += n;
                const bool sample_end = kc == ke;
                if (sample_end) {
                    kc = kb;
                    sb += sh.Gs;
                    if (sh.mk_info && sb < sh.nb) neg_kc = sh.mk_info[sb].neg_kc;
                }
                if (sample_end || sgc >= seg) {
                    sgc = 0;
                    if (PAIR) tc_commit_pair(tfull0 + 8 * abuf);  // accumulator segment complete
                    else tc_commit(tfull0 + 8 * abuf);
                    aph ^= 1u << abuf;
                    abuf ^= 1;
                }
            }
        }
        // TMEM is freed once every epilogue warp has read its last accumulator
        // (pair: in both CTAs -- each CTA's warp 1 arrives on both pair_done)
        __syncwarp();
        bar_wait(tdone, 0);
        if (PAIR) {
            if (lane == 0) {
                bar_arrive_remote(cluster_addr(pdone, 0));
                bar_arrive_remote(cluster_addr(pdone, 1));
            }
            __syncwarp();
            bar_wait_cluster(pdone, 0);
        }
        tc_fence_after();
        if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
    return;  // warps 2, 3: idle
    }
    {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(EPI_REGS));
        // --------------------------------------------------- epilogue
        const int ew = warp - CTRL_WARPS;      // 0 .. EPI_WARPS-1
        const int q = warp & 3;                // TMEM lane quadrant of this warp
        const int h = ew >> 2;                 // column quarter
        const int row = q * 32 + lane;         // tile row owned by this thread
        constexpr int HC = TBN / (EPI_WARPS / 4);  // columns per epilogue warp
        float R[HC];
#pragma unroll
        for (int i = 0; i < HC; ++i) R[i] = 0.f;
        double sq = 0.0;
        // per-CTA partial tile, column-major ([col][row]): for a fixed column the
        // 32 lanes (rows) of a warp touch 256 contiguous bytes, so a flush is 2 x 64
        // coalesced accesses per thread (row-major flushes cost 0.9 ms per config-3
        // level 0: one 32-byte sector per 8-byte access)
        double* out = part + (int64_t)g * (TBM * TBN) + (int64_t)(h * HC) * TBM + row;
        // segmented samples (one flush per sample): an fp32 partial tile in
        // the same column-major layout, summed by red.add (zeroed per launch)
        float* outf = reinterpret_cast<float*>(part) + (int64_t)g * (TBM * TBN) + (int64_t)(h * HC) * TBM + row;
        int abuf = 0;
        uint32_t aph = 0;  // bit a = phase of accumulator a (no indexed local array)
        // R: the fp32 running sum S over samples when a sample is one TMEM
        // segment (flushed every FLUSH samples); with several segments per
        // sample, the sample's Y accumulated over its segments (flushed every
        // sample)
        constexpr bool segmented = SEGM;  // R holds the sample's Y, flushed every sample
        // one 16-column piece of the accumulator in buffer `ab` (|w| applied)
        auto load = [&](int ab, int ch, float (&y)[16]) {
#ifdef MLSK_TC_ABL_NOEPI  // ablation: no accumulator reads
            for (int i = 0; i < 16; ++i) y[i] = (float)i;
#else
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * TBN + h * HC + ch * 16), y);
#endif
            if (sh.escale != 1.0f) {  // shared panel: |w| (a power of two, exact)
#pragma unroll
                for (int i = 0; i < 16; ++i) y[i] = __fmul_rn(y[i], sh.escale);
            }
        };
        auto wait_full = [&]() {
            if (PAIR) bar_wait_cluster(tfull0 + 8 * abuf, (aph >> abuf) & 1u);  // the leader's multicast commit
            else bar_wait(tfull0 + 8 * abuf, (aph >> abuf) & 1u);
            tc_fence_after();
        };
        const uint32_t lead_tempty0 = PAIR ? cluster_addr(tempty0, 0) : tempty0;
        auto release = [&]() {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (PAIR) bar_arrive_remote(lead_tempty0 + 8 * abuf);  // the leader issues the next MMAs
                else bar_arrive(tempty0 + 8 * abuf);
            }
            aph ^= 1u << abuf;
            abuf ^= 1;
        };
        for (int smp = 0; smp < my_samples; ++smp) {
            float ssq = 0.f;
            // split sample (one sample per launch): the partial Y of earlier K-segments
            float4* yp = SPLIT ? reinterpret_cast<float4*>(ypart + (int64_t)((kpar ? grp * sh.T : 0) + tile) * (TBM * TBN) +
                                                           (int64_t)row * TBN + h * HC)
                               : nullptr;
            if (segmented && nseg > 1) {
                // all but the last segment: R = Y so far (round-to-nearest adds)
                wait_full();
#pragma unroll
                for (int ch = 0; ch < HC / 16; ++ch) {
                    float y[16];
                    load(abuf, ch, y);
#pragma unroll
                    for (int i = 0; i < 16; ++i) R[ch * 16 + i] = y[i];
                }
                release();
                for (int sg = 1; sg + 1 < nseg; ++sg) {
                    wait_full();
#pragma unroll
                    for (int ch = 0; ch < HC / 16; ++ch) {
                        float y[16];
                        load(abuf, ch, y);
#pragma unroll
                        for (int i = 0; i < 16; ++i) R[ch * 16 + i] = __fadd_rn(R[ch * 16 + i], y[i]);
                    }
                    release();
                }
            }
            wait_full();  // the sample's last (or only) segment
#pragma unroll
            for (int ch = 0; ch < HC / 16; ++ch) {
                float y[16];
                load(abuf, ch, y);
                if (segmented && nseg > 1) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) y[i] = __fadd_rn(R[ch * 16 + i], y[i]);
                }
                if (SPLIT && split_part >= 2) {  // middle / last launch: add the carried partial
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const float4 pv = yp[ch * 4 + v];
                        y[4 * v] = __fadd_rn(pv.x, y[4 * v]);
                        y[4 * v + 1] = __fadd_rn(pv.y, y[4 * v + 1]);
                        y[4 * v + 2] = __fadd_rn(pv.z, y[4 * v + 2]);
                        y[4 * v + 3] = __fadd_rn(pv.w, y[4 * v + 3]);
                    }
                }
                if (SPLIT && split_part <= 2) {  // not the last launch: carry Y on
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        yp[ch * 4 + v] = make_float4(y[4 * v], y[4 * v + 1], y[4 * v + 2], y[4 * v + 3]);
                    continue;
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    ssq = __fmaf_rn(y[i], y[i], ssq);
#ifndef MLSK_TC_ABL_NOSUM  // ablation (timing only, wrong sums): no register running sum
                    // one segment: R = running sum S; several: R = this sample's Y
                    R[ch * 16 + i] = segmented ? y[i] : __fadd_rn(R[ch * 16 + i], y[i]);
#endif
                }
            }
            release();
            sq += (double)ssq;
#ifdef MLSK_TC_ABL_NOSUM
            if (false) {
#else
            if (!(SPLIT && split_part <= 2) && (segmented || (smp + 1) % FLUSH == 0 || smp + 1 == my_samples)) {
#endif
                if (segmented && !sh.direct) {
                    // the sample's Y into this CTA's fp32 partial tile by
                    // reductions in L2: a load-add-store of an fp64 partial per
                    // sample stalled the operand stream (config 3, c = 1024:
                    // tensor pipe 95% -> 78% active, 300 MB of extra DRAM writes)
#pragma unroll
                    for (int i = 0; i < HC; ++i) red_add_f32(outf + i * TBM, R[i]);
                } else if (sh.direct) {
                    // (tile-aligned outputs, one CTA per tile, one sample per
                    // CTA) this thread's 64 consecutive columns of the row-major
                    // level total, by reductions in L2: a load-add-store here
                    // sat in the CTA's tail (config 5, c = 2048: 1.39 ms vs
                    // 1.14 at the same flops with the reductions)
                    double* o = sh.direct + ((int64_t)tm * TBM + row) * sh.cols + (int64_t)tn * TBN + h * HC;
#pragma unroll
                    for (int i = 0; i < HC; ++i) {
                        red_add_f64(o + i, (double)R[i]);
                        R[i] = 0.f;
                    }
                } else {
                    // the running sum into this CTA's fp64 partial tile by
                    // reductions in L2 (no load round trip in the CTA's tail)
#pragma unroll
                    for (int i = 0; i < HC; ++i) {
                        red_add_f64(out + i * TBM, (double)R[i]);
                        R[i] = 0.f;
                    }
                }
            }
        }
        sq = warp_sum(sq);
        if (lane == 0) s_sq[ew] = sq;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) bar_arrive(tdone);
        // the CTA's ||Y||^2: named barrier over the epilogue warps only
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
        if (ew == 0 && lane == 0 && !kpar) {  // kpar: the squares come from k_kpar_combine
            double t = 0.0;
            for (int w = 0; w < EPI_WARPS; ++w) t += s_sq[w];
            part_sq[g] = sh.sym_nb && (tm >> 1) != tn ? 2.0 * t : t;  // a mirrored block counts twice
        }
    }
}

// level total (row-major rows x cols) += sum over the Gs group partials of
// each tile (column-major [col][row] per CTA); 32 x 32 cell blocks through
// shared memory so both the partial reads and the total updates coalesce.
// Block (32, 8); grid covers the cell blocks (grid-stride).
__global__ void __launch_bounds__(256) k_reduce_tiles_tc(const double* __restrict__ part,
                                                         const double* __restrict__ part_sq, TcShape sh,
                                                         int64_t rows, int64_t cols, double* __restrict__ total,
                                                         double* __restrict__ total_sq, int f32part) {
    const float* partf = reinterpret_cast<const float*>(part);  // segmented launches: fp32 partials
    __shared__ double blk[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t brows = (rows + 31) / 32, bcols = (cols + 31) / 32;
    for (int64_t bi = blockIdx.x; bi < brows * bcols; bi += gridDim.x) {
        const int64_t r0 = (bi / bcols) * 32, q0 = (bi % bcols) * 32;
        // read: lane = row (contiguous in the column-major partial)
        for (int k = ty; k < 32; k += 8) {
            const int64_t r = r0 + tx, q = q0 + k;
            double acc = 0.0;
            const int tile = r < rows && q < cols ? tile_index(sh, (int)(r / TBM), (int)(q / TBN)) : -1;
            if (tile >= 0) {  // (cells of the lower blocks of a symmetric output: filled by the mirror)
                const int64_t off = (q % TBN) * TBM + (r % TBM);
                for (int grp = 0; grp < sh.Gs; ++grp) {
                    const int64_t e = (int64_t)(grp * sh.T + tile) * (TBM * TBN) + off;
                    acc += f32part ? (double)partf[e] : part[e];
                }
            }
            blk[tx][k] = acc;
        }
        __syncthreads();
        // write: lane = column (contiguous in the row-major total)
        for (int k = ty; k < 32; k += 8) {
            const int64_t r = r0 + k, q = q0 + tx;
            if (r < rows && q < cols) total[r * cols + q] += blk[k][tx];
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && ty == 0) {
        const double acc = warp_sum_array(part_sq, sh.T * sh.Gs, tx);
        if (tx == 0) *total_sq += acc;
    }
}

// kpar: Y = Y_0 + Y_1 (fp32, as a carried K-segment), level total += Y,
// per-block sum of Y^2 in fp64 into blk_sq (then summed by one warp)
__global__ void __launch_bounds__(256) k_kpar_combine(const float* __restrict__ yp, TcShape sh, int64_t rows,
                                                      int64_t cols, double* __restrict__ total,
                                                      double* __restrict__ blk_sq) {
    const int T = sh.T;
    __shared__ double s_red[8];
    double sq = 0.0;
    const int64_t cells = rows * cols;
    for (int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cell < cells;
         cell += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = cell / cols, q = cell - r * cols;
        const int tile = tile_index(sh, (int)(r / TBM), (int)(q / TBN));
        const int64_t off = (int64_t)tile * (TBM * TBN) + (r % TBM) * TBN + (q % TBN);
        const float y = __fadd_rn(yp[off], yp[(int64_t)T * (TBM * TBN) + off]);
        total[cell] += (double)y;
        sq = __fma_rn((double)y, (double)y, sq);
    }
    sq = warp_sum(sq);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x < 32) {
        const double v = warp_sum(threadIdx.x < 8 ? s_red[threadIdx.x] : 0.0);
        if (threadIdx.x == 0) blk_sq[blockIdx.x] = v;
    }
}

// symmetric output: total[r][q] = total[q][r] for every r > q (n % 256 == 0):
// the 256 x 256 blocks below the diagonal were not computed, and inside the
// diagonal blocks (computed in full) the copy makes the estimate exactly
// symmetric.  32 x 32 cell blocks through shared memory, both sides
// coalesced.  Block (32, 8).
__global__ void __launch_bounds__(256) k_mirror_lower(double* __restrict__ total, int64_t n) {
    __shared__ double blk[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t nb = n / 32;
    for (int64_t bi = blockIdx.x; bi < nb * nb; bi += gridDim.x) {
        const int64_t r0 = (bi / nb) * 32, q0 = (bi % nb) * 32;
        if (r0 < q0) continue;  // above the diagonal (uniform per CTA)
        for (int k = ty; k < 32; k += 8) blk[k][tx] = total[(q0 + k) * n + r0 + tx];
        __syncthreads();
        for (int k = ty; k < 32; k += 8)
            if (r0 > q0 || k > tx) total[(r0 + k) * n + q0 + tx] = blk[tx][k];
        __syncthreads();
    }
}

__global__ void k_sum_sq(const double* __restrict__ blk_sq, int n, double* __restrict__ total_sq) {
    const double v = warp_sum_array(blk_sq, n, threadIdx.x);
    if (threadIdx.x == 0) *total_sq += v;
}

int sms() {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

}  // namespace

bool tc_supported(const Model& M, int target) {
    return target == MLSK_TARGET_IDENTITY && M.dm.stream == MLSK_STREAM_PHILOX && !M.vector &&
           M.dm.dtype == MLSK_F32 &&
           (M.dm.kind == MLSK_MODEL_GAUSS_MEAN || M.dm.kind == MLSK_MODEL_STUDENT_T || M.dm.kind == MLSK_MODEL_RFF);
}

namespace {

class TcEngine final : public PanelEngine {
   public:
    TcEngine(const Model& M, Workspace& ws) : M_(M), ws_(ws) {
        nsm_ = sms();
        MP_ = (M.rows + TBM - 1) / TBM * TBM;
        PP_ = (M.cols + TBN - 1) / TBN * TBN;
        tiles_n_ = (int)(PP_ / TBN);
        T_ = (int)(MP_ / TBM) * tiles_n_;
        // RFF Gram (Y symmetric): upper-triangle blocks only (MLSK_TC_SYM=0: full grid)
        const char* sym_env = std::getenv("MLSK_TC_SYM");
        if (M.dm.kind == MLSK_MODEL_RFF && M.rows == M.cols && M.rows % TBN == 0 &&
            !(sym_env && std::strcmp(sym_env, "0") == 0)) {
            sym_nb_ = (int)(M.rows / TBN);
            T_ = sym_nb_ * (sym_nb_ + 1);  // nb (nb + 1) / 2 blocks of two tiles
        }
        const char* sh_env = std::getenv("MLSK_TC_SHARED");
        shared_env_ = !(sh_env && std::strcmp(sh_env, "0") == 0);
        Gs_ = std::max(1, nsm_ / T_);
        // TMEM accumulation segment (K-chunks): samples longer than one segment
        // sum their segments in registers (TcShape::seg).  MLSK_TC_SEG overrides
        // (0: never segment -- accuracy experiments only)
        const char* seg_env = std::getenv("MLSK_TC_SEG");
        seg_ = seg_env ? std::max(0, atoi(seg_env)) : TC_SEG;
        S_.M = M.dm;
        smem_ = std::max(TSTAGES * TSTAGE_BYTES, PSTAGES * PSTAGE_BYTES) + 1024;
        ws_.partial.ensure((size_t)T_ * Gs_ * (TBM * TBN) + (size_t)T_ * Gs_);
        // generator grid cap (CTAs; grid-stride beyond it).  MLSK_TC_GEN_CTAS_PER_SM
        // (experiments): 0 = one work item per CTA
        gen_cap_ = (int64_t)nsm_ * 8;
        rff_smem_ = RFF_SMEM;
        const int smem = smem_, rsmem = rff_smem_;
        // CTA pairs (cta_group::2) when the tile rows pair up (an even number of
        // 128-row tiles; the rasterised / symmetric tile orders then put the two
        // tiles of a pair at indices 2u, 2u + 1).  MLSK_TC_PAIR=0: single CTAs.
        const char* pair_env = std::getenv("MLSK_TC_PAIR");
        pair_ = (MP_ / TBM) % 2 == 0 && T_ % 2 == 0 && !(pair_env && std::strcmp(pair_env, "0") == 0);
        // BF16 cross terms.  MLSK_TC_BF16X=0: three TF32 MMAs per K-step
        const char* bfx_env = std::getenv("MLSK_TC_BF16X");
        bfx_ = !(bfx_env && std::strcmp(bfx_env, "0") == 0) ? 1 : 0;
        // FP16 pairs for models with bounded entries (fp32 Gaussian draws, random
        // Fourier features with the fast generator).  MLSK_TC_H16=0: BF16 cross terms
        const char* h16_env = std::getenv("MLSK_TC_H16");
        const bool bounded = M.dm.kind == MLSK_MODEL_GAUSS_MEAN ||
                             (M.dm.kind == MLSK_MODEL_RFF && M.dm.rff_dim <= RFF_DMAX);
        if (bfx_ && !(h16_env && std::strcmp(h16_env, "0") == 0)) bfx_ = bounded ? 2 : 3;
        // panel scale (a power of two): RFF features are ~ sqrt(2 / n); scaled to [1, 2)
        // so that the lo halves stay normal fp16 numbers
        pscale_ = 1.0f;
        if (bfx_ == 2 && M.dm.kind == MLSK_MODEL_RFF && M.dm.rff_scale > 0) {
            int e = 0;
            std::frexp(M.dm.rff_scale, &e);  // rff_scale = f 2^e, f in [0.5, 1)
            pscale_ = std::ldexp(1.0f, 1 - e);
        }
        once_per_device((const void*)&k_gemm_tf32x3<false, false, false>, [smem, rsmem] {
            for (auto f : {k_gemm_tf32x3<false, false, false>, k_gemm_tf32x3<false, true, false>,
                           k_gemm_tf32x3<true, false, false>, k_gemm_tf32x3<true, true, false>,
                           k_gemm_tf32x3<false, false, true>, k_gemm_tf32x3<false, true, true>,
                           k_gemm_tf32x3<true, false, true>, k_gemm_tf32x3<true, true, true>}) {
                MLSK_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                MLSK_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                // setmaxnreg redistributes the launch's registers: the launch must
                // hold what the warps ask for (else the epilogue's inc never returns)
                cudaFuncAttributes fa{};
                MLSK_CUDA(cudaFuncGetAttributes(&fa, f));
                if (fa.numRegs * TC_THREADS < 32 * (CTRL_WARPS * CTRL_REGS + EPI_WARPS * EPI_REGS))
                    throw Error(MLSK_ERUNTIME, "tcgen05 GEMM built with " + std::to_string(fa.numRegs) +
                                                  " registers per thread: too few for its setmaxnreg split");
            }
            MLSK_CUDA(cudaFuncSetAttribute(k_gen_panels_rff, cudaFuncAttributeMaxDynamicSharedMemorySize, rsmem));
            // full shared-memory carveout for every kernel of the pipeline, so a
            // generator CTA never leaves an SM configured too small for a GEMM CTA
            MLSK_CUDA(cudaFuncSetAttribute(k_gen_panels_tf32<GK_GAUSS>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            MLSK_CUDA(cudaFuncSetAttribute(k_gen_panels_tf32<GK_STUDENT_T>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            MLSK_CUDA(cudaFuncSetAttribute(k_gen_panels_tf32<GK_GENERIC>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        });
    }
    // FP16 hi + BF16 (bfx_ == 3): entries of A times 2^-6, weights of B times 2^-6 / 2^floor(log2 |w_fine|)
    float a_scale() const { return bfx_ == 3 ? 0.015625f : 1.0f; }
    float w_scale(double w_fine) const {
        if (bfx_ != 3 || !(std::fabs(w_fine) > 0)) return 1.0f;
        int e = 0;
        std::frexp(std::fabs(w_fine), &e);  // |w_fine| = f 2^e, f in [0.5, 1)
        return std::ldexp(0.015625f, 1 - e);
    }
    int64_t chunk_cols() const override { return TBK; }
    // merged sampled columns: on the shared RFF panel the columns carry the scale
    // sqrt(|W_j| / |w|) in sign groups (mode 2); otherwise the summed weights
    // fold into B (mode 1)
    int merge_mode(int64_t c, int64_t cc, double w_fine, double w_coarse) const override {
        return shared_panel(c, cc, w_fine, w_coarse) ? 2 : 1;
    }
    // hi + lo: 8 bytes per entry (FP16 pairs: 4, FP16 hi + BF16: 6)
    int64_t chunk_bytes() const override { return (MP_ + PP_) * TBK * (bfx_ == 2 ? 4 : bfx_ == 3 ? 6 : 8); }
    bool splits_k() const override { return true; }
    int64_t group_size() const override { return Gs_; }
    void gen(cudaStream_t s, uint64_t seed, uint64_t tag, const int64_t* ks, int nb, int64_t c, int64_t cc,
             double w_fine, double w_coarse, void* panels, uint32_t* idx, const KRange& kr) override {
        const int64_t k = kr.nkc >= 0 ? kr.nkc : nkc(c);
        float *Ahi, *Alo, *Bhi, *Blo;
        split(panels, nb, k, Ahi, Alo, Bhi, Blo);
        Prof p("gen_panels_tf32", s);
        if (M_.dm.kind == MLSK_MODEL_RFF && M_.dm.rff_dim <= RFF_DMAX) {
            k_gen_panels_rff<<<(int)std::min<int64_t>((int64_t)nb * ((k + RFF_CH - 1) / RFF_CH) * RFF_RSPLIT,
                                                      (int64_t)nsm_ * 5),
                               RFF_T, rff_smem_, s>>>(
                S_, seed, tag, ks, nb, c, cc, (float)w_fine, (float)w_coarse, MP_, PP_, k, kr.kc0,
                shared_panel(c, cc, w_fine, w_coarse) ? 0 : 1, Ahi, Alo, Bhi, Blo, idx, kr.mk, kr.mk_stride, kr.mk_info, bfx_, pscale_);
        } else {
            const int grid = (int)std::min<int64_t>((int64_t)nb * k, gen_cap_);
            if (M_.dm.kind == MLSK_MODEL_GAUSS_MEAN)
                k_gen_panels_tf32<GK_GAUSS><<<grid, GEN_T, 0, s>>>(S_, seed, tag, ks, nb, c, cc, (float)w_fine,
                                                                  (float)w_coarse, MP_, PP_, k, kr.kc0, Ahi, Alo, Bhi,
                                                                  Blo, idx, kr.mk, kr.mk_stride, kr.mk_info, bfx_, a_scale(), w_scale(w_fine));
            else if (M_.dm.kind == MLSK_MODEL_STUDENT_T)
                k_gen_panels_tf32<GK_STUDENT_T><<<grid, GEN_T, 0, s>>>(S_, seed, tag, ks, nb, c, cc, (float)w_fine,
                                                                      (float)w_coarse, MP_, PP_, k, kr.kc0, Ahi, Alo,
                                                                      Bhi, Blo, idx, kr.mk, kr.mk_stride, kr.mk_info, bfx_, a_scale(), w_scale(w_fine));
            else
                k_gen_panels_tf32<GK_GENERIC><<<grid, GEN_T, 0, s>>>(S_, seed, tag, ks, nb, c, cc, (float)w_fine,
                                                                    (float)w_coarse, MP_, PP_, k, kr.kc0, Ahi, Alo, Bhi,
                                                                    Blo, idx, kr.mk, kr.mk_stride, kr.mk_info, bfx_, a_scale(), w_scale(w_fine));
        }
        launched();
    }
    void gemm(cudaStream_t s, const void* panels, int nb, int64_t c, int64_t cc, double w_fine, double w_coarse,
              LevelState& st, const KRange& kr) override {
        const int64_t k = kr.nkc >= 0 ? kr.nkc : nkc(c);
        float *Ahi, *Alo, *Bhi, *Blo;
        split(const_cast<void*>(panels), nb, k, Ahi, Alo, Bhi, Blo);
        int64_t neg_kc = 0;
        float escale = 1.0f;
        if (shared_panel(c, cc, w_fine, w_coarse)) {  // B tiles from the A panel (MP == PP)
            Bhi = Ahi;
            Blo = Alo;
            neg_kc = w_coarse < 0 ? cc / TBK : 0;
            escale = (float)std::fabs(w_fine);
        }
        escale *= 1.0f / (pscale_ * pscale_);  // FP16 pairs: both operands carry the panel scale
        escale *= 1.0f / (a_scale() * w_scale(w_fine));  // FP16 hi + BF16: the A / weight scales (powers of two)
        // merged sampled columns: sign groups only on the shared panel (mode 2)
        const MkInfo* mk_info = kr.mk && shared_panel(c, cc, w_fine, w_coarse) ? kr.mk_info : nullptr;
        double* part = ws_.partial.p;
        double* part_sq = part + (size_t)T_ * Gs_ * (TBM * TBN);
        const bool finishes = kr.part == 0 || kr.part == 3;  // samples complete in this launch
        // one CTA per tile and a tile-aligned output: sums straight into the level total
        // Only a launch of one sample per CTA writes the level total directly: with
        // several, the CTA partials (flushed by reductions) and one reduction pass
        // are faster (config 5, c = 256, 8 samples per CTA: 1.41 -> 1.14 ms) --
        // the direct flush is a load-add-store of 256 KB in each CTA's tail.
        const bool direct = Gs_ == 1 && M_.rows % TBM == 0 && M_.cols % TBN == 0 && nb == 1;
        // one sample whose tiles fill the last CTA wave poorly (config 4: 512
        // tiles = 3.5 waves): split its K range over two CTA groups, 7 waves of
        // half the work, and combine the two partial Y afterwards
        const int64_t w1 = (T_ + nsm_ - 1) / nsm_, w2 = (2 * T_ + nsm_ - 1) / nsm_;
        if (kr.part == 0 && nb == 1 && direct && w2 < 2 * w1 && k >= 16 && !sym_nb_) {
            ws_.ypart.ensure((size_t)2 * T_ * TBM * TBN);
            TcShape sh{1, k, MP_, PP_, T_, 2, tiles_n_, nullptr, M_.rows, M_.cols, 1, 0, 0, 0, escale, nullptr, bfx_, seg_};
            {
                Prof p("gemm_tf32x3", s);
                launch_gemm(true, segmented(k - (k + 1) / 2), 2 * T_, s, Ahi, Alo, Bhi, Blo, sh, part, part_sq, 1,
                            ws_.ypart.p);
            }
            {
                Prof p("reduce_tiles_tc", s);
                const int blocks = nsm_ * 4;  // blk_sq scratch: the (unused) partial buffer
                k_kpar_combine<<<blocks, 256, 0, s>>>(ws_.ypart.p, sh, M_.rows, M_.cols, st.total(), part);
                k_sum_sq<<<1, 32, 0, s>>>(part, blocks, st.total_sq());
            }
            launched(3);
            return;
        }
        if (finishes && !direct)  // (segmented launches: the fp32 partials, half the bytes)
            MLSK_CUDA(cudaMemsetAsync(part, 0, (segmented(k) ? sizeof(float) : sizeof(double)) * (size_t)T_ * Gs_ *
                                                   (TBM * TBN), s));
        float* ypart = nullptr;
        if (kr.part != 0) {
            ws_.ypart.ensure((size_t)T_ * TBM * TBN);  // the carried partial Y of a split sample
            ypart = ws_.ypart.p;
        }
        TcShape sh{nb,      k,       MP_,     PP_,    T_,     Gs_,        tiles_n_, direct ? st.total() : nullptr,
                   M_.rows, M_.cols, 0,       sym_nb_, neg_kc, kr.kc0, escale, mk_info, bfx_, seg_};
        {
            Prof p("gemm_tf32x3", s);
            if (kr.part == 0)
                launch_gemm(false, segmented(k), T_ * Gs_, s, Ahi, Alo, Bhi, Blo, sh, part, part_sq, 0, nullptr);
            else
                launch_gemm(true, segmented(k), T_ * Gs_, s, Ahi, Alo, Bhi, Blo, sh, part, part_sq, kr.part, ypart);
        }
        if (!finishes) {
            launched();
            return;
        }
        {
            Prof p("reduce_tiles_tc", s);
            const int64_t cells = M_.rows * M_.cols;
            // direct mode: only the squares are left to add (cells = 0)
            k_reduce_tiles_tc<<<direct ? 1 : (int)std::min<int64_t>((cells + 1023) / 1024, (int64_t)nsm_ * 8),
                                dim3(32, 8), 0, s>>>(part, part_sq, sh, direct ? 0 : M_.rows, M_.cols, st.total(),
                                                     st.total_sq(), segmented(k) ? 1 : 0);
        }
        launched(2);
        // symmetric output: the lower blocks are copied from the upper ones once
        // per level and pass (KRange::finish), after the level's last reduction
        // (a per-batch reduction stream with double-buffered partials was measured
        // too: config 3 14.4 -> 15.3 ms -- the generator fills the SMs during the
        // reductions, so taking them off the GEMM stream only starves it)
        if (sym_nb_ && kr.finish) {
            Prof p("mirror_tc", s);
            const int64_t n = M_.rows;
            k_mirror_lower<<<(int)std::min<int64_t>((n / 32) * (n / 32), (int64_t)nsm_ * 8), dim3(32, 8), 0, s>>>(
                st.total(), n);
            launched();
        }
    }

   private:
    using GemmFn = void (*)(const float*, const float*, const float*, const float*, TcShape, double*, double*, int,
                            float*);
    // the GEMM instantiation for (split, segmented, pair); pair launches as
    // clusters of two CTAs
    void launch_gemm(bool split, bool segm, int grid, cudaStream_t s, const float* Ahi, const float* Alo,
                     const float* Bhi, const float* Blo, const TcShape& sh, double* part, double* part_sq, int split_part,
                     float* ypart) const {
        static const GemmFn fns[8] = {k_gemm_tf32x3<false, false, false>, k_gemm_tf32x3<false, true, false>,
                                      k_gemm_tf32x3<true, false, false>,  k_gemm_tf32x3<true, true, false>,
                                      k_gemm_tf32x3<false, false, true>,  k_gemm_tf32x3<false, true, true>,
                                      k_gemm_tf32x3<true, false, true>,   k_gemm_tf32x3<true, true, true>};
        const GemmFn f = fns[(pair_ ? 4 : 0) + (split ? 2 : 0) + (segm ? 1 : 0)];
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(TC_THREADS);
        cfg.dynamicSmemBytes = (size_t)smem_;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = pair_ ? 2 : 1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        MLSK_CUDA(cudaLaunchKernelEx(&cfg, f, Ahi, Alo, Bhi, Blo, sh, part, part_sq, split_part, ypart));
    }
    static int64_t nkc(int64_t c) { return (c + TBK - 1) / TBK; }
    // a CTA K-range of `k` chunks (at least) runs as several TMEM segments
    bool segmented(int64_t k) const { return seg_ > 0 && k > seg_; }
    // RFF Gram with the fast generator: the B panel is diag(w) A^T.  When every
    // |w| is the same power of two and the coarse prefix is whole K-chunks, the
    // GEMM reads B from the A panel (negated prefix chunks, Y scaled by |w|):
    // the products and their fp32 sums are the same bits scaled by |w|, and
    // the generator writes half the panel bytes.  MLSK_TC_SHARED=0 disables.
    bool shared_panel(int64_t c, int64_t cc, double w_fine, double w_coarse) const {
        if (!sym_nb_ || M_.dm.rff_dim > RFF_DMAX || cc % TBK != 0 || c <= 0) return false;
        if (cc > 0 && std::fabs(w_coarse) != std::fabs(w_fine)) return false;
        int e = 0;
        if (std::frexp(std::fabs(w_fine), &e) != 0.5 || e < -100 || e > 100) return false;
        return shared_env_;
    }
    // panels of nb samples x k K-chunks: A hi, A lo, B hi, B lo
    void split(void* panels, int nb, int64_t k, float*& Ahi, float*& Alo, float*& Bhi, float*& Blo) const {
        const size_t na = (size_t)nb * k * MP_ * TBK, nbp = (size_t)nb * k * PP_ * TBK;
        Ahi = static_cast<float*>(panels);
        if (bfx_ == 2) {  // FP16 pairs: one array per operand (64-byte rows, like a hi array)
            Alo = nullptr;
            Bhi = Ahi + na;
            Blo = nullptr;
            return;
        }
        Alo = Ahi + na;
        if (bfx_ == 3) {  // the lo arrays hold 32-byte rows: half the floats
            Bhi = Alo + na / 2;
            Blo = Bhi + nbp;
            return;
        }
        Bhi = Alo + na;
        Blo = Bhi + nbp;
    }
    const Model& M_;
    Workspace& ws_;
    TcModel S_{};
    int nsm_, T_, Gs_, tiles_n_, smem_, rff_smem_;
    int sym_nb_ = 0;  // symmetric output: 256-blocks per side (0 = full tile grid)
    bool pair_ = false;  // CTA-pair GEMM (cta_group::2)
    int bfx_ = 0;        // 1: BF16 cross terms; 2: FP16 pairs (one tile per operand); 3: FP16 hi + BF16 cross terms
    float pscale_ = 1.0f;  // FP16 pairs: power-of-two scale of the generated entries (undone in the epilogue)
    int seg_ = TC_SEG;
    bool shared_env_ = true;
    int64_t gen_cap_;
    int64_t MP_, PP_;
};

}  // namespace

std::unique_ptr<PanelEngine> make_tc_engine(const Model& M, Workspace& ws) {
    return std::unique_ptr<PanelEngine>(new TcEngine(M, ws));
}

}  // namespace mlsk
