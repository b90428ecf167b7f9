// mlsk_exact.cu -- the exact-order engine.
//
// Reproduces the reference's arithmetic order on the device, so that given
// bit-identical draws the per-level sums are bit-identical to
// estimators.cpp:128-169:
//   * reference stream: each replication's mt19937_64 substream
//     (rng.hpp:19,39-41) is materialised by one warp (parallel twist of the
//     312-word state in shared memory), then the model draw and the index
//     draws read their positions in it (estimators.cpp:134-136);
//   * philox stream: entries and indices come straight from the counters;
//   * sketch: o += (a_ij * inv_j) * b_jk in index order, scaled by 1/s
//     (sketch.cpp:60-75); the coarse sketch is the same running sum read
//     after the first c/M indices (identical operands and order to the
//     reference's second pass over the prefix span);
//   * reduction: 64-replication chunks, s[t] += v in replication order,
//     s2 serial in (k, t) order, chunk partials summed in chunk order.
// Used for the parity configurations, nonlinear targets and the reference
// stream; the throughput path is mlsk_fused.cu.
#include <algorithm>
#include <cstring>

#include "mlsk_internal.h"

namespace mlsk {

namespace {

constexpr uint64_t MT_UPPER = 0xFFFFFFFF80000000ULL;
constexpr uint64_t MT_LOWER = 0x000000007FFFFFFFULL;
constexpr uint64_t MT_A = 0xB5026F5AA96619E9ULL;

__device__ __forceinline__ uint64_t mt_temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    return z ^ (z >> 43);
}

// In-place mt19937_64 twist by one warp; same result as the sequential loop
// of libstdc++'s _M_gen_rand (three dependency phases).
__device__ void mt_twist_warp(uint64_t* mt, int lane) {
    for (int base = 0; base < 156; base += 32) {
        const int k = base + lane;
        uint64_t nv = 0;
        if (k < 156) {
            const uint64_t y = (mt[k] & MT_UPPER) | (mt[k + 1] & MT_LOWER);
            nv = mt[k + 156] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
        }
        __syncwarp();
        if (k < 156) mt[k] = nv;
        __syncwarp();
    }
    for (int base = 156; base < 311; base += 32) {
        const int k = base + lane;
        uint64_t nv = 0;
        if (k < 311) {
            const uint64_t y = (mt[k] & MT_UPPER) | (mt[k + 1] & MT_LOWER);
            nv = mt[k - 156] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
        }
        __syncwarp();
        if (k < 311) mt[k] = nv;
        __syncwarp();
    }
    if (lane == 0) {
        const uint64_t y = (mt[311] & MT_UPPER) | (mt[0] & MT_LOWER);
        mt[311] = mt[155] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
    }
    __syncwarp();
}

constexpr int STREAM_WARPS = 4;

// One warp per replication: out[b][0..len) = first len outputs of
// std::mt19937_64(derive_seed(seed, tag, ks[b])).
__global__ void __launch_bounds__(32 * STREAM_WARPS)
k_ref_stream(uint64_t seed, uint64_t tag, const int64_t* __restrict__ ks, int nb, int64_t len,
             uint64_t* __restrict__ out) {
    __shared__ uint64_t state[STREAM_WARPS][312];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * STREAM_WARPS + w;
    if (b >= nb) return;
    uint64_t* mt = state[w];
    if (lane == 0) {
        uint64_t x = derive_seed(seed, tag, (uint64_t)ks[b]);
        mt[0] = x;
        for (int i = 1; i < 312; ++i) {
            x = 6364136223846793005ULL * (x ^ (x >> 62)) + (uint64_t)i;
            mt[i] = x;
        }
    }
    __syncwarp();
    uint64_t* o = out + (int64_t)b * len;
    for (int64_t pos = 0; pos < len; pos += 312) {
        mt_twist_warp(mt, lane);
        const int64_t n = min((int64_t)312, len - pos);
        for (int i = lane; i < n; i += 32) o[pos + i] = mt_temper(mt[i]);
        __syncwarp();
    }
}

// Index draws: idx[b][t] (1-based), from the stream (ref) or the counters.
__global__ void k_indices(DevModel M, uint64_t seed, uint64_t tag, const int64_t* __restrict__ ks, int nb,
                          int64_t c, const uint64_t* __restrict__ stream, int64_t stream_len, int64_t ref_off,
                          uint32_t* __restrict__ idx) {
    const int64_t total = (int64_t)nb * c;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / c, t = e - b * c;
        uint64_t x;
        if (M.stream == MLSK_STREAM_REF) {
            x = stream[b * stream_len + ref_off + t];
        } else {
            const uint64_t key = derive_seed(seed, tag, (uint64_t)ks[b]);
            const u32x4 r = philox((uint32_t)(t >> 1), 0, 0, MLSK_CTR_INDEX, key);
            x = (t & 1) ? hi64(r) : lo64(r);
        }
        idx[e] = index_from_u64(x, M.n, M.log2n, M.cum);
    }
}

// Reference-value draws use every column in order (no index stream).
__global__ void k_iota(int nb, int64_t c, uint32_t* __restrict__ idx) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)nb * c;
         e += (int64_t)gridDim.x * blockDim.x)
        idx[e] = (uint32_t)(e % c) + 1u;
}

// Gather of the sampled columns of A (a_cols[b][r][t]) and rows of B
// (b_rows[b][t][q]) -- the model draw restricted to the sampled indices.
__global__ void k_gather(DevModel M, uint64_t seed, uint64_t tag, const int64_t* __restrict__ ks, int nb,
                         int64_t c, const uint64_t* __restrict__ stream, int64_t stream_len,
                         const uint32_t* __restrict__ idx, double* __restrict__ a_cols,
                         double* __restrict__ b_rows) {
    const int64_t na = (int64_t)nb * M.rows * c, nbb = (int64_t)nb * c * M.cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < na + nbb;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (e < na) {
            const int64_t b = e / (M.rows * c);
            const int64_t rem = e - b * M.rows * c;
            const int64_t r = rem / c, t = rem - r * c;
            const int64_t j = (int64_t)idx[b * c + t] - 1;
            double v;
            if (M.stream == MLSK_STREAM_REF) v = ref_a(M, stream + b * stream_len, j, r);
            else v = philox_a(M, derive_seed(seed, tag, (uint64_t)ks[b]), j, r);
            a_cols[e] = v;
        } else {
            const int64_t f = e - na;
            const int64_t b = f / (c * M.cols);
            const int64_t rem = f - b * c * M.cols;
            const int64_t t = rem / M.cols, q = rem - t * M.cols;
            const int64_t j = (int64_t)idx[b * c + t] - 1;
            double v;
            if (M.stream == MLSK_STREAM_REF) v = ref_b(M, stream + b * stream_len, j, q);
            else v = philox_b(M, derive_seed(seed, tag, (uint64_t)ks[b]), j, q);
            b_rows[f] = v;
        }
    }
}

// v[b][cell] = f(fine) - f(coarse) in the reference's operation order.
__global__ void k_sketch(int vector, int64_t rows, int64_t cols, int nb, int64_t c, int64_t cc, double w,
                         double vdiv, double sf, double sc, int target, double tparam,
                         const double* __restrict__ a_cols, const double* __restrict__ b_rows,
                         double* __restrict__ v) {
    const int64_t cells = rows * cols, total = (int64_t)nb * cells;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / cells, cell = e - b * cells;
        double fine, coarse = 0.0;
        if (vector) {  // sketch.cpp:32-37
            const double* a = a_cols + b * c;
            const double* bb = b_rows + b * c;
            double sum = 0.0, pre = 0.0;
            for (int64_t t = 0; t < c; ++t) {
                sum = __dadd_rn(sum, __dmul_rn(__dmul_rn(a[t], bb[t]), w));
                if (t + 1 == cc) pre = sum;
            }
            fine = __ddiv_rn(sum, vdiv);
            if (cc > 0) coarse = __ddiv_rn(pre, (double)cc);
        } else {  // sketch.cpp:60-75
            const int64_t r = cell / cols, q = cell - r * cols;
            const double* a = a_cols + (b * rows + r) * c;
            const double* bb = b_rows + b * c * cols + q;
            double o = 0.0, pre = 0.0;
            for (int64_t t = 0; t < c; ++t) {
                o = __dadd_rn(o, __dmul_rn(__dmul_rn(a[t], w), bb[t * cols]));
                if (t + 1 == cc) pre = o;
            }
            fine = __dmul_rn(o, sf);
            if (cc > 0) coarse = __dmul_rn(pre, sc);
        }
        double x = apply_target(target, tparam, fine);
        if (cc > 0) x = __dadd_rn(x, -apply_target(target, tparam, coarse));
        v[e] = x;
    }
}

// Segment partials: s[cell] (replication order) and s2 serial in (k, cell)
// order, optionally continuing the level's open chunk.  One block per segment.
// seg_desc[s] = {first batch row, count, resumes}
constexpr int RED_THREADS = 256;
constexpr int RED_TILE = 2048;

__global__ void __launch_bounds__(RED_THREADS)
k_segments(const double* __restrict__ v, int64_t cells, const int64_t* __restrict__ seg_desc,
           const double* __restrict__ open, const double* __restrict__ open_sq, double* __restrict__ part) {
    __shared__ double tile[RED_TILE];
    const int s = blockIdx.x;
    const int64_t first = seg_desc[3 * s], count = seg_desc[3 * s + 1];
    const bool resumes = seg_desc[3 * s + 2] != 0;
    double* out = part + (int64_t)s * (cells + 1);
    for (int64_t cell = threadIdx.x; cell < cells; cell += blockDim.x) {
        double acc = resumes ? open[cell] : 0.0;
        for (int64_t k = 0; k < count; ++k) acc = __dadd_rn(acc, v[(first + k) * cells + cell]);
        out[cell] = acc;
    }
    // serial sum of squares over the (k, cell) sequence, staged through smem
    double s2 = resumes ? *open_sq : 0.0;
    const int64_t len = count * cells;
    const double* base = v + first * cells;
    for (int64_t off = 0; off < len; off += RED_TILE) {
        const int64_t n = min((int64_t)RED_TILE, len - off);
        __syncthreads();
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) tile[i] = base[off + i];
        __syncthreads();
        if (threadIdx.x == 0)
            for (int64_t i = 0; i < n; ++i) s2 = __dadd_rn(s2, __dmul_rn(tile[i], tile[i]));
    }
    if (threadIdx.x == 0) out[cells] = s2;
}

// Commit segments in order: closed ones are added to the chunk-order total,
// a trailing unclosed one becomes the open chunk.  flags[s] = closes.
__global__ void k_commit(int nseg, int64_t cells, const double* __restrict__ part,
                         const int64_t* __restrict__ closes, double* __restrict__ total,
                         double* __restrict__ total_sq, double* __restrict__ open, double* __restrict__ open_sq) {
    for (int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cell <= cells;
         cell += (int64_t)gridDim.x * blockDim.x) {
        double* tot = cell < cells ? total + cell : total_sq;
        double* op = cell < cells ? open + cell : open_sq;
        double acc = *tot;
        for (int s = 0; s < nseg; ++s) {
            const double x = part[(int64_t)s * (cells + 1) + cell];
            if (closes[s]) acc = __dadd_rn(acc, x);
            else *op = x;
        }
        *tot = acc;
    }
}

int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

std::vector<Segment> plan_segments(int64_t k_begin, int64_t k_end, int rank, int world, const LevelState& st) {
    std::vector<Segment> out;
    if (k_end <= k_begin) return out;
    const int64_t q0 = k_begin / 64, q1 = (k_end - 1) / 64;
    for (int64_t q = q0; q <= q1; ++q) {
        if (q % world != rank) continue;
        const int64_t a = std::max(k_begin, q * 64), b = std::min(k_end, q * 64 + 64);
        Segment s{q, a, b - a, false, b == q * 64 + 64};
        s.resumes = (st.open_chunk == q && st.open_count > 0);
        out.push_back(s);
    }
    return out;
}

void exact_run(const RunArgs& a, const LevelSpec& lv, const std::vector<Segment>& segs, LevelState& st) {
    const Model& M = *a.model;
    Workspace& ws = *a.ws;
    cudaStream_t s = a.stream;
    const int64_t c = lv.c, cells = M.rows * M.cols;
    const bool ref = M.dm.stream == MLSK_STREAM_REF;
    const int64_t stream_len = ref ? M.ref_u64 + (lv.full ? 0 : c) : 0;
    // bytes per replication of workspace
    const int64_t per = (ref ? stream_len * 8 : 0) + c * 4 + (M.rows + M.cols) * c * 8 + cells * 8 + 8;
    const int64_t budget = int64_t(1) << 30;
    int64_t max_rep = std::max<int64_t>(1, budget / per);
    // uniform inv_probs = n (sampling.cpp:39), scaled by 1/s (sketch.cpp:37,73);
    // the full draw is the plain product: exact_inner / exact_matmul
    // (tensor.cpp:97-131) -- (a*b)*1 and o*1 are exact, so the same kernel serves
    const double w = lv.full ? 1.0 : (double)M.desc.n * kRescalePerturb;  // (1 unless the negative control)
    const double vdiv = lv.full ? 1.0 : (double)c;
    const double sf = lv.full ? 1.0 : 1.0 / (double)c;
    const double sc = lv.cc > 0 ? 1.0 / (double)lv.cc : 0.0;

    size_t i = 0;
    std::vector<int64_t> ks, desc, closes;
    while (i < segs.size()) {
        // a batch of whole segments
        ks.clear(); desc.clear(); closes.clear();
        size_t j = i;
        while (j < segs.size() && (ks.empty() || (int64_t)ks.size() + segs[j].count <= max_rep)) {
            desc.push_back((int64_t)ks.size());
            desc.push_back(segs[j].count);
            desc.push_back(segs[j].resumes ? 1 : 0);
            closes.push_back(segs[j].closes ? 1 : 0);
            for (int64_t k = 0; k < segs[j].count; ++k) ks.push_back(segs[j].k0 + k);
            ++j;
        }
        const int nb = (int)ks.size();
        const int nseg = (int)(j - i);
        ws.ks.ensure(nb);
        ws.idx.ensure((size_t)nb * c);
        ws.a_cols.ensure((size_t)nb * M.rows * c);
        ws.b_rows.ensure((size_t)nb * c * M.cols);
        ws.v.ensure((size_t)nb * cells);
        ws.seg_part.ensure((size_t)nseg * (cells + 1));
        ws.seg_desc.ensure((size_t)4 * nseg);
        MLSK_CUDA(cudaMemcpyAsync(ws.ks.p, ks.data(), sizeof(int64_t) * nb, cudaMemcpyHostToDevice, s));
        if (ref) {
            ws.stream.ensure((size_t)nb * stream_len);
            k_ref_stream<<<(nb + STREAM_WARPS - 1) / STREAM_WARPS, 32 * STREAM_WARPS, 0, s>>>(
                a.seed, lv.tag, ws.ks.p, nb, stream_len, ws.stream.p);
            launched();
        }
        if (lv.full)
            k_iota<<<grid_for((int64_t)nb * c), 256, 0, s>>>(nb, c, ws.idx.p);
        else
            k_indices<<<grid_for((int64_t)nb * c), 256, 0, s>>>(M.dm, a.seed, lv.tag, ws.ks.p, nb, c, ws.stream.p,
                                                                  stream_len, M.ref_u64, ws.idx.p);
        k_gather<<<grid_for((int64_t)nb * (M.rows + M.cols) * c), 256, 0, s>>>(
            M.dm, a.seed, lv.tag, ws.ks.p, nb, c, ws.stream.p, stream_len, ws.idx.p, ws.a_cols.p, ws.b_rows.p);
        k_sketch<<<grid_for((int64_t)nb * cells), 256, 0, s>>>(M.vector, M.rows, M.cols, nb, c, lv.cc, w, vdiv, sf, sc,
                                                                a.target, a.target_param, ws.a_cols.p,
                                                                ws.b_rows.p, ws.v.p);
        launched(3);
        if (a.probe_host && a.probe_k > 0) {
            for (int b = 0; b < nb; ++b) {
                if (ks[b] < a.probe_k) {
                    MLSK_CUDA(cudaMemcpyAsync(a.probe_host + ks[b] * c, ws.idx.p + (int64_t)b * c,
                                              sizeof(uint32_t) * c, cudaMemcpyDeviceToHost, s));
                }
            }
        }
        // segment partials + in-order commit
        std::vector<int64_t> both(desc);
        both.insert(both.end(), closes.begin(), closes.end());
        ws.seg_desc.ensure(both.size());
        MLSK_CUDA(cudaMemcpyAsync(ws.seg_desc.p, both.data(), sizeof(int64_t) * both.size(),
                                  cudaMemcpyHostToDevice, s));
        k_segments<<<nseg, RED_THREADS, 0, s>>>(ws.v.p, cells, ws.seg_desc.p, st.open(), st.open_sq(),
                                                ws.seg_part.p);
        k_commit<<<grid_for(cells + 1), 256, 0, s>>>(nseg, cells, ws.seg_part.p, ws.seg_desc.p + 3 * nseg,
                                                     st.total(), st.total_sq(), st.open(), st.open_sq());
        launched(2);
        // host bookkeeping of the open chunk
        for (size_t t = i; t < j; ++t) {
            st.count += segs[t].count;
            if (segs[t].closes) {
                st.open_chunk = -1;
                st.open_count = 0;
            } else {
                st.open_count = (segs[t].resumes ? st.open_count : 0) + segs[t].count;
                st.open_chunk = segs[t].chunk;
            }
        }
        // the host vectors are reused next batch; make sure the copies are done
        MLSK_CUDA(cudaStreamSynchronize(s));
        i = j;
    }
}

void exact_gather_sample(const Model& M, uint64_t seed, uint64_t tag, int64_t k, int64_t c, uint32_t* idx_host,
                         double* a_host, double* b_host, cudaStream_t s, Workspace& ws) {
    const bool ref = M.dm.stream == MLSK_STREAM_REF;
    const int64_t stream_len = ref ? M.ref_u64 + c : 0;
    ws.ks.ensure(1);
    ws.idx.ensure(c);
    ws.a_cols.ensure((size_t)M.rows * c);
    ws.b_rows.ensure((size_t)c * M.cols);
    MLSK_CUDA(cudaMemcpyAsync(ws.ks.p, &k, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    if (ref) {
        ws.stream.ensure(stream_len);
        k_ref_stream<<<1, 32 * STREAM_WARPS, 0, s>>>(seed, tag, ws.ks.p, 1, stream_len, ws.stream.p);
        launched();
    }
    k_indices<<<grid_for(c), 256, 0, s>>>(M.dm, seed, tag, ws.ks.p, 1, c, ws.stream.p, stream_len, M.ref_u64,
                                           ws.idx.p);
    k_gather<<<grid_for((M.rows + M.cols) * c), 256, 0, s>>>(M.dm, seed, tag, ws.ks.p, 1, c, ws.stream.p,
                                                             stream_len, ws.idx.p, ws.a_cols.p, ws.b_rows.p);
    launched(2);
    if (idx_host) MLSK_CUDA(cudaMemcpyAsync(idx_host, ws.idx.p, sizeof(uint32_t) * c, cudaMemcpyDeviceToHost, s));
    if (a_host) MLSK_CUDA(cudaMemcpyAsync(a_host, ws.a_cols.p, sizeof(double) * M.rows * c, cudaMemcpyDeviceToHost, s));
    if (b_host) MLSK_CUDA(cudaMemcpyAsync(b_host, ws.b_rows.p, sizeof(double) * c * M.cols, cudaMemcpyDeviceToHost, s));
    MLSK_CUDA(cudaStreamSynchronize(s));
}

}  // namespace mlsk
