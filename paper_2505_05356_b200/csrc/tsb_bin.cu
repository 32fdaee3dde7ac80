// The global (depth, index) order (splat.cpp:179-184) and the scan arrays the raster
// kernels read in place of per-tile lists (splat.cpp:187-200):
//   1. depth sort: stable LSD radix sort of compressed fp32 depth keys (tsb_sort.cu,
//      value = Gaussian index, so ties keep index order); runs of equal keys are ordered
//      by the fp64 depth on read (tsb_ties.cuh), or the exact 64-bit sort (below).
//   2. k_order_ranks: rank -> (Gaussian, tile rect).  Each raster block scans these in
//      rank order and keeps the ranks whose tile rect covers its tile -- the reference's
//      tile list -- until its pixels have terminated (tsb_raster.cu), so no list is ever
//      materialised; k_tile_lists builds the complete lists for parity checks only.
#include <algorithm>

#include "tsb_internal.h"
#include "tsb_ties.cuh"

namespace tsb {

int launch_sort_depth(uint32_t* keys_a, uint32_t* keys_b, uint32_t* vals_a, uint32_t* vals_b,
                      const uint32_t* key_range, int n, uint32_t* scratch, cudaStream_t st) {
    if (n <= 0) return 0;
    return radix_sort24(keys_a, keys_b, vals_a, vals_b, n, scratch, key_range, st);
}

__global__ void k_materialize_order(const uint32_t* __restrict__ sorted, TieK T, const int32_t* __restrict__ n_visible,
                                    uint32_t* __restrict__ out) {
    const int V = *n_visible;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < V; r += gridDim.x * blockDim.x)
        out[r] = sorted_at(sorted, T, r, V);
}

void launch_materialize_order(const uint32_t* sorted, const TieK& T, const int32_t* n_visible, int n, uint32_t* out,
                              cudaStream_t st) {
    if (n <= 0) return;
    k_materialize_order<<<std::min(148 * 8, (n + 255) / 256), 256, 0, st>>>(sorted, T, n_visible, out);
}

// Exact fallback for long equal-fp32 runs: stable LSD on the fp64 depth bits as two
// 32-bit sorts (low word, then high word gathered through the permutation).
__global__ void k_key_lo(const double* __restrict__ depth64, const uint32_t* __restrict__ touched,
                         uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, int n) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    keys[g] = touched[g] ? (uint32_t)(__double_as_longlong(depth64[g]) & 0xffffffffull) : 0u;
    vals[g] = (uint32_t)g;
}

__global__ void k_key_hi(const double* __restrict__ depth64, const uint32_t* __restrict__ touched,
                         uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t g = vals[i];
    keys[i] = touched[g] ? (uint32_t)((unsigned long long)__double_as_longlong(depth64[g]) >> 32) : 0xffffffffu;
}

int launch_sort_depth64(const double* depth64, const uint32_t* touched, uint32_t* keys_a, uint32_t* keys_b,
                        uint32_t* vals_a, uint32_t* vals_b, int n, uint32_t* scratch, cudaStream_t st) {
    if (n <= 0) return 0;
    k_key_lo<<<(n + 255) / 256, 256, 0, st>>>(depth64, touched, keys_a, vals_a, n);
    int l = radix_sort32(keys_a, keys_b, vals_a, vals_b, n, scratch, st);
    k_key_hi<<<(n + 255) / 256, 256, 0, st>>>(depth64, touched, keys_a, vals_a, n);
    l += radix_sort32(keys_a, keys_b, vals_a, vals_b, n, scratch, st);
    return l + 2;
}

// ---------------------------------------------------------------------------
// The scan arrays of the raster kernels (ScanK): rank -> Gaussian (runs of equal
// compressed keys resolved once here, not by every reader) and its tile rect.
__global__ void __launch_bounds__(256) k_order_ranks(const uint32_t* __restrict__ sorted, TieK T,
                                                     const uint2* __restrict__ rect, int ts,
                                                     const int32_t* __restrict__ n_rank, uint32_t* __restrict__ ord,
                                                     uint2* __restrict__ trect) {
    if (*T.abort) return;
    const int V = *n_rank;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < V; r += gridDim.x * blockDim.x) {
        const uint32_t g = sorted_at(sorted, T, r, V);
        const uint2 rc = rect[g];
        const int x0 = rc.x & 0xffff, x1 = rc.x >> 16, y0 = rc.y & 0xffff, y1 = rc.y >> 16;
        ord[r] = g;
        trect[r] = make_uint2((uint32_t)(x0 / ts) | ((uint32_t)((x1 - 1) / ts) << 16),
                              (uint32_t)(y0 / ts) | ((uint32_t)((y1 - 1) / ts) << 16));
    }
}

void launch_order_ranks(const uint32_t* sorted, const TieK& T, const uint2* rect, int ts, const int32_t* n_rank,
                        int n, uint32_t* ord, uint2* trect, cudaStream_t st) {
    if (n <= 0) return;
    k_order_ranks<<<std::min(148 * 8, (n + 255) / 256), 256, 0, st>>>(sorted, T, rect, ts, n_rank, ord, trect);
}

// Deterministic backward: det_off[r] = sum over ranks r' < r of (rect area in tiles) x
// sub-blocks, one block (a mode for bit-reproducible gradients, not the fast path).
__global__ void __launch_bounds__(1024) k_det_offsets(ScanK sc, uint32_t* __restrict__ det_off,
                                                      uint32_t* __restrict__ total) {
    __shared__ uint32_t part[1024];
    const int V = *sc.n_rank, tid = threadIdx.x;
    const int per = (V + 1023) / 1024, r0 = min(V, tid * per), r1 = min(V, r0 + per);
    auto area = [&](int r) {
        const uint2 tr = sc.trect[r];
        return (uint32_t)(((tr.x >> 16) - (tr.x & 0xffff) + 1) * ((tr.y >> 16) - (tr.y & 0xffff) + 1) * sc.nsub2);
    };
    uint32_t sum = 0;
    for (int r = r0; r < r1; ++r) sum += area(r);
    part[tid] = sum;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {  // inclusive scan of the thread sums
        const uint32_t v = tid >= d ? part[tid - d] : 0u;
        __syncthreads();
        part[tid] += v;
        __syncthreads();
    }
    uint32_t off = part[tid] - sum;
    for (int r = r0; r < r1; ++r) {
        det_off[r] = off;
        off += area(r);
    }
    if (tid == 1023) det_off[V] = *total = part[1023];
}

void launch_det_offsets(const ScanK& sc, uint32_t* det_off, uint32_t* total, cudaStream_t st) {
    k_det_offsets<<<1, 1024, 0, st>>>(sc, det_off, total);
}

// Each visible Gaussian's screen-space gradients: its slots summed over its rect's tiles
// (row-major) and the tiles' raster sub-blocks, always in that order.
__global__ void __launch_bounds__(256) k_det_reduce(ScanK sc, double* __restrict__ screen, int scap) {
    if (*sc.abort) return;
    const int V = *sc.n_rank;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < V; r += gridDim.x * blockDim.x) {
        const uint32_t s0 = sc.det_off[r], s1 = sc.det_off[r + 1];
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint32_t sl = s0; sl < s1; ++sl) {
            const float4 a = reinterpret_cast<const float4*>(sc.det_part)[2 * (size_t)sl];
            const float4 b = reinterpret_cast<const float4*>(sc.det_part)[2 * (size_t)sl + 1];
            acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
            acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
        }
        const uint32_t g = sc.ord[r];
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if (acc[c] != 0.0) screen[(size_t)c * scap + g] += acc[c];
    }
}

void launch_det_reduce(const ScanK& sc, int n, double* screen, int scap, cudaStream_t st) {
    if (n <= 0) return;
    k_det_reduce<<<std::min(148 * 8, (n + 255) / 256), 256, 0, st>>>(sc, screen, scap);
}

// Parity / debug: each tile's complete list (splat.cpp:187-200) -- a block per tile
// scans every rank of the order and keeps the covering ones (their ranks), in order.
__global__ void __launch_bounds__(256) k_tile_lists(ScanK sc, int tiles_x, const int64_t* __restrict__ offsets,
                                                    uint32_t* __restrict__ counts, uint32_t* __restrict__ ids) {
    __shared__ int wsum[8];
    const int tile = blockIdx.x, tx = tile % tiles_x, ty = tile / tiles_x;
    const int V = *sc.n_rank, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t pos = offsets ? offsets[tile] : 0;
    uint32_t total = 0;
    for (int r0 = 0; r0 < V; r0 += 256) {
        const int r = r0 + threadIdx.x;
        const bool cov = r < V && tile_covers(sc.trect[r], tx, ty);
        const unsigned b = __ballot_sync(0xffffffffu, cov);
        if (lane == 0) wsum[warp] = __popc(b);
        __syncthreads();
        int off = __popc(b & ((1u << lane) - 1u)), tot = 0;
        for (int w = 0; w < 8; ++w) {
            off += w < warp ? wsum[w] : 0;
            tot += wsum[w];
        }
        if (cov && ids) ids[pos + off] = (uint32_t)r;  // the reference lists hold ranks
        pos += tot;
        total += tot;
        __syncthreads();
    }
    if (counts && threadIdx.x == 0) counts[tile] = total;
}

void launch_tile_counts(const ScanK& sc, int tiles_x, int ntiles, uint32_t* counts, cudaStream_t st) {
    k_tile_lists<<<ntiles, 256, 0, st>>>(sc, tiles_x, nullptr, counts, nullptr);
}

void launch_tile_lists(const ScanK& sc, int tiles_x, int ntiles, const int64_t* offsets, uint32_t* ids,
                       cudaStream_t st) {
    k_tile_lists<<<ntiles, 256, 0, st>>>(sc, tiles_x, offsets, nullptr, ids);
}

}  // namespace tsb
