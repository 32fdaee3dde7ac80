// The global (depth, index) order (splat.cpp:179-184) and the scan arrays the raster
// kernels read in place of per-tile lists (splat.cpp:187-200):
//   1. depth sort: stable LSD radix sort of compressed fp32 depth keys (tsb_sort.cu,
//      value = Gaussian index, so ties keep index order); runs of equal keys are ordered
//      by the fp64 depth on read (tsb_ties.cuh), or the exact 64-bit sort (below).
//   2. k_order_ranks: rank -> (Gaussian, tile rect).  Each raster block scans these in
//      rank order and keeps the ranks whose tile rect covers its tile -- the reference's
//      tile list -- until its pixels have terminated (tsb_raster.cu), so no tile list is
//      ever materialised; k_tile_lists builds the complete lists for parity checks only.
//   3. long orders (> kSlMinRanks): per 8 x 8-tile super-tile, the ranks meeting it, in
//      rank order (k_order_ranks counts, k_sl_rowscan, k_sl_emit); a block then scans its
//      super-tile's list instead of the whole order.
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
// compressed keys resolved once here, not by every reader) and its tile rect, and the
// super-tile lists -- a stable counting sort of the (rank, super-tile) pairs by super-
// tile, with the pairs never materialised:
//   k_order_ranks  ord / trect; per block (a contiguous range of 256-rank chunks) the
//                  pair count per super-tile -> hist[s][block]
//   k_sl_rowscan   a block per super-tile: hist row -> exclusive offsets, row total
//   k_sl_emit      the rows' bases (a scan of the totals, per block), then each chunk's
//                  pairs at their stable positions
// A rect is a product of a column range and a row range of super-tiles, so a warp's
// coverage of super-tile (sx, sy) is colmask[sx] & rowmask[sy]: sup_x + sup_y ballots
// per warp instead of one per super-tile.
__device__ __forceinline__ void super_rect(uint2 tr, int lg, int& sx0, int& sx1, int& sy0, int& sy1) {
    sx0 = (int)(tr.x & 0xffffu) >> lg;
    sx1 = (int)(tr.x >> 16) >> lg;
    sy0 = (int)(tr.y & 0xffffu) >> lg;
    sy1 = (int)(tr.y >> 16) >> lg;
}

// The block's contiguous range of chunks (the same in k_order_ranks and k_sl_emit: the
// histogram holds one column per block).
__device__ __forceinline__ void block_chunks(int V, int& c0, int& c1) {
    const int nch = (V + kSlChunk - 1) / kSlChunk, per = (nch + gridDim.x - 1) / gridDim.x;
    c0 = min(nch, (int)blockIdx.x * per);
    c1 = min(nch, c0 + per);
}

// The warp's column / row coverage masks of its lanes' super rects (wm[0 .. sup_x) columns,
// wm[sup_x .. sup_x + sup_y) rows).
__device__ __forceinline__ void warp_masks(bool valid, int sx0, int sx1, int sy0, int sy1, const SuperK& sk,
                                           uint32_t* wm, int lane) {
    const int sup_y = sk.nsup / sk.sup_x;
    for (int sx = 0; sx < sk.sup_x; ++sx) {
        const unsigned b = __ballot_sync(0xffffffffu, valid && sx0 <= sx && sx <= sx1);
        if (lane == 0) wm[sx] = b;
    }
    for (int sy = 0; sy < sup_y; ++sy) {
        const unsigned b = __ballot_sync(0xffffffffu, valid && sy0 <= sy && sy <= sy1);
        if (lane == 0) wm[sk.sup_x + sy] = b;
    }
    __syncwarp();
}

__global__ void __launch_bounds__(kSlChunk) k_order_ranks(const uint32_t* __restrict__ sorted, TieK T,
                                                          const uint2* __restrict__ rect, int ts,
                                                          const int32_t* __restrict__ n_rank, uint32_t* __restrict__ ord,
                                                          uint2* __restrict__ trect, SuperK sk) {
    __shared__ uint32_t cnt[kSlMaxSup];
    __shared__ uint32_t wmask[kSlChunk / 32][2 * kSlMaxSupSide];
    if (block_aborted(T.abort)) return;
    const int V = *n_rank, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int c0, c1;
    block_chunks(V, c0, c1);
    for (int s = tid; s < sk.nsup; s += kSlChunk) cnt[s] = 0;
    __syncthreads();
    uint32_t* wm = wmask[warp];
    for (int c = c0; c < c1; ++c) {
        const int r = c * kSlChunk + tid;
        int sx0 = 1, sx1 = 0, sy0 = 1, sy1 = 0;
        if (r < V) {
            const uint32_t g = sorted_at(sorted, T, r, V);
            const uint2 rc = rect[g];
            const int x0 = rc.x & 0xffff, x1 = rc.x >> 16, y0 = rc.y & 0xffff, y1 = rc.y >> 16;
            const uint2 tr = make_uint2((uint32_t)(x0 / ts) | ((uint32_t)((x1 - 1) / ts) << 16),
                                        (uint32_t)(y0 / ts) | ((uint32_t)((y1 - 1) / ts) << 16));
            ord[r] = g;
            trect[r] = tr;
            super_rect(tr, sk.sup_log, sx0, sx1, sy0, sy1);
        }
        if (sk.nsup > 0 && __any_sync(0xffffffffu, r < V)) {
            warp_masks(r < V, sx0, sx1, sy0, sy1, sk, wm, lane);
            for (int s = lane; s < sk.nsup; s += 32) {
                const int sy = s / sk.sup_x, sx = s - sy * sk.sup_x;
                const uint32_t k = __popc(wm[sx] & wm[sk.sup_x + sy]);
                if (k) atomicAdd(&cnt[s], k);
            }
            __syncwarp();
        }
    }
    __syncthreads();
    for (int s = tid; s < sk.nsup; s += kSlChunk) sk.hist[(size_t)s * sk.hist_stride + blockIdx.x] = cnt[s];
    if (sk.work && blockIdx.x == 0 && tid == 0) atomicAdd(&sk.work[2], (unsigned long long)V);  // profiling
}

// Row s of the histogram (one column per k_order_ranks block) -> exclusive offsets within
// the row; row_total[s] = its sum.
__global__ void __launch_bounds__(256) k_sl_rowscan(SuperK sk, int G, const int32_t* __restrict__ abort) {
    __shared__ uint32_t part[256];
    if (block_aborted(abort)) return;
    uint32_t* row = sk.hist + (size_t)blockIdx.x * sk.hist_stride;
    const int tid = threadIdx.x, per = (G + 255) / 256, c0 = min(G, tid * per), c1 = min(G, c0 + per);
    uint32_t v[(kSlMaxBlocks + 255) / 256];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < (kSlMaxBlocks + 255) / 256; ++k) {
        v[k] = c0 + k < c1 ? row[c0 + k] : 0u;
        sum += v[k];
    }
    part[tid] = sum;
    __syncthreads();
    for (int d = 1; d < 256; d <<= 1) {
        const uint32_t u = tid >= d ? part[tid - d] : 0u;
        __syncthreads();
        part[tid] += u;
        __syncthreads();
    }
    uint32_t off = part[tid] - sum;
#pragma unroll
    for (int k = 0; k < (kSlMaxBlocks + 255) / 256; ++k) {
        if (c0 + k < c1) row[c0 + k] = off;
        off += v[k];
    }
    if (tid == 255) sk.row_total[blockIdx.x] = part[255];
}

__global__ void __launch_bounds__(kSlChunk) k_sl_emit(const int32_t* __restrict__ n_rank,
                                                      const uint2* __restrict__ trect, SuperK sk,
                                                      int32_t* __restrict__ abort) {
    __shared__ uint32_t base[kSlMaxSup];
    __shared__ uint16_t wpre[kSlChunk / 32][kSlMaxSup];  // warps before w: their pairs per super-tile
    __shared__ uint32_t wmask[kSlChunk / 32][2 * kSlMaxSupSide];
    __shared__ uint32_t part[kSlChunk];
    if (block_aborted(abort)) return;
    const int V = *n_rank, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t below = (1u << lane) - 1u;
    // the rows' bases: exclusive scan of the row totals (nsup <= 1024: 4 per thread)
    constexpr int kPer = kSlMaxSup / kSlChunk;
    uint32_t t[kPer], sum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int s = tid * kPer + k;
        t[k] = s < sk.nsup ? sk.row_total[s] : 0u;
        sum += t[k];
    }
    part[tid] = sum;
    __syncthreads();
    for (int d = 1; d < kSlChunk; d <<= 1) {
        const uint32_t u = tid >= d ? part[tid - d] : 0u;
        __syncthreads();
        part[tid] += u;
        __syncthreads();
    }
    const uint32_t total = part[kSlChunk - 1];
    {
        uint32_t off = part[tid] - sum;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int s = tid * kPer + k;
            if (s < sk.nsup) {
                base[s] = off + sk.hist[(size_t)s * sk.hist_stride + blockIdx.x];
                if (blockIdx.x == 0) sk.off[s] = off;
            }
            off += t[k];
        }
    }
    if (blockIdx.x == 0 && tid == 0) {
        sk.off[sk.nsup] = total;
        *sk.total = (int32_t)min(total, 0x7fffffffu);
        if (total > (uint32_t)sk.cap) atomicOr(abort, 1);  // the lists need more storage: redo
        if (sk.work) atomicAdd(&sk.work[3], (unsigned long long)total);
    }
    if (total > (uint32_t)sk.cap) return;  // (block-uniform)
    int c0, c1;
    block_chunks(V, c0, c1);
    uint32_t* wm = wmask[warp];
    for (int c = c0; c < c1; ++c) {
        const int r = c * kSlChunk + tid;
        int sx0 = 1, sx1 = 0, sy0 = 1, sy1 = 0;
        uint2 tr = make_uint2(0u, 0u);
        if (r < V) {
            tr = trect[r];
            super_rect(tr, sk.sup_log, sx0, sx1, sy0, sy1);
        }
        warp_masks(r < V, sx0, sx1, sy0, sy1, sk, wm, lane);
        __syncthreads();
        // per super-tile: the warps' exclusive prefix of their pair counts, the chunk total
        for (int s = tid; s < sk.nsup; s += kSlChunk) {
            const int sy = s / sk.sup_x, sx = s - sy * sk.sup_x;
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kSlChunk / 32; ++w) {
                wpre[w][s] = (uint16_t)run;
                run += __popc(wmask[w][sx] & wmask[w][sk.sup_x + sy]);
            }
        }
        __syncthreads();
        for (int sy = sy0; sy <= sy1; ++sy) {
            const uint32_t rm = wm[sk.sup_x + sy];
            for (int sx = sx0; sx <= sx1; ++sx) {
                const int s = sy * sk.sup_x + sx;
                const uint32_t pos = base[s] + wpre[warp][s] + __popc(wm[sx] & rm & below);
                sk.rank[pos] = (uint32_t)r;
                sk.rect[pos] = tr;
            }
        }
        __syncthreads();
        for (int s = tid; s < sk.nsup; s += kSlChunk) {
            const int sy = s / sk.sup_x, sx = s - sy * sk.sup_x;
            base[s] += wpre[kSlChunk / 32 - 1][s] +
                       __popc(wmask[kSlChunk / 32 - 1][sx] & wmask[kSlChunk / 32 - 1][sk.sup_x + sy]);
        }
        __syncthreads();
    }
}

int launch_order_ranks(const uint32_t* sorted, const TieK& T, const uint2* rect, int ts, const int32_t* n_rank,
                       int n, uint32_t* ord, uint2* trect, const SuperK& sk, cudaStream_t st) {
    if (n <= 0) return 0;
    const int grid = std::min(sk.hist_stride, (n + kSlChunk - 1) / kSlChunk);
    k_order_ranks<<<grid, kSlChunk, 0, st>>>(sorted, T, rect, ts, n_rank, ord, trect, sk);
    if (sk.nsup == 0) return 1;  // a short order: no lists
    k_sl_rowscan<<<sk.nsup, 256, 0, st>>>(sk, grid, T.abort);
    k_sl_emit<<<grid, kSlChunk, 0, st>>>(n_rank, trect, sk, T.abort);
    return 3;
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
    if (block_aborted(sc.abort)) return;
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
