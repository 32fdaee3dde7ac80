// Tile binning: global (depth, index) order -> per-tile lists in that order.
// Replaces the reference's std::sort of Prepared structs (splat.cpp:179-184)
// and build_tiles (splat.cpp:187-200).
//
//   1. depth sort: stable LSD radix sort of the fp64 depth bits (value = Gaussian
//      index, input in index order -> ties broken by index exactly as the
//      reference's comparator does).  The position in this order is the rank.
//   2. depth-chunked counting sort by tile, no key materialisation:
//      ranks are cut into segments of kSeg (one warp each) and segments into
//      geometrically growing chunks.  Per chunk:
//        k_bin_count  per (tile, segment) entry counts.  A warp handles 32 ranks
//                     at a time; a tile is covered by lane j iff bit j of
//                     colmask[tx] & rowmask[ty] (two ballot-built masks), so the
//                     covering lanes of any tile are known in O(1).
//        k_bin_scan   per tile: exclusive scan over the chunk's segments; tile
//                     lengths; exclusive scan over tiles -> chunk ranges.
//        k_bin_emit   stable scatter of Gaussian indices: position = cursor of
//                     (tile, segment) + number of lower lanes covering the tile.
//      The tile lists of a chunk are exactly the reference's lists restricted
//      to that chunk's ranks, so their concatenation over chunks is the
//      reference list.  Tiles whose pixels have all terminated are skipped by
//      later chunks (the composite never reads past termination), unless the
//      caller asks for full lists (parity mode).
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
namespace {

constexpr int kBinThreads = 128;  // one CTA per segment; all threads share a batch's tiles
constexpr int kSmemTiles = 8192;  // per-CTA shared-memory tile counters up to this many tiles

// Tiles whose pixels have all terminated are not binned again.  No tile can be
// finished before the first chunk's raster, so chunk 0 skips the (global) check.
__device__ __forceinline__ bool tile_done(const BinK& B, int t) {
    return B.skip_done && B.chunk > 0 && B.tile_blocks_done[t] >= B.blocks_per_tile;
}

// Every planned chunk is launched; a chunk is live only while the frame is not
// aborted, visible ranks remain and (unless full lists are requested) some raster
// block has not terminated.  The host never waits between chunks.  Inputs are
// written only by earlier kernels of the stream, so all kernels of a chunk agree
// (the abort word can only turn on, which every later kernel honours anyway).
__device__ __forceinline__ bool chunk_live(const BinK& B) {
    if (*B.overflow) return false;
    if (B.chunk == 0) return true;
    if (B.seg0 * kSeg >= *B.n_visible) return false;
    return !(B.skip_done && *B.blocks_done_total >= B.nblocks);
}

struct Box {
    int x0, x1, y0, y1;  // union of the batch's tile rects (inclusive); empty when x0 > x1
};

// Warp 0 loads the 32 ranks of one batch and builds the per-column / per-row
// lane masks: lane j covers tile (tx, ty) iff bit j of colmask[tx] & rowmask[ty].
// Returns the union box (valid in every thread after the caller's barrier).
__device__ __forceinline__ void load_batch_warp0(const BinK& B, int r, int V, uint32_t* colmask, uint32_t* rowmask,
                                                 uint32_t* gids, int* box, int lane) {
    int tx0 = 1, tx1 = 0, ty0 = 1, ty1 = 0;
    uint32_t g = 0;
    if (r < V) {
        g = sorted_at(B.sorted_gidx, B.ties, r, V);
        const uint2 rc = B.rect[g];
        const int x0 = rc.x & 0xffff, x1 = rc.x >> 16, y0 = rc.y & 0xffff, y1 = rc.y >> 16;
        tx0 = x0 / B.ts;
        tx1 = (x1 - 1) / B.ts;
        ty0 = y0 / B.ts;
        ty1 = (y1 - 1) / B.ts;
    }
    gids[lane] = g;
    const bool valid = tx0 <= tx1;
    const int ux0 = __reduce_min_sync(0xffffffffu, valid ? tx0 : 0x7fffffff);
    const int ux1 = __reduce_max_sync(0xffffffffu, valid ? tx1 : -1);
    const int uy0 = __reduce_min_sync(0xffffffffu, valid ? ty0 : 0x7fffffff);
    const int uy1 = __reduce_max_sync(0xffffffffu, valid ? ty1 : -1);
    for (int tx = ux0; tx <= ux1; ++tx) {
        const uint32_t m = __ballot_sync(0xffffffffu, valid && tx0 <= tx && tx <= tx1);
        if (lane == 0) colmask[tx] = m;
    }
    for (int ty = uy0; ty <= uy1; ++ty) {
        const uint32_t m = __ballot_sync(0xffffffffu, valid && ty0 <= ty && ty <= ty1);
        if (lane == 0) rowmask[ty] = m;
    }
    if (lane == 0) {
        box[0] = ux0;
        box[1] = ux1;
        box[2] = uy0;
        box[3] = uy1;
    }
}

// done[t / 32] bit t: tile t is not binned by this chunk
__device__ __forceinline__ void stage_done(const BinK& B, uint32_t* done) {
    const bool check = B.skip_done && B.chunk > 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int t0 = warp * 32; t0 < B.ntiles; t0 += nwarps * 32) {
        const int t = t0 + lane;
        const bool d = check && t < B.ntiles && B.tile_blocks_done[t] >= B.blocks_per_tile;
        const uint32_t bits = __ballot_sync(0xffffffffu, d);
        if (lane == 0) done[t0 >> 5] = bits;
    }
}
__device__ __forceinline__ bool is_done(const uint32_t* done, int t) { return (done[t >> 5] >> (t & 31)) & 1u; }

}  // namespace

// Per (segment, tile) entry counts of one depth chunk.  CTAs stride over the
// chunk's segments of kSeg ranks; per batch of 32 ranks the threads walk the
// tiles of the batch's union box (the number of coverers of a tile is popc of
// two masks).
template <bool SMEM>
__global__ void __launch_bounds__(kBinThreads) k_bin_count(BinK B) {
    extern __shared__ uint32_t smem[];
    __shared__ int box[4];
    if (!chunk_live(B)) return;
    const int tid = threadIdx.x, lane = tid & 31;
    uint32_t* done = smem;
    uint32_t* gids = done + ((B.ntiles + 31) >> 5);
    uint32_t* colmask = gids + 32;
    uint32_t* rowmask = colmask + B.tiles_x;
    stage_done(B, done);
    const int V = *B.n_visible;
    for (int segl = blockIdx.x; segl < B.nseg; segl += gridDim.x) {
        uint32_t* cnt = SMEM ? rowmask + B.tiles_y : B.hist + (size_t)segl * B.ntiles;
        const int r0 = (B.seg0 + segl) * kSeg;
        for (int t = tid; t < B.ntiles; t += kBinThreads) cnt[t] = 0u;
        __syncthreads();
        for (int b = 0; b < kSeg && r0 + b < V; b += 32) {
            if (tid < 32) load_batch_warp0(B, r0 + b + lane, V, colmask, rowmask, gids, box, lane);
            __syncthreads();
            const int bw = box[1] - box[0] + 1;
            const int area = bw > 0 ? bw * (box[3] - box[2] + 1) : 0;
            for (int i = tid; i < area; i += kBinThreads) {
                const int q = i / bw;
                const int ty = box[2] + q, tx = box[0] + (i - q * bw);
                const uint32_t m = colmask[tx] & rowmask[ty];
                if (m) {
                    const int t = ty * B.tiles_x + tx;
                    if (!is_done(done, t)) cnt[t] += (uint32_t)__popc(m);
                }
            }
            __syncthreads();
        }
        if (SMEM) {
            uint32_t* h = B.hist + (size_t)segl * B.ntiles;
            for (int t = tid; t < B.ntiles; t += kBinThreads) h[t] = cnt[t];
        }
        __syncthreads();
    }
}

// Per tile: exclusive scan over the chunk's segments (in place, segment-major
// layout) and the tile's length.  Block = 32 tiles x 32 warps; warp w owns a
// contiguous range of segments.
__global__ void __launch_bounds__(1024) k_bin_scan_segments(BinK B) {
    __shared__ uint32_t part[32][33];
    if (!chunk_live(B)) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int t = blockIdx.x * 32 + lane;
    const int per = (B.nseg + 31) / 32;
    const int s0 = w * per, s1 = min(B.nseg, s0 + per);
    uint32_t sum = 0;
    if (t < B.ntiles) {
#pragma unroll 4
        for (int s = s0; s < s1; ++s) sum += B.hist[(size_t)s * B.ntiles + t];
    }
    part[w][lane] = sum;
    __syncthreads();
    uint32_t off = 0, tot = 0;
    for (int i = 0; i < 32; ++i) {
        const uint32_t v = part[i][lane];
        off += i < w ? v : 0u;
        tot += v;
    }
    if (t < B.ntiles) {
        for (int s = s0; s < s1; ++s) {
            uint32_t* h = B.hist + (size_t)s * B.ntiles + t;
            const uint32_t v = *h;
            *h = off;
            off += v;
        }
        if (w == 0) B.tile_len[t] = tot;
    }
}

// Exclusive scan of tile lengths -> this chunk's ranges; advances the running
// list offset.  One block.  SEGS: also does k_bin_scan_segments' per-tile scan over
// the chunk's segments first (small chunks: one launch instead of two).
template <bool SEGS>
__global__ void k_bin_scan_tiles(BinK B) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t s_carry;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    const uint32_t base = *B.list_off;
    if (!chunk_live(B)) {  // empty chunk: every tile skipped (the fix-up scans ranks from here)
        for (int t = tid; t < B.ntiles; t += blockDim.x) {
            const uint32_t cum = B.chunk == 0 ? 0u : B.prev_ranges[t].z + B.prev_ranges[t].y;
            B.ranges[t] = make_uint4(base, 0u, cum, 1u);
        }
        return;
    }
    if (SEGS) {
        for (int t = tid; t < B.ntiles; t += blockDim.x) {
            uint32_t off = 0;
            for (int sg = 0; sg < B.nseg; ++sg) {
                uint32_t* h = B.hist + (size_t)sg * B.ntiles + t;
                const uint32_t c = *h;
                *h = off;
                off += c;
            }
            B.tile_len[t] = off;
        }
        __syncthreads();
    }
    for (int t0 = 0; t0 < B.ntiles; t0 += blockDim.x) {
        const int t = t0 + tid;
        const uint32_t v = t < B.ntiles ? B.tile_len[t] : 0u;
        uint32_t inc = v;
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += u;
        }
        if (lane == 31) warp_sums[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            uint32_t ws = lane < nw ? warp_sums[lane] : 0u;
            uint32_t wi = ws;
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, wi, d);
                if (lane >= d) wi += u;
            }
            if (lane < nw) warp_sums[lane] = wi - ws;
        }
        __syncthreads();
        const uint32_t carry = s_carry;
        if (t < B.ntiles) {
            const uint32_t start = base + carry + warp_sums[wid] + inc - v;
            const uint32_t cum = B.chunk == 0 ? 0u : B.prev_ranges[t].z + B.prev_ranges[t].y;
            const uint32_t skipped = (B.skip_done && B.tile_blocks_done[t] >= B.blocks_per_tile) ? 1u : 0u;
            B.ranges[t] = make_uint4(start, v, cum, skipped);
            B.tile_start[t] = start;
        }
        __syncthreads();
        if (tid == blockDim.x - 1) s_carry = carry + warp_sums[wid] + inc;
        __syncthreads();
    }
    if (tid == 0) {
        const uint32_t end = base + s_carry;
        *B.list_off = end;
        if (end > B.capacity) atomicOr(B.overflow, 1);
    }
}

// Stable scatter of one depth chunk.  CTAs stride over segments; per batch of
// 32 ranks the threads walk the batch's union tiles and the coverers of tile t
// (bits of colmask & rowmask, in rank order) form one contiguous run at the
// (segment, tile) cursor.  STAGED: runs are first laid out tile-major in a
// shared-memory buffer (local exclusive scan of the segment's per-tile counts),
// then flushed with consecutive threads writing consecutive list entries -- a
// few coalesced runs per tile instead of one scattered 4-byte store per entry.
// A segment with more entries than the buffer holds writes directly.
template <bool STAGED>
__global__ void __launch_bounds__(kBinThreads) k_bin_emit(BinK B, int cap) {
    extern __shared__ uint32_t smem[];
    __shared__ int box[4];
    __shared__ uint32_t s_wsum[kBinThreads / 32];
    __shared__ uint32_t s_total;
    if (!chunk_live(B)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nt = B.ntiles;
    uint32_t* done = smem;
    uint32_t* gids = done + ((nt + 31) >> 5);
    uint32_t* colmask = gids + 32;
    uint32_t* rowmask = colmask + B.tiles_x;
    uint32_t* cur_s = rowmask + B.tiles_y;  // STAGED: local cursor (or global cursor when over capacity)
    uint32_t* delta = cur_s + nt;          // STAGED: global list position - local position
    uint32_t* seg_g = delta + nt;          // STAGED: the segment's Gaussian indices
    uint16_t* buf_t = reinterpret_cast<uint16_t*>(seg_g + kSeg);
    uint8_t* buf_r = reinterpret_cast<uint8_t*>(buf_t + cap);
    stage_done(B, done);
    const int V = *B.n_visible;
    for (int segl = blockIdx.x; segl < B.nseg; segl += gridDim.x) {
        const int r0 = (B.seg0 + segl) * kSeg;
        if (r0 >= V) break;  // uniform; later segments of this CTA are past V too
        uint32_t* h = B.hist + (size_t)segl * nt;
        uint32_t* cur = STAGED ? cur_s : h;  // !STAGED: the hist row becomes the cursor in place
        uint32_t total = 0xffffffffu;
        if (STAGED) {
            // this segment's per-tile counts -> tile-major local offsets (exclusive scan)
            const uint32_t* hn = segl + 1 < B.nseg ? h + nt : B.tile_len;
            for (int t = tid; t < nt; t += kBinThreads) {
                const uint32_t ht = h[t];
                cur[t] = hn[t] - ht;
                delta[t] = B.tile_start[t] + ht;
            }
            for (int i = tid; i < kSeg; i += kBinThreads) seg_g[i] = r0 + i < V ? sorted_at(B.sorted_gidx, B.ties, r0 + i, V) : 0u;
            __syncthreads();
            const int per = (nt + kBinThreads - 1) / kBinThreads;
            const int t0 = tid * per, t1 = min(nt, t0 + per);
            uint32_t sum = 0;
            for (int t = t0; t < t1; ++t) sum += cur[t];
            uint32_t inc = sum;
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += u;
            }
            if (lane == 31) s_wsum[warp] = inc;
            __syncthreads();
            uint32_t run = inc - sum;
            for (int w = 0; w < warp; ++w) run += s_wsum[w];
            if (tid == kBinThreads - 1) s_total = run + sum;
            for (int t = t0; t < t1; ++t) {
                const uint32_t c = cur[t];
                cur[t] = run;
                delta[t] -= run;
                run += c;
            }
            __syncthreads();
            total = s_total;
        }
        const bool staged = STAGED && total <= (uint32_t)cap;
        if (!staged) {
            for (int t = tid; t < nt; t += kBinThreads) cur[t] = B.tile_start[t] + h[t];
            __syncthreads();
        }
        for (int b = 0; b < kSeg && r0 + b < V; b += 32) {
            if (tid < 32) load_batch_warp0(B, r0 + b + lane, V, colmask, rowmask, gids, box, lane);
            __syncthreads();
            const int bw = box[1] - box[0] + 1;
            const int area = bw > 0 ? bw * (box[3] - box[2] + 1) : 0;
            for (int i = tid; i < area; i += kBinThreads) {
                const int q = i / bw;
                const int ty = box[2] + q, tx = box[0] + (i - q * bw);
                uint32_t m = colmask[tx] & rowmask[ty];
                if (!m) continue;
                const int t = ty * B.tiles_x + tx;
                if (is_done(done, t)) continue;
                uint32_t c = cur[t];
                cur[t] = c + (uint32_t)__popc(m);
                if (staged) {
                    while (m) {
                        const int j = __ffs(m) - 1;
                        m &= m - 1u;
                        buf_t[c] = (uint16_t)t;
                        buf_r[c] = (uint8_t)(b + j);
                        ++c;
                    }
                } else {
                    while (m) {
                        const int j = __ffs(m) - 1;
                        m &= m - 1u;
                        B.vals[c++] = gids[j];
                    }
                }
            }
            __syncthreads();
        }
        if (staged)
            for (uint32_t i = tid; i < total; i += kBinThreads) B.vals[delta[buf_t[i]] + i] = seg_g[buf_r[i]];
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Segment-parallel binning (default).  One CTA of kSeg threads per segment of
// kSeg ranks (CTAs stride over the chunk's segments); warp w builds the column /
// row ballot masks of batch w (ranks 32w..32w+31), all batches at once.  Each
// thread then owns tiles t = tid, tid + kSeg, ...: the coverers of tile t in
// batch b are the bits of colm[b][tx] & rowm[b][ty], in rank order, so a thread
// emits its tiles' complete runs for the segment with no cursor shared across
// threads and no barrier between batches.
//   count: hist[segment][t] = sum_b popc(...)            (coalesced row store)
//   emit:  runs are laid out in a shared-memory buffer (thread-major order, a
//          block scan of the per-thread totals), then flushed with consecutive
//          threads writing consecutive list entries.  Over capacity: direct.
// ---------------------------------------------------------------------------
constexpr int kSegThreads = kSeg;
constexpr int kSegBatches = kSeg / 32;

struct SegSmem {
    uint32_t* done;
    uint32_t* colm;  // [kSegBatches][tiles_x]
    uint32_t* rowm;  // [kSegBatches][tiles_y]
    uint32_t* seg_g; // [kSeg]
};

__device__ __forceinline__ size_t seg_fixed_words(const BinK& B) {
    return (size_t)((B.ntiles + 31) >> 5) + (size_t)kSegBatches * (B.tiles_x + B.tiles_y) + kSeg;
}

__device__ __forceinline__ SegSmem seg_smem(const BinK& B, uint32_t* smem) {
    SegSmem m;
    m.done = smem;
    m.colm = m.done + ((B.ntiles + 31) >> 5);
    m.rowm = m.colm + kSegBatches * B.tiles_x;
    m.seg_g = m.rowm + kSegBatches * B.tiles_y;
    return m;
}

// Load the segment's ranks and build every batch's masks (ends with a barrier).
__device__ __forceinline__ void seg_masks(const BinK& B, const SegSmem& m, int r0, int V) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int tx0 = 1, tx1 = 0, ty0 = 1, ty1 = 0;
    uint32_t g = 0;
    const int r = r0 + tid;
    if (r < V) {
        g = sorted_at(B.sorted_gidx, B.ties, r, V);
        const uint2 rc = B.rect[g];
        const int x0 = rc.x & 0xffff, x1 = rc.x >> 16, y0 = rc.y & 0xffff, y1 = rc.y >> 16;
        tx0 = x0 / B.ts;
        tx1 = (x1 - 1) / B.ts;
        ty0 = y0 / B.ts;
        ty1 = (y1 - 1) / B.ts;
    }
    m.seg_g[tid] = g;
    for (int i = tid; i < kSegBatches * (B.tiles_x + B.tiles_y); i += kSegThreads) m.colm[i] = 0u;  // colm, rowm
    __syncthreads();
    const bool valid = tx0 <= tx1 && ty0 <= ty1;
    const int ux0 = __reduce_min_sync(0xffffffffu, valid ? tx0 : 0x7fffffff);
    const int ux1 = __reduce_max_sync(0xffffffffu, valid ? tx1 : -1);
    const int uy0 = __reduce_min_sync(0xffffffffu, valid ? ty0 : 0x7fffffff);
    const int uy1 = __reduce_max_sync(0xffffffffu, valid ? ty1 : -1);
    uint32_t* cm = m.colm + warp * B.tiles_x;
    uint32_t* rm = m.rowm + warp * B.tiles_y;
    for (int tx = ux0; tx <= ux1; ++tx) {
        const uint32_t b = __ballot_sync(0xffffffffu, valid && tx0 <= tx && tx <= tx1);
        if (lane == 0) cm[tx] = b;
    }
    for (int ty = uy0; ty <= uy1; ++ty) {
        const uint32_t b = __ballot_sync(0xffffffffu, valid && ty0 <= ty && ty <= ty1);
        if (lane == 0) rm[ty] = b;
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t tile_count(const BinK& B, const SegSmem& m, int tx, int ty) {
    uint32_t c = 0;
#pragma unroll
    for (int b = 0; b < kSegBatches; ++b) c += __popc(m.colm[b * B.tiles_x + tx] & m.rowm[b * B.tiles_y + ty]);
    return c;
}

__global__ void __launch_bounds__(kSegThreads) k_bin_count_seg(BinK B) {
    extern __shared__ uint32_t smem[];
    if (!chunk_live(B)) return;
    const SegSmem m = seg_smem(B, smem);
    stage_done(B, m.done);
    const int V = *B.n_visible;
    for (int segl = blockIdx.x; segl < B.nseg; segl += gridDim.x) {
        const int r0 = (B.seg0 + segl) * kSeg;
        uint32_t* h = B.hist + (size_t)segl * B.ntiles;
        if (r0 >= V) {  // uniform
            for (int t = threadIdx.x; t < B.ntiles; t += kSegThreads) h[t] = 0u;
            continue;
        }
        seg_masks(B, m, r0, V);
        for (int t = threadIdx.x; t < B.ntiles; t += kSegThreads) {
            const int ty = t / B.tiles_x, tx = t - ty * B.tiles_x;
            h[t] = is_done(m.done, t) ? 0u : tile_count(B, m, tx, ty);
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kSegThreads) k_bin_emit_seg(BinK B, int cap) {
    extern __shared__ uint32_t smem[];
    __shared__ uint32_t s_wsum[kSegThreads / 32];
    if (!chunk_live(B)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nt = B.ntiles;
    const SegSmem m = seg_smem(B, smem);
    uint32_t* delta = m.seg_g + kSeg;  // [ntiles] global list position - buffer position
    uint16_t* buf_t = reinterpret_cast<uint16_t*>(delta + nt);
    uint8_t* buf_r = reinterpret_cast<uint8_t*>(buf_t + cap);
    stage_done(B, m.done);
    const int V = *B.n_visible;
    for (int segl = blockIdx.x; segl < B.nseg; segl += gridDim.x) {
        const int r0 = (B.seg0 + segl) * kSeg;
        if (r0 >= V) break;  // uniform; later segments of this CTA are past V too
        const uint32_t* h = B.hist + (size_t)segl * nt;
        seg_masks(B, m, r0, V);
        // this thread's entry total -> its buffer base (block exclusive scan)
        uint32_t mine = 0;
        for (int t = tid; t < nt; t += kSegThreads) {
            const int ty = t / B.tiles_x, tx = t - ty * B.tiles_x;
            if (!is_done(m.done, t)) mine += tile_count(B, m, tx, ty);
        }
        uint32_t inc = mine;
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += u;
        }
        if (lane == 31) s_wsum[warp] = inc;
        __syncthreads();
        uint32_t c = inc - mine, total = 0;
#pragma unroll
        for (int w = 0; w < kSegThreads / 32; ++w) {
            const uint32_t v = s_wsum[w];
            c += w < warp ? v : 0u;
            total += v;
        }
        const bool staged = total <= (uint32_t)cap;
        for (int t = tid; t < nt; t += kSegThreads) {
            if (is_done(m.done, t)) continue;
            const int ty = t / B.tiles_x, tx = t - ty * B.tiles_x;
            uint32_t gpos = B.tile_start[t] + h[t];
            if (staged) delta[t] = gpos - c;
#pragma unroll
            for (int b = 0; b < kSegBatches; ++b) {
                uint32_t mm = m.colm[b * B.tiles_x + tx] & m.rowm[b * B.tiles_y + ty];
                while (mm) {
                    const int j = __ffs(mm) - 1;
                    mm &= mm - 1u;
                    if (staged) {
                        buf_t[c] = (uint16_t)t;
                        buf_r[c] = (uint8_t)(b * 32 + j);
                        ++c;
                    } else {
                        B.vals[gpos++] = m.seg_g[b * 32 + j];
                    }
                }
            }
        }
        __syncthreads();
        if (staged)
            for (uint32_t i = tid; i < total; i += kSegThreads) B.vals[delta[buf_t[i]] + i] = m.seg_g[buf_r[i]];
        __syncthreads();
    }
}

// Graph gate of a depth chunk (c >= 1): the chunk's conditional node runs its
// binning + raster body only when the chunk is live; a dead chunk's ranges are
// written here exactly as k_bin_scan_tiles would (empty, every tile skipped).
__global__ void k_chunk_gate(BinK B, cudaGraphConditionalHandle h, int32_t* body_launches, int nkern) {
    const bool live = chunk_live(B);
    if (threadIdx.x == 0) {
        cudaGraphSetConditional(h, live ? 1u : 0u);
        if (live) atomicAdd(body_launches, nkern);
    }
    if (live) return;
    const uint32_t base = *B.list_off;
    for (int t = threadIdx.x; t < B.ntiles; t += blockDim.x) {
        const uint32_t cum = B.chunk == 0 ? 0u : B.prev_ranges[t].z + B.prev_ranges[t].y;
        B.ranges[t] = make_uint4(base, 0u, cum, 1u);
    }
}

void launch_chunk_gate(const BinK& B, cudaGraphConditionalHandle h, int32_t* body_launches, cudaStream_t st) {
    k_chunk_gate<<<1, 1024, 0, st>>>(B, h, body_launches, bin_chunk_kernels(B) + 1);
}

int bin_chunk_kernels(const BinK& B) { return B.nseg <= 0 ? 0 : (B.nseg <= 64 ? 3 : 4); }

// Kernel attributes (outside any stream capture: called when a pass is created).
void bin_init() {
    static bool attr = false;
    if (!attr) {
        const int mx = 200 * 1024;
        cudaFuncSetAttribute(k_bin_count<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_bin_count<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_bin_emit<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_bin_emit<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_bin_count_seg, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_bin_emit_seg, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        attr = true;
    }
}

namespace {
struct BinPlan {
    bool seg;            // segment kernels (else batch-walk kernels with global cursors)
    size_t seg_fixed, seg_emit, base, cnt_smem;
    bool cnt_sm;
    int cap;
};
BinPlan bin_plan(const BinK& B) {
    BinPlan P;
    P.seg_fixed = sizeof(uint32_t) * ((size_t)((B.ntiles + 31) >> 5) + (size_t)kSegBatches * (B.tiles_x + B.tiles_y) +
                                      kSeg);
    P.cap = B.ntiles <= 2048 ? 6144 : 16384;
    P.seg_emit = P.seg_fixed + sizeof(uint32_t) * (size_t)B.ntiles + 3 * (size_t)P.cap + 16;
    P.seg = P.seg_emit <= 200 * 1024 && B.ntiles <= 65535;
    P.base = sizeof(uint32_t) * (size_t)((B.ntiles + 31) / 32 + 32 + B.tiles_x + B.tiles_y);
    P.cnt_sm = B.ntiles <= kSmemTiles;
    P.cnt_smem = P.base + (P.cnt_sm ? sizeof(uint32_t) * (size_t)B.ntiles : 0);
    return P;
}
}  // namespace

void launch_bin_count(const BinK& B, cudaStream_t st) {
    const BinPlan P = bin_plan(B);
    if (P.seg) {
        k_bin_count_seg<<<std::min(B.nseg, 148 * 12), kSegThreads, P.seg_fixed, st>>>(B);
    } else if (P.cnt_sm) {
        k_bin_count<true><<<std::min(B.nseg, 148 * 8), kBinThreads, P.cnt_smem, st>>>(B);
    } else {
        k_bin_count<false><<<std::min(B.nseg, 148 * 8), kBinThreads, P.cnt_smem, st>>>(B);
    }
}

void launch_bin_scan(const BinK& B, cudaStream_t st) {
    if (B.nseg <= 64) {  // small depth chunk: one block does both scans
        k_bin_scan_tiles<true><<<1, 1024, 0, st>>>(B);
        return;
    }
    k_bin_scan_segments<<<(B.ntiles + 31) / 32, 1024, 0, st>>>(B);
    k_bin_scan_tiles<false><<<1, 1024, 0, st>>>(B);
}

void launch_bin_emit(const BinK& B, cudaStream_t st) {
    const BinPlan P = bin_plan(B);
    if (P.seg)
        k_bin_emit_seg<<<std::min(B.nseg, 148 * 8), kSegThreads, P.seg_emit, st>>>(B, P.cap);
    else  // very large tile grids: batch walk with global cursors (hist row, in place)
        k_bin_emit<false><<<std::min(B.nseg, 148 * 8), kBinThreads, P.base, st>>>(B, 0);
}

}  // namespace tsb
