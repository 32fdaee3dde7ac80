// Hand-written stable LSD radix sort (Onesweep: one kernel per 8-bit digit pass
// with decoupled look-back) of 32-bit keys with 32-bit values.  Used for the
// global (depth, index) order: keys are fp32 depth bits, values Gaussian indices
// in index order, so stability gives the reference's index tie-break
// (splat.cpp:181-184).
//
//   k_sort_hist      one pass over the keys: histograms of all four digits
//                    (warp-aggregated shared-memory atomics), into global.
//   k_sort_scan      exclusive scan of each digit histogram -> digit offsets.
//   k_onesweep       per pass: a CTA takes the next tile (atomic ticket, so
//                    earlier tiles are always running -> forward progress),
//                    ranks its 2048 items stably (warp-striped slots, match_any
//                    peers, per-warp digit counters), publishes its per-digit
//                    counts, looks back over earlier tiles' published counts /
//                    inclusive prefixes, stages the tile in shared memory in
//                    digit order and writes it out with consecutive threads
//                    writing consecutive positions of each digit run.
#include <cuda_runtime.h>

#include "tsb_internal.h"

namespace tsb {

namespace {
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortIPT = 16;
constexpr int kSortTile = kSortThreads * kSortIPT;  // 4096 items
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kCountMask = (1u << 30) - 1u;

// Lanes holding the same 8-bit digit, from 8 ballots (cheaper than match.any).
__device__ __forceinline__ unsigned peers8(uint32_t d, bool valid) {
    unsigned m = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const unsigned bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        m &= ((d >> b) & 1u) ? bb : ~bb;
    }
    return valid ? m : 0u;
}
}  // namespace

// All four digit histograms in one pass.  Per-warp sub-histograms; the lanes that
// share lane 0's digit (the common case for the high, low-entropy digits) are
// counted with one atomic by lane 0, the others add their own.
// Keys are compressed to 24 bits: k' = (k - kmin) >> shift (< 0xffffff), with kmin and
// shift from the key range the preprocess recorded (range[0] = min, range[1] = max of
// the keys that are not 0xffffffff).  Culled keys (0xffffffff) map to 0xffffff.
__device__ __forceinline__ void key_xform(const uint32_t* range, uint32_t& kmin, uint32_t& shift) {
    kmin = range[0];
    const uint32_t span = range[1] >= range[0] ? range[1] - range[0] : 0u;
    const int bits = span ? 32 - __clz(span) : 0;
    shift = bits > 24 ? (uint32_t)(bits - 24) : 0u;
    if ((span >> shift) >= 0xffffffu) ++shift;  // visible keys stay below the culled sentinel
}
__device__ __forceinline__ uint32_t key24(uint32_t k, uint32_t kmin, uint32_t shift) {
    return k == 0xffffffffu ? 0xffffffu : ((k - kmin) >> shift);
}

// TOP_ONLY (the prefix sort's selection): the top digit's histogram alone.
template <bool TOP_ONLY>
__global__ void __launch_bounds__(kSortThreads) k_sort_hist(const uint32_t* __restrict__ keys, int n,
                                                            uint32_t* __restrict__ hist /* [3][256] */,
                                                            uint32_t* __restrict__ status, int status_words,
                                                            const uint32_t* __restrict__ range) {
    uint32_t kmin, kshift;
    key_xform(range, kmin, kshift);
    __shared__ uint32_t h[kSortWarps][3][256];
    // clear the look-back status words of all four passes (used only after this kernel)
    for (int i = blockIdx.x * kSortThreads + threadIdx.x; i < status_words; i += gridDim.x * kSortThreads)
        status[i] = 0u;
    for (int i = threadIdx.x; i < kSortWarps * 3 * 256; i += kSortThreads) (&h[0][0][0])[i] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n4 = n >> 2;
    const uint4* k4 = reinterpret_cast<const uint4*>(keys);
    for (int i = blockIdx.x * kSortThreads + threadIdx.x; i - (int)threadIdx.x < n4 + 1;
         i += gridDim.x * kSortThreads) {
        uint32_t kk[4];
        bool valid[4];
        if (i < n4) {
            const uint4 q = k4[i];
            kk[0] = q.x; kk[1] = q.y; kk[2] = q.z; kk[3] = q.w;
            valid[0] = valid[1] = valid[2] = valid[3] = true;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int idx = 4 * n4 + 4 * (i - n4) + j;
                valid[j] = i >= n4 && (i - n4) == 0 && idx < n;
                kk[j] = valid[j] ? keys[idx] : 0u;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) kk[j] = key24(kk[j], kmin, kshift);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int p = TOP_ONLY ? 2 : 0; p < 3; ++p) {
                const uint32_t d = (kk[j] >> (8 * p)) & 255u;
                const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
                const bool v0 = __shfl_sync(0xffffffffu, valid[j], 0);
                const unsigned same = __ballot_sync(0xffffffffu, valid[j] && v0 && d == d0);
                if (lane == 0 && same) atomicAdd(&h[warp][p][d0], (uint32_t)__popc(same));
                else if (valid[j] && !((same >> lane) & 1u)) atomicAdd(&h[warp][p][d], 1u);
            }
        }
    }
    __syncthreads();
    for (int i = TOP_ONLY ? 2 * 256 + threadIdx.x : threadIdx.x; i < 3 * 256; i += kSortThreads) {
        uint32_t v = 0;
        for (int w = 0; w < kSortWarps; ++w) v += (&h[w][0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

__global__ void k_sort_scan(uint32_t* __restrict__ hist /* in: counts, out: exclusive offsets */) {
    // one warp per digit pass; each lane owns 8 consecutive bins
    const int p = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* h = hist + 256 * p;
    uint32_t v[8], s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        v[j] = h[lane * 8 + j];
        s += v[j];
    }
    uint32_t inc = s;
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += u;
    }
    uint32_t run = inc - s;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        h[lane * 8 + j] = run;
        run += v[j];
    }
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) { return *(const volatile uint32_t*)p; }

__global__ void __launch_bounds__(kSortThreads, 3) k_onesweep(const uint32_t* __restrict__ keys_in,
                                                           const uint32_t* __restrict__ vals_in,
                                                           uint32_t* __restrict__ keys_out,
                                                           uint32_t* __restrict__ vals_out, int n, int shift,
                                                           const uint32_t* __restrict__ digit_off,
                                                           uint32_t* status, uint32_t* tile_ticket,
                                                           const uint32_t* __restrict__ range,
                                                           const int32_t* __restrict__ n_dev) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t warp_cnt[kSortWarps][256];  // counts, then exclusive offsets across warps
    __shared__ uint32_t block_start[256];            // exclusive scan over digits of the tile counts
    __shared__ uint32_t global_base[256];
    __shared__ uint32_t s_keys[kSortTile];
    __shared__ uint32_t s_vals[kSortTile];
    __shared__ uint32_t s_wsum[kSortWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_ticket, 1u);
    for (int i = tid; i < kSortWarps * 256; i += kSortThreads) (&warp_cnt[0][0])[i] = 0u;
    __syncthreads();
    const int tile = (int)s_tile;
    const int base = tile * kSortTile;
    if (n_dev) {  // element count known on the device only: tiles past it have nothing to do
        n = *n_dev;
        if (base >= n) return;
    }

    // load warp-striped: slot i of lane l is item (warp*32*IPT + i*32 + l) of the tile
    uint32_t k[kSortIPT], v[kSortIPT], lr[kSortIPT];
#pragma unroll
    for (int i = 0; i < kSortIPT; ++i) {
        const int idx = base + warp * 32 * kSortIPT + i * 32 + lane;
        const bool valid = idx < n;
        k[i] = valid ? keys_in[idx] : 0u;
        v[i] = valid ? vals_in[idx] : 0u;
        lr[i] = valid ? 0u : 0xffffffffu;
    }
    if (range) {  // first pass: compress the raw fp32 keys to 24 bits
        uint32_t kmin, kshift;
        key_xform(range, kmin, kshift);
#pragma unroll
        for (int i = 0; i < kSortIPT; ++i) k[i] = key24(k[i], kmin, kshift);
    }
    // stable rank within the warp (slot order, then lane order == item order)
    const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < kSortIPT; ++i) {
        const bool valid = lr[i] == 0u;
        const uint32_t d = (k[i] >> shift) & 255u;
        const unsigned peers = peers8(d, valid);
        uint32_t cur = 0;
        if (valid) {
            cur = warp_cnt[warp][d];
            lr[i] = cur + (uint32_t)__popc(peers & lt_mask);
        }
        __syncwarp();
        if (valid && (peers & lt_mask) == 0u) warp_cnt[warp][d] = cur + (uint32_t)__popc(peers);
        __syncwarp();
    }
    __syncthreads();

    // per digit (thread d): exclusive offsets across warps, tile count, block scan
    const int d = tid;  // kSortThreads == 256 digits
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
        const uint32_t c = warp_cnt[w][d];
        warp_cnt[w][d] = total;
        total += c;
    }
    {
        uint32_t inc = total;
        for (int s = 1; s < 32; s <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, s);
            if (lane >= s) inc += u;
        }
        if (lane == 31) s_wsum[warp] = inc;
        __syncthreads();
        uint32_t woff = 0;
        for (int w = 0; w < warp; ++w) woff += s_wsum[w];
        block_start[d] = woff + inc - total;
    }
    // decoupled look-back for this digit's global offset
    uint32_t* st = status + (size_t)tile * 256;
    if (tile == 0) {
        atomicExch(&st[d], kFlagInc | total);
        global_base[d] = digit_off[d];
    } else {
        atomicExch(&st[d], kFlagAgg | total);
        // look back 8 predecessors per round trip: sum aggregates until an inclusive prefix
        uint32_t prefix = 0;
        int t = tile - 1;
        bool found = false;
        while (!found) {
            uint32_t sv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) sv[j] = t - j >= 0 ? ld_volatile(status + (size_t)(t - j) * 256 + d) : kFlagInc;
            int j = 0;
            for (; j < 8; ++j) {
                const uint32_t f = sv[j] & ~kCountMask;
                if (f == 0u) break;  // not published yet: re-poll from here
                prefix += sv[j] & kCountMask;
                if (f == kFlagInc) {
                    found = true;
                    break;
                }
            }
            t -= j;
        }
        atomicExch(&st[d], kFlagInc | (prefix + total));
        global_base[d] = digit_off[d] + prefix;
    }
    __syncthreads();

    // stage the tile in digit order
#pragma unroll
    for (int i = 0; i < kSortIPT; ++i) {
        if (lr[i] == 0xffffffffu) continue;
        const uint32_t dd = (k[i] >> shift) & 255u;
        const uint32_t pos = block_start[dd] + warp_cnt[warp][dd] + lr[i];
        s_keys[pos] = k[i];
        s_vals[pos] = v[i];
    }
    __syncthreads();
    const int count = min(kSortTile, n - base);
    for (int j = tid; j < count; j += kSortThreads) {
        const uint32_t key = s_keys[j];
        const uint32_t dd = (key >> shift) & 255u;
        const uint32_t o = global_base[dd] + (uint32_t)j - block_start[dd];
        keys_out[o] = key;
        vals_out[o] = s_vals[j];
    }
}

size_t radix_sort_scratch_words(int n) {
    const int tiles = (n + kSortTile - 1) / kSortTile;
    return (size_t)4 * 256 + 4 + (size_t)4 * tiles * 256;  // hist/offsets, tickets, status per pass
}

// 24-bit compressed keys, 3 passes; the output keys are the compressed keys (equal
// compressed keys stay in input order -- callers re-sort such runs exactly).
int radix_sort24(uint32_t* keys_a, uint32_t* keys_b, uint32_t* vals_a, uint32_t* vals_b, int n, uint32_t* scratch,
                 const uint32_t* range, cudaStream_t st) {
    if (n <= 0) return 0;
    const int tiles = (n + kSortTile - 1) / kSortTile;
    uint32_t* hist = scratch;
    uint32_t* tickets = scratch + 4 * 256;
    uint32_t* status = tickets + 4;
    cudaMemsetAsync(scratch, 0, sizeof(uint32_t) * (4 * 256 + 4), st);
    const int hgrid = max(1, min(148 * 2, (n / 4 + kSortThreads - 1) / kSortThreads));
    k_sort_hist<false><<<hgrid, kSortThreads, 0, st>>>(keys_a, n, hist, status, 3 * 256 * tiles, range);
    k_sort_scan<<<1, 96, 0, st>>>(hist);
    // 3 passes ping-pong a->b->a->b; finish in b, then the caller uses b
    k_onesweep<<<tiles, kSortThreads, 0, st>>>(keys_a, vals_a, keys_b, vals_b, n, 0, hist, status, tickets, range, nullptr);
    k_onesweep<<<tiles, kSortThreads, 0, st>>>(keys_b, vals_b, keys_a, vals_a, n, 8, hist + 256,
                                               status + (size_t)256 * tiles, tickets + 1, nullptr, nullptr);
    k_onesweep<<<tiles, kSortThreads, 0, st>>>(keys_a, vals_a, keys_b, vals_b, n, 16, hist + 512,
                                               status + (size_t)512 * tiles, tickets + 2, nullptr, nullptr);
    return 5;
}

// keys/vals: double buffers; result ends in (keys_b, vals_b) after 4 passes
// when the pass count is even it ends in *_a -- we always do 4 passes and
// return the buffer holding the result.
// Full 32-bit keys, 4 passes (exact 64-bit fallback uses two of these).  Result in (keys_a, vals_a).
__global__ void k_sort_hist32(const uint32_t* __restrict__ keys, int n, uint32_t* __restrict__ hist,
                              uint32_t* __restrict__ status, int status_words) {
    __shared__ uint32_t h[4][256];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < status_words; i += gridDim.x * blockDim.x) status[i] = 0u;
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&h[0][0])[i] = 0u;
    __syncthreads();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        for (int p = 0; p < 4; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 255u], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x)
        if ((&h[0][0])[i]) atomicAdd(&hist[i], (&h[0][0])[i]);
}

int radix_sort32(uint32_t* keys_a, uint32_t* keys_b, uint32_t* vals_a, uint32_t* vals_b, int n, uint32_t* scratch,
                 cudaStream_t st) {
    if (n <= 0) return 0;
    const int tiles = (n + kSortTile - 1) / kSortTile;
    uint32_t* hist = scratch;
    uint32_t* tickets = scratch + 4 * 256;
    uint32_t* status = tickets + 4;
    cudaMemsetAsync(scratch, 0, sizeof(uint32_t) * (4 * 256 + 4), st);
    k_sort_hist32<<<148 * 2, 256, 0, st>>>(keys_a, n, hist, status, 4 * 256 * tiles);
    k_sort_scan<<<1, 128, 0, st>>>(hist);
    uint32_t *ki = keys_a, *ko = keys_b, *vi = vals_a, *vo = vals_b;
    for (int p = 0; p < 4; ++p) {
        k_onesweep<<<tiles, kSortThreads, 0, st>>>(ki, vi, ko, vo, n, 8 * p, hist + 256 * p,
                                                   status + (size_t)p * 256 * tiles, tickets + p, nullptr, nullptr);
        uint32_t* t = ki; ki = ko; ko = t;
        t = vi; vi = vo; vo = t;
    }
    return 6;
}

// ---- Nearest-prefix depth order ----
// A frame reads the order only up to the rank where its last tile terminates; on
// dense scenes that is a few thousand of a million ranks.  The prefix sort orders
// only the Gaussians whose top key digit is at most b*, the largest digit whose
// cumulative visible count fits in `cap`: those are exactly ranks [0, n_bin) of the
// full order (equal compressed keys share their top digit, so no run is split).
// The readers treat n_bin as the end of the order; a pixel still alive there while
// n_bin < n_visible raises bit 3 of the abort word and the host redoes the frame
// with the full sort (the raw keys are left intact for that).
//
//   k_sort_hist       (shared with the full sort) digit histograms of all keys
//   k_prefix_select   one warp: b*, n_bin, the selection's top-digit histogram
//   k_prefix_compact  gathers the selection (warp-aggregated slots) + its low-digit
//                     histograms; clears the look-back status of the 3 passes
//   k_sort_scan, 3 x k_onesweep over the selection (count read on the device)
namespace {
constexpr int kPrefHistC = 0, kPrefTickets = 768, kPrefSel = 772, kPrefCount = 773, kPrefStatus = 776;
}

__global__ void k_prefix_select(const uint32_t* __restrict__ hist, int n, int cap,
                                const int32_t* __restrict__ n_visible, uint32_t* __restrict__ ps,
                                int32_t* __restrict__ n_bin, int32_t* __restrict__ abort_word) {
    const int lane = threadIdx.x;
    const int V = *n_visible;
    uint32_t v[8], s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int b = lane * 8 + j;
        v[j] = hist[512 + b] - (b == 255 ? (uint32_t)(n - V) : 0u);  // culled keys sit in digit 255
        s += v[j];
    }
    uint32_t inc = s;
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += u;
    }
    // digits whose inclusive cumulative count fits in cap (a prefix of the digits)
    uint32_t run = inc - s;
    int fit = 0;
    uint32_t fit_cum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        run += v[j];
        if (run <= (uint32_t)cap) {
            ++fit;
            fit_cum = run;
        }
    }
    int nfit = fit;
    for (int d = 16; d; d >>= 1) nfit += __shfl_xor_sync(0xffffffffu, nfit, d);
    uint32_t nb = fit_cum;  // the largest fitting cumulative count (lanes' values are monotone)
    for (int d = 16; d; d >>= 1) nb = max(nb, __shfl_xor_sync(0xffffffffu, nb, d));
    if (nfit == 0) nb = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int b = lane * 8 + j;
        ps[kPrefHistC + b] = 0u;
        ps[kPrefHistC + 256 + b] = 0u;
        ps[kPrefHistC + 512 + b] = b < nfit ? v[j] : 0u;
    }
    if (lane < 4) ps[kPrefTickets + lane] = 0u;
    if (lane == 0) {
        ps[kPrefSel] = (uint32_t)nfit;  // selected: top digit < nfit
        ps[kPrefCount] = 0u;
        *n_bin = (int32_t)nb;
        if (nb == 0 && V > 0) atomicOr(abort_word, 8);  // the nearest digit alone exceeds cap
    }
}

__global__ void __launch_bounds__(kSortThreads) k_prefix_compact(const uint32_t* __restrict__ keys, int n,
                                                                 const uint32_t* __restrict__ range,
                                                                 uint32_t* __restrict__ ps, int status_words,
                                                                 uint32_t* __restrict__ sel_keys,
                                                                 uint32_t* __restrict__ sel_vals) {
    uint32_t kmin, kshift;
    key_xform(range, kmin, kshift);
    for (int i = blockIdx.x * kSortThreads + threadIdx.x; i < status_words; i += gridDim.x * kSortThreads)
        ps[kPrefStatus + i] = 0u;
    const uint32_t nsel = ps[kPrefSel];
    uint32_t* hist = ps + kPrefHistC;
    uint32_t* count = ps + kPrefCount;
    __shared__ uint32_t s_wcnt[kSortWarps];
    __shared__ uint32_t s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int n4 = (n + 3) >> 2;
    const bool aligned_tail = (n & 3) == 0;
    const uint4* k4 = reinterpret_cast<const uint4*>(keys);
    for (int i = blockIdx.x * kSortThreads + threadIdx.x; i - (int)threadIdx.x < n4; i += gridDim.x * kSortThreads) {
        uint32_t kk[4];
        if (i < n4 && (aligned_tail || i + 1 < n4)) {
            const uint4 q = k4[i];
            kk[0] = q.x; kk[1] = q.y; kk[2] = q.z; kk[3] = q.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) kk[j] = i < n4 && 4 * i + j < n ? keys[4 * i + j] : 0xffffffffu;
        }
        uint32_t c[4];
        unsigned m[4];
        uint32_t wtot = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            c[j] = key24(kk[j], kmin, kshift);
            m[j] = __ballot_sync(0xffffffffu, kk[j] != 0xffffffffu && (c[j] >> 16) < nsel);
            wtot += (uint32_t)__popc(m[j]);
        }
        // one global slot reservation per block and iteration (a single counter word
        // cannot take one atomic per warp at this rate)
        if (lane == 0) s_wcnt[warp] = wtot;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int w = 0; w < kSortWarps; ++w) {
                const uint32_t v = s_wcnt[w];
                s_wcnt[w] = t;
                t += v;
            }
            s_base = t ? atomicAdd(count, t) : 0u;
        }
        __syncthreads();
        uint32_t slot = s_base + s_wcnt[warp];
        __syncthreads();  // s_wcnt / s_base are rewritten by the next iteration
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if ((m[j] >> lane) & 1u) {
                const uint32_t sl = slot + (uint32_t)__popc(m[j] & lt_mask);
                sel_keys[sl] = kk[j];
                sel_vals[sl] = (uint32_t)(4 * i + j);
                atomicAdd(&hist[c[j] & 255u], 1u);
                atomicAdd(&hist[256 + ((c[j] >> 8) & 255u)], 1u);
            }
            slot += (uint32_t)__popc(m[j]);
        }
    }
}

// A selection that fits one tile (the common prefix cap): all three 8-bit LSD passes in one
// CTA, in shared memory -- the same stable in-tile ranking as k_onesweep, with the tile's own
// digit scan as the offsets (no histograms, look-back or global round trips between passes;
// one launch instead of k_sort_scan + 3 x k_onesweep).
__global__ void __launch_bounds__(kSortThreads) k_sort_small(const uint32_t* __restrict__ keys_in,
                                                           const uint32_t* __restrict__ vals_in,
                                                           uint32_t* __restrict__ keys_out,
                                                           uint32_t* __restrict__ vals_out,
                                                           const uint32_t* __restrict__ range,
                                                           const int32_t* __restrict__ n_dev) {
    __shared__ uint32_t warp_cnt[kSortWarps][256];
    __shared__ uint32_t block_start[256];
    __shared__ uint32_t s_keys[kSortTile];
    __shared__ uint32_t s_vals[kSortTile];
    __shared__ uint32_t s_wsum[kSortWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = min(*n_dev, kSortTile);
    uint32_t kmin, kshift;
    key_xform(range, kmin, kshift);
    uint32_t k[kSortIPT], v[kSortIPT], lr[kSortIPT];
#pragma unroll
    for (int i = 0; i < kSortIPT; ++i) {
        const int idx = warp * 32 * kSortIPT + i * 32 + lane;
        const bool valid = idx < n;
        k[i] = valid ? key24(keys_in[idx], kmin, kshift) : 0u;
        v[i] = valid ? vals_in[idx] : 0u;
    }
    const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll 1
    for (int shift = 0; shift < 24; shift += 8) {
        for (int i = tid; i < kSortWarps * 256; i += kSortThreads) (&warp_cnt[0][0])[i] = 0u;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kSortIPT; ++i) {
            const int idx = warp * 32 * kSortIPT + i * 32 + lane;
            const bool valid = idx < n;
            const uint32_t d = (k[i] >> shift) & 255u;
            const unsigned peers = peers8(d, valid);
            uint32_t cur = 0;
            lr[i] = 0xffffffffu;
            if (valid) {
                cur = warp_cnt[warp][d];
                lr[i] = cur + (uint32_t)__popc(peers & lt_mask);
            }
            __syncwarp();
            if (valid && (peers & lt_mask) == 0u) warp_cnt[warp][d] = cur + (uint32_t)__popc(peers);
            __syncwarp();
        }
        __syncthreads();
        {  // per digit (thread d): exclusive offsets across warps, then the block scan
            const int d = tid;
            uint32_t total = 0;
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) {
                const uint32_t c = warp_cnt[w][d];
                warp_cnt[w][d] = total;
                total += c;
            }
            uint32_t inc = total;
            for (int s2 = 1; s2 < 32; s2 <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, inc, s2);
                if (lane >= s2) inc += u;
            }
            if (lane == 31) s_wsum[warp] = inc;
            __syncthreads();
            uint32_t woff = 0;
            for (int w = 0; w < warp; ++w) woff += s_wsum[w];
            block_start[d] = woff + inc - total;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kSortIPT; ++i) {
            if (lr[i] == 0xffffffffu) continue;
            const uint32_t dd = (k[i] >> shift) & 255u;
            const uint32_t pos = block_start[dd] + warp_cnt[warp][dd] + lr[i];
            s_keys[pos] = k[i];
            s_vals[pos] = v[i];
        }
        __syncthreads();
        if (shift < 16) {  // the next pass reads the tile in its new order
#pragma unroll
            for (int i = 0; i < kSortIPT; ++i) {
                const int idx = warp * 32 * kSortIPT + i * 32 + lane;
                k[i] = idx < n ? s_keys[idx] : 0u;
                v[i] = idx < n ? s_vals[idx] : 0u;
            }
            __syncthreads();  // (s_wsum / warp_cnt / the tile are rewritten by the next pass)
        }
    }
    for (int j = tid; j < n; j += kSortThreads) {
        keys_out[j] = s_keys[j];
        vals_out[j] = s_vals[j];
    }
}

size_t prefix_sort_scratch_words(int cap) {
    const int tiles = (cap + kSortTile - 1) / kSortTile;
    return (size_t)kPrefStatus + (size_t)3 * 256 * tiles;
}

int radix_sort24_prefix(const uint32_t* keys, uint32_t* keys_out, uint32_t* vals_out, uint32_t* tmp_keys,
                        uint32_t* tmp_vals, int n, int cap, uint32_t* scratch, uint32_t* ps, const uint32_t* range,
                        const int32_t* n_visible, int32_t* n_bin, int32_t* abort_word, cudaStream_t st) {
    if (n <= 0) return 0;
    const int ctiles = (cap + kSortTile - 1) / kSortTile;
    uint32_t* hist = scratch;
    cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 3 * 256, st);
    const int hgrid = max(1, min(148 * 2, (n / 4 + kSortThreads - 1) / kSortThreads));
    k_sort_hist<true><<<hgrid, kSortThreads, 0, st>>>(keys, n, hist, nullptr, 0, range);
    k_prefix_select<<<1, 32, 0, st>>>(hist, n, cap, n_visible, ps, n_bin, abort_word);
    k_prefix_compact<<<hgrid, kSortThreads, 0, st>>>(keys, n, range, ps, 3 * 256 * ctiles, tmp_keys, tmp_vals);
    if (ctiles == 1) {  // the whole selection in one tile: one kernel, three passes in shared memory
        k_sort_small<<<1, kSortThreads, 0, st>>>(tmp_keys, tmp_vals, keys_out, vals_out, range, n_bin);
        return 4;
    }
    uint32_t* hc = ps + kPrefHistC;
    uint32_t* tk = ps + kPrefTickets;
    uint32_t* status = ps + kPrefStatus;
    k_sort_scan<<<1, 96, 0, st>>>(hc);
    k_onesweep<<<ctiles, kSortThreads, 0, st>>>(tmp_keys, tmp_vals, keys_out, vals_out, cap, 0, hc, status, tk, range,
                                                n_bin);
    k_onesweep<<<ctiles, kSortThreads, 0, st>>>(keys_out, vals_out, tmp_keys, tmp_vals, cap, 8, hc + 256,
                                                status + (size_t)256 * ctiles, tk + 1, nullptr, n_bin);
    k_onesweep<<<ctiles, kSortThreads, 0, st>>>(tmp_keys, tmp_vals, keys_out, vals_out, cap, 16, hc + 512,
                                                status + (size_t)512 * ctiles, tk + 2, nullptr, n_bin);
    return 7;
}

}  // namespace tsb
