// The global (depth, index) order on read (splat.cpp:181-184).  The depth sort orders
// Gaussians by 24-bit compressed fp32 depth keys (stable, so equal keys stay in index
// order); a run of equal keys must still be ordered by the fp64 depth.  Instead of a
// separate pass over every rank, the readers of the order (the binning kernels, the
// fix-up's rank scan, the debug copy) resolve a rank that sits in a run on the fly:
// they sort the run's Gaussians -- at most kMaxTieRun, in registers -- and take their
// own position.  A longer run raises bit 1 of the frame's abort word; the host then
// redoes the frame with the exact 64-bit sort.  Runs the frame never reads (behind the
// termination of every tile) cost nothing.
#pragma once

#include "tsb_internal.h"

namespace tsb {

constexpr int kMaxTieRun = 8;

static __device__ __forceinline__ uint32_t sorted_in_run(const uint32_t* __restrict__ sorted, const TieK& T, int r, int V,
                                               uint32_t k) {
    int s = r;
    while (s > 0 && T.keys[s - 1] == k && r - s < kMaxTieRun) --s;
    int e = r + 1;
    while (e < V && T.keys[e] == k && e - s <= kMaxTieRun) ++e;
    const int L = e - s;
    if (L > kMaxTieRun || (s > 0 && T.keys[s - 1] == k)) {
        atomicOr(T.abort, 2);  // long run: the frame is redone with the exact sort
        return sorted[r];
    }
    uint32_t g[kMaxTieRun];
    double d[kMaxTieRun];
#pragma unroll
    for (int i = 0; i < kMaxTieRun; ++i) {
        g[i] = i < L ? sorted[s + i] : 0xffffffffu;
        d[i] = i < L ? T.depth64[g[i]] : __longlong_as_double(0x7ff0000000000000ll);  // +inf sorts last
    }
    // odd-even transposition network: kMaxTieRun rounds sort any L <= kMaxTieRun
#pragma unroll
    for (int round = 0; round < kMaxTieRun; ++round) {
#pragma unroll
        for (int i = round & 1; i + 1 < kMaxTieRun; i += 2) {
            const bool sw = d[i] > d[i + 1] || (d[i] == d[i + 1] && g[i] > g[i + 1]);
            const double dt = sw ? d[i + 1] : d[i], du = sw ? d[i] : d[i + 1];
            const uint32_t gt = sw ? g[i + 1] : g[i], gu = sw ? g[i] : g[i + 1];
            d[i] = dt; d[i + 1] = du; g[i] = gt; g[i + 1] = gu;
        }
    }
    uint32_t out = g[0];
#pragma unroll
    for (int i = 1; i < kMaxTieRun; ++i)
        if (i == r - s) out = g[i];
    return out;
}

// Gaussian at rank r (< V) of the exact (depth, index) order.
__device__ __forceinline__ uint32_t sorted_at(const uint32_t* __restrict__ sorted, const TieK& T, int r, int V) {
    if (!T.keys) return sorted[r];  // the exact 64-bit order: no runs to resolve
    const uint32_t k = T.keys[r];
    const bool prev = r > 0 && T.keys[r - 1] == k;
    const bool next = r + 1 < V && T.keys[r + 1] == k;
    if (!prev && !next) return sorted[r];
    return sorted_in_run(sorted, T, r, V, k);
}

}  // namespace tsb
