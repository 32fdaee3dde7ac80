// Tile binning: global (depth, index) order -> per-tile lists in that order.
// Replaces the reference's std::sort of Prepared structs (splat.cpp:179-184)
// and build_tiles (splat.cpp:187-200).
//
//   1. depth sort: stable LSD radix sort of the fp64 depth bits (value = Gaussian
//      index, input in index order -> ties broken by index exactly as the
//      reference's comparator does).  The position in this order is the rank.
//   2. gather tiles-touched into rank order, exclusive scan -> key offsets.
//   3. duplicate: rank r writes (tile, gidx) for every tile of its rect, in rank
//      order (values are Gaussian indices; records stay Gaussian-indexed).
//   4. tile sort: stable radix sort of the 16-bit tile ids only (the emission
//      is already rank-ordered, so only ceil(log2 tiles) bits need sorting).
//   5. tile ranges [start, end) by boundary detection.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "tsb_internal.h"

namespace tsb {

size_t binning_temp_bytes(int n, int64_t k_cap) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (uint64_t*)nullptr, (uint64_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, n > 0 ? n : 1, 0, 64);
    cub::DeviceRadixSort::SortPairs(nullptr, b, (uint16_t*)nullptr, (uint16_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int)(k_cap > 0 ? k_cap : 1), 0, 16);
    cub::DeviceScan::ExclusiveSum(nullptr, c, (uint32_t*)nullptr, (uint32_t*)nullptr, n > 0 ? n : 1);
    size_t m = a > b ? a : b;
    return m > c ? m : c;
}

void launch_sort_depth(uint64_t* keys_in, uint64_t* keys_out, uint32_t* vals_in, uint32_t* vals_out, int n,
                       void* temp, size_t temp_bytes, cudaStream_t st) {
    if (n <= 0) return;
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, n, 0, 64, st);
}

__global__ void k_gather_counts(const uint32_t* __restrict__ sorted_gidx, const uint32_t* __restrict__ touched,
                                uint32_t* __restrict__ cnt_sorted, int n) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) cnt_sorted[r] = touched[sorted_gidx[r]];
}

void launch_gather_counts(const uint32_t* sorted_gidx, const uint32_t* touched, uint32_t* cnt_sorted, int n,
                          cudaStream_t st) {
    if (n <= 0) return;
    k_gather_counts<<<(n + 255) / 256, 256, 0, st>>>(sorted_gidx, touched, cnt_sorted, n);
}

void launch_scan(const uint32_t* in, uint32_t* out, int n, void* temp, size_t temp_bytes, cudaStream_t st) {
    if (n <= 0) return;
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, n, st);
}

__global__ void __launch_bounds__(256) k_duplicate(const uint32_t* __restrict__ sorted_gidx,
                                                   const uint32_t* __restrict__ offsets,
                                                   const uint32_t* __restrict__ cnt_sorted,
                                                   const uint2* __restrict__ rect,
                                                   uint16_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                   int n, int ts, int tiles_x) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    if (cnt_sorted[r] == 0) return;  // culled Gaussians sort to the end with 0 tiles
    const uint32_t g = sorted_gidx[r];
    const uint2 rc = rect[g];
    const int x0 = rc.x & 0xffff, x1 = rc.x >> 16, y0 = rc.y & 0xffff, y1 = rc.y >> 16;
    const int tx0 = x0 / ts, tx1 = (x1 - 1) / ts, ty0 = y0 / ts, ty1 = (y1 - 1) / ts;
    uint32_t o = offsets[r];
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
            keys[o] = (uint16_t)(ty * tiles_x + tx);
            vals[o] = g;
            ++o;
        }
}

void launch_duplicate(const uint32_t* sorted_gidx, const uint32_t* offsets, const uint32_t* cnt_sorted,
                      const uint2* rect, uint16_t* keys, uint32_t* vals, int n, int ts, int tiles_x,
                      cudaStream_t st) {
    if (n <= 0) return;
    k_duplicate<<<(n + 255) / 256, 256, 0, st>>>(sorted_gidx, offsets, cnt_sorted, rect, keys, vals, n, ts,
                                                 tiles_x);
}

void launch_sort_tiles(uint16_t* keys_in, uint16_t* keys_out, uint32_t* vals_in, uint32_t* vals_out, int64_t k,
                       int bits, void* temp, size_t temp_bytes, cudaStream_t st) {
    if (k <= 0) return;
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, (int)k, 0, bits, st);
}

__global__ void k_ranges(const uint16_t* __restrict__ keys, int64_t k, uint2* __restrict__ ranges) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    const uint32_t t = keys[i];
    if (i == 0 || keys[i - 1] != t) ranges[t].x = (uint32_t)i;
    if (i == k - 1 || keys[i + 1] != t) ranges[t].y = (uint32_t)(i + 1);
}

void launch_ranges(const uint16_t* keys, int64_t k, uint2* ranges, int ntiles, cudaStream_t st) {
    cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)ntiles, st);
    if (k <= 0) return;
    k_ranges<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(keys, k, ranges);
}

}  // namespace tsb
