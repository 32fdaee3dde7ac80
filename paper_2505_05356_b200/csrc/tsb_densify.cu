// Densification surgery on the device (trainer.cpp:385-470) and the Adam state
// reindex it implies (AdamState::reindex, trainer.cpp:33-47).
//
//   k_dens_classify  per Gaussian: transparent (sigmoid(logit) < opacity_floor),
//                    mean positional-gradient norm (densify statistic / count),
//                    largest scale;
//   exclusive scan   of the transparent flags: Gaussian i is pruned when it is
//                    transparent and fewer than n - min_count transparent ones precede
//                    it (the reference's sequential loop stops at the floor);
//   k_dens_decide    survivors with mean gradient > threshold split in two (largest
//                    scale > split_scale_fraction x scene extent) or clone; keep / extra
//                    counts;
//   exclusive scans  of keep flags and extra counts -> new slots: kept Gaussians in
//                    index order, then the extras in their parents' order (split
//                    children -1 then +1 along the parent's largest axis), as the
//                    reference assembles `np`;
//   k_dens_scatter   every parameter array (mean + opacity, log-scale + reflectivity,
//                    rotation, keyframe offsets, SH) and the Adam moments (copied for
//                    kept Gaussians, zero for new ones).
#include <cuda_runtime.h>

#include "tsb_fp64.cuh"
#include "tsb_internal.h"

namespace tsb {

namespace {
constexpr int kScanBlock = 1024;

__global__ void k_scan_blocks(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint32_t* __restrict__ sums,
                              int n) {
    __shared__ uint32_t ws[32];
    const int i = blockIdx.x * kScanBlock + threadIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t v = i < n ? in[i] : 0u;
    uint32_t inc = v;
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += u;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
        uint32_t s = ws[lane], si = s;
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, si, d);
            if (lane >= d) si += u;
        }
        ws[lane] = si - s;
        if (lane == 31) sums[blockIdx.x] = si;
    }
    __syncthreads();
    if (i < n) out[i] = ws[w] + inc - v;
}

__global__ void k_scan_sums(uint32_t* __restrict__ sums, int nb, uint32_t* __restrict__ total) {
    if (threadIdx.x != 0) return;
    uint32_t run = 0;
    for (int b = 0; b < nb; ++b) {
        const uint32_t v = sums[b];
        sums[b] = run;
        run += v;
    }
    *total = run;
}

__global__ void k_scan_add(uint32_t* __restrict__ out, const uint32_t* __restrict__ sums, int n) {
    const int i = blockIdx.x * kScanBlock + threadIdx.x;
    if (i < n) out[i] += sums[blockIdx.x];
}

// exclusive scan of n counts; *total = sum.  tmp: >= ceil(n / 1024) words.
void exclusive_scan(const uint32_t* in, uint32_t* out, int n, uint32_t* tmp, uint32_t* total, cudaStream_t st) {
    const int nb = std::max(1, (n + kScanBlock - 1) / kScanBlock);
    k_scan_blocks<<<nb, kScanBlock, 0, st>>>(in, out, tmp, n);
    k_scan_sums<<<1, 32, 0, st>>>(tmp, nb, total);
    k_scan_add<<<nb, kScanBlock, 0, st>>>(out, tmp, n);
}

__global__ void k_dens_transparent(SceneK S, double floor_op, uint32_t* __restrict__ transparent) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S.n) return;
    transparent[i] = opacity64(S, i) < floor_op ? 1u : 0u;
}

// decision: 0 keep, 1 clone (keep + 1 extra), 2 split (drop + 2 extras), 3 pruned
__global__ void k_dens_decide(SceneK S, DensifyK D, const uint32_t* __restrict__ tprefix,
                              const uint32_t* __restrict__ transparent, uint32_t* __restrict__ keep,
                              uint32_t* __restrict__ extra, uint8_t* __restrict__ decision) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S.n) return;
    uint8_t dec = 0;
    if (transparent[i] && (int64_t)tprefix[i] < (int64_t)S.n - D.min_count) {
        dec = 3;
    } else if (D.count > 0) {
        const double mean_grad = (double)D.grad_sum[i] / (double)D.count;
        if (mean_grad > D.grad_threshold) {
            const float4 sa = S.scale_amp[i];
            const double max_scale = fmax(exp((double)sa.x), fmax(exp((double)sa.y), exp((double)sa.z)));
            dec = max_scale > D.split_scale ? 2 : 1;
        }
    }
    decision[i] = dec;
    keep[i] = (dec == 0 || dec == 1) ? 1u : 0u;
    extra[i] = dec == 2 ? 2u : (dec == 1 ? 1u : 0u);
}

// new[slot] <- old[i] for every float4 array a (params, m, v) and the extras.
__global__ void k_dens_scatter(SceneK S, DensifyK D, const uint8_t* __restrict__ decision,
                               const uint32_t* __restrict__ kpos, const uint32_t* __restrict__ epos,
                               uint32_t n_kept, int narrays, const float4* __restrict__ P, const float4* __restrict__ M,
                               const float4* __restrict__ V, float4* __restrict__ P2, float4* __restrict__ M2,
                               float4* __restrict__ V2, int n_new) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S.n) return;
    const uint8_t dec = decision[i];
    const size_t n = (size_t)S.n, nn = (size_t)n_new;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (dec == 0 || dec == 1) {
        const size_t j = kpos[i];
        for (int a = 0; a < narrays; ++a) {
            P2[a * nn + j] = P[a * n + i];
            M2[a * nn + j] = M[a * n + i];
            V2[a * nn + j] = V[a * n + i];
        }
    }
    if (dec == 1) {  // clone in place (trainer.cpp:431-439)
        const size_t j = n_kept + epos[i];
        for (int a = 0; a < narrays; ++a) {
            P2[a * nn + j] = P[a * n + i];
            M2[a * nn + j] = z4;
            V2[a * nn + j] = z4;
        }
    } else if (dec == 2) {  // split along the largest axis (trainer.cpp:413-429)
        const float4 po = S.pos_op[i], sa = S.scale_amp[i], qf = S.quat[i];
        const double ls[3] = {sa.x, sa.y, sa.z};
        int axis = 0;
        for (int c = 1; c < 3; ++c)
            if (ls[c] > ls[axis]) axis = c;  // Eigen maxCoeff: first maximum
        const double max_scale = fmax(exp(ls[0]), fmax(exp(ls[1]), exp(ls[2])));
        const double q[4] = {qf.x, qf.y, qf.z, qf.w};
        double u[4], R[9];
        quat_rot(q, u, R);
        const double d[3] = {R[0 * 3 + axis] * 0.25 * max_scale, R[1 * 3 + axis] * 0.25 * max_scale,
                             R[2 * 3 + axis] * 0.25 * max_scale};
        const double lshrink = log(D.split_shrink);
        for (int k = 0; k < 2; ++k) {
            const double sgn = k == 0 ? -1.0 : 1.0;
            const size_t j = n_kept + epos[i] + k;
            for (int a = 0; a < narrays; ++a) {
                P2[a * nn + j] = P[a * n + i];
                M2[a * nn + j] = z4;
                V2[a * nn + j] = z4;
            }
            P2[j] = make_float4((float)((double)po.x + sgn * d[0]), (float)((double)po.y + sgn * d[1]),
                                (float)((double)po.z + sgn * d[2]), po.w);
            P2[nn + j] = make_float4((float)(ls[0] - lshrink), (float)(ls[1] - lshrink), (float)(ls[2] - lshrink),
                                     sa.w);
        }
    }
}
}  // namespace

// Phase 1: decisions and counts; returns (via *counts) n_kept and n_extra.
void launch_densify_plan(const SceneK& S, const DensifyK& D, DensifyScratch& w, cudaStream_t st) {
    const int n = S.n;
    if (n <= 0) {
        cudaMemsetAsync(w.totals, 0, 3 * sizeof(uint32_t), st);
        return;
    }
    const int bs = 256, g = (n + bs - 1) / bs;
    k_dens_transparent<<<g, bs, 0, st>>>(S, D.opacity_floor, w.transparent);
    exclusive_scan(w.transparent, w.tprefix, n, w.scan_tmp, w.totals + 2, st);
    k_dens_decide<<<g, bs, 0, st>>>(S, D, w.tprefix, w.transparent, w.keep, w.extra, w.decision);
    exclusive_scan(w.keep, w.kpos, n, w.scan_tmp, w.totals + 0, st);
    exclusive_scan(w.extra, w.epos, n, w.scan_tmp, w.totals + 1, st);
}

void launch_densify_scatter(const SceneK& S, const DensifyK& D, const DensifyScratch& w, uint32_t n_kept, int narrays,
                            const float4* P, const float4* M, const float4* V, float4* P2, float4* M2, float4* V2,
                            int n_new, cudaStream_t st) {
    if (S.n <= 0) return;
    const int bs = 128, g = (S.n + bs - 1) / bs;
    k_dens_scatter<<<g, bs, 0, st>>>(S, D, w.decision, w.kpos, w.epos, n_kept, narrays, P, M, V, P2, M2, V2, n_new);
}

}  // namespace tsb
