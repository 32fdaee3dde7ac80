// Parameter packing and the fused Adam step.
//
// Parameters, gradients and Adam moments share one layout: (3 + n_keyframes)
// float4 arrays of n Gaussians each, contiguous (see tsb_internal.h).  One
// thread per Gaussian walks every array (each access is a coalesced 16-B
// vector load across the warp), which lets the densification statistic
// (trainer.cpp:381-384) and the gradient clear ride along in the same pass.
#include <cuda_runtime.h>

#include <algorithm>

#include "tsb_internal.h"

namespace tsb {

// dst[i].comp[comp0 + c] = src[i*comps + c] for c < comps (AoS-3/4 -> float4 lanes).
__global__ void k_pack(float4* __restrict__ dst, const float* __restrict__ src, int n, int comps, int comp0) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float* d = reinterpret_cast<float*>(dst + i);
    for (int c = 0; c < comps; ++c) d[comp0 + c] = src[(size_t)i * comps + c];
}

__global__ void k_unpack(const float4* __restrict__ src, float* __restrict__ dst, int n, int comps, int comp0) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* s = reinterpret_cast<const float*>(src + i);
    for (int c = 0; c < comps; ++c) dst[(size_t)i * comps + c] = s[comp0 + c];
}

__global__ void k_pack_sh(float4* __restrict__ dst, float4* __restrict__ scale_amp, const float* __restrict__ src,
                          int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* s = src + (size_t)i * 16;
    scale_amp[i].w = s[0];
    for (int a = 0; a < 4; ++a) {
        const int k = 1 + 4 * a;
        dst[(size_t)a * n + i] = make_float4(s[k], s[k + 1], s[k + 2], a < 3 ? s[k + 3] : 0.f);
    }
}

__global__ void k_unpack_sh(const float4* __restrict__ src, float* __restrict__ dst, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float* d = dst + (size_t)i * 16;
    for (int a = 0; a < 4; ++a) {
        const float4 v = src[(size_t)a * n + i];
        const int k = 1 + 4 * a;
        d[k] = v.x;
        d[k + 1] = v.y;
        d[k + 2] = v.z;
        if (a < 3) d[k + 3] = v.w;
    }
}

// Rows of na * comps floats <-> na float4 arrays (lanes >= comps zero).
__global__ void k_pack_rows(float4* __restrict__ dst, const float* __restrict__ src, int n, int na, int comps) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* s = src + (size_t)i * na * comps;
    for (int a = 0; a < na; ++a) {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        for (int c = 0; c < comps; ++c) v[c] = s[a * comps + c];
        dst[(size_t)a * n + i] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

__global__ void k_unpack_rows(const float4* __restrict__ src, float* __restrict__ dst, int n, int na, int comps) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float* d = dst + (size_t)i * na * comps;
    for (int a = 0; a < na; ++a) {
        const float4 q = src[(size_t)a * n + i];
        const float v[4] = {q.x, q.y, q.z, q.w};
        for (int c = 0; c < comps; ++c) d[a * comps + c] = v[c];
    }
}

void launch_pack_rows(float4* dst, const float* src, int n, int na, int comps, cudaStream_t st) {
    if (n > 0) k_pack_rows<<<(n + 255) / 256, 256, 0, st>>>(dst, src, n, na, comps);
}
void launch_unpack_rows(const float4* src, float* dst, int n, int na, int comps, cudaStream_t st) {
    if (n > 0) k_unpack_rows<<<(n + 255) / 256, 256, 0, st>>>(src, dst, n, na, comps);
}

void launch_pack_sh(float4* dst4, float4* scale_amp, const float* src16, int n, cudaStream_t st) {
    if (n > 0) k_pack_sh<<<(n + 255) / 256, 256, 0, st>>>(dst4, scale_amp, src16, n);
}
void launch_unpack_sh(const float4* src4, float* dst16, int n, cudaStream_t st) {
    if (n > 0) k_unpack_sh<<<(n + 255) / 256, 256, 0, st>>>(src4, dst16, n);
}

void launch_pack_params(float4* dst, const float* src, int n, int comps, int comp0, int, cudaStream_t st) {
    if (n <= 0) return;
    k_pack<<<(n + 255) / 256, 256, 0, st>>>(dst, src, n, comps, comp0);
}

void launch_unpack(const float4* src, float* dst, int n, int comps, int comp0, cudaStream_t st) {
    if (n <= 0) return;
    k_unpack<<<(n + 255) / 256, 256, 0, st>>>(src, dst, n, comps, comp0);
}

struct LrTable {
    float lr_bc1[kMaxArrays * 4];  // lr / (1 - beta1^t) per array component (0 for padding)
};

// AdamState::step (trainer.cpp:18-31) for every group at once:
//   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;  p -= (lr/bc1) m / (sqrt(v/bc2) + eps)
__global__ void __launch_bounds__(256) k_adam(float4* __restrict__ P, float4* __restrict__ G,
                                              float4* __restrict__ M, float4* __restrict__ V, int n, int narrays,
                                              LrTable lr, float b1, float b2, float c1, float c2, float eps,
                                              float inv_bc2, float* __restrict__ densify) {
    // c1 = 1 - beta1, c2 = 1 - beta2 are formed in double on the host: 1 - fp32(0.999)
    // would carry a 1.3e-5 relative error into every second moment.
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int a = 0; a < narrays; ++a) {
        const size_t k = (size_t)a * n + i;
        const float4 g4 = G[k];
        if (a == 0 && densify) densify[i] += sqrtf(g4.x * g4.x + g4.y * g4.y + g4.z * g4.z);
        float4 p4 = P[k], m4 = M[k], v4 = V[k];
        float* p = &p4.x;
        float* m = &m4.x;
        float* v = &v4.x;
        const float* g = &g4.x;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            m[c] = b1 * m[c] + c1 * g[c];
            v[c] = b2 * v[c] + c2 * (g[c] * g[c]);
            p[c] -= lr.lr_bc1[a * 4 + c] * (m[c] / (sqrtf(v[c] * inv_bc2) + eps));
        }
        P[k] = p4;
        M[k] = m4;
        V[k] = v4;
        G[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

void launch_adam(float4* params, float4* grads, float4* m, float4* v, int n, int narrays, const double* lr4,
                 double beta1, double beta2, double eps, double bc1, double bc2, float* densify, cudaStream_t st) {
    if (n <= 0) return;
    LrTable t;
    for (int i = 0; i < kMaxArrays * 4; ++i) t.lr_bc1[i] = i < narrays * 4 ? (float)(lr4[i] / bc1) : 0.f;
    k_adam<<<(n + 255) / 256, 256, 0, st>>>(params, grads, m, v, n, narrays, t, (float)beta1, (float)beta2,
                                            (float)(1.0 - beta1), (float)(1.0 - beta2), (float)eps,
                                            (float)(1.0 / bc2), densify);
}

// AdamState::step on a flat vector (trainer.cpp:18-31).
__global__ void k_adam_flat(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, size_t n, float lr_bc1, float b1, float b2, float c1, float c2,
                            float eps, float inv_bc2) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const float gi = g[i];
        const float mi = b1 * m[i] + c1 * gi;
        const float vi = b2 * v[i] + c2 * (gi * gi);
        m[i] = mi;
        v[i] = vi;
        p[i] -= lr_bc1 * (mi / (sqrtf(vi * inv_bc2) + eps));
    }
}

void launch_adam_flat(float* p, const float* g, float* m, float* v, size_t n, double lr, double b1, double b2,
                      double eps, double bc1, double bc2, cudaStream_t st) {
    if (n == 0) return;
    const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 8);
    k_adam_flat<<<grid, 256, 0, st>>>(p, g, m, v, n, (float)(lr / bc1), (float)b1, (float)b2, (float)(1.0 - b1),
                                      (float)(1.0 - b2), (float)eps, (float)(1.0 / bc2));
}

// AdamState::reindex (trainer.cpp:33-47): moments of new slot i are those of old slot src[i]
// (stride values each), zero where src[i] < 0.
__global__ void k_adam_reindex(const float* __restrict__ m, const float* __restrict__ v, const int32_t* __restrict__ src,
                               size_t n_new, int stride, float* __restrict__ m2, float* __restrict__ v2) {
    const size_t total = n_new * (size_t)stride;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int s = src[i / stride];
        const size_t j = (size_t)s * stride + i % stride;
        m2[i] = s < 0 ? 0.f : m[j];
        v2[i] = s < 0 ? 0.f : v[j];
    }
}

void launch_adam_reindex(const float* m, const float* v, const int32_t* src, size_t n_new, int stride, float* m2,
                         float* v2, cudaStream_t st) {
    const size_t total = n_new * (size_t)stride;
    if (total == 0) return;
    const int grid = (int)std::min<size_t>((total + 255) / 256, 148 * 8);
    k_adam_reindex<<<grid, 256, 0, st>>>(m, v, src, n_new, stride, m2, v2);
}

}  // namespace tsb
