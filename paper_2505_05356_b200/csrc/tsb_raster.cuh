// fp32 splat evaluation shared by the raster kernels (tsb_raster.cu) and the
// colour / flow channel kernels (tsb_ext.cu): both must reproduce the forward's
// per-entry decisions bit for bit, so every operation is an explicit-rounding
// intrinsic (unaffected by -fmad).
#pragma once

#include <cuda_runtime.h>

namespace tsb {

constexpr float kNegHalfLog2e = -0.72134752044448170368f;  // -0.5 * log2(e)

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Same bits in the forward and backward kernels: every operation is pinned with
// an explicit-rounding intrinsic so the compiler cannot contract differently.
struct Eval {
    float dx, dy, p, q, maha, g, alpha;
};

// A (staged) = (mean.x - block origin, mean.y - block origin, error scale x, error scale y);
// (lx, ly) = pixel centre relative to the block origin (exact).
__device__ __forceinline__ void eval_entry(const float4& A, const float4& B, float lx, float ly, Eval& e) {
    e.dx = __fsub_rn(lx, A.x);
    e.dy = __fsub_rn(ly, A.y);
    e.p = __fmaf_rn(B.x, e.dx, __fmul_rn(B.y, e.dy));
    e.q = __fmul_rn(B.z, e.dy);
    e.maha = __fmaf_rn(e.p, e.p, __fmul_rn(e.q, e.q));
}
__device__ __forceinline__ void eval_alpha(const float4& B, Eval& e) {
    e.g = ex2_approx(__fmul_rn(e.maha, kNegHalfLog2e));
    e.alpha = __fmul_rn(B.w, e.g);
}

// Decision error bounds.  An evaluation whose maha
// or alpha lands within a coarse window of its threshold gets a first-order bound
// on its fp32 error (rare branch); the pixel is sent to the fp64 fix-up when the
// decision lies inside twice that bound.
constexpr float kEps = 5.9604645e-8f;      // 2^-24
constexpr float kEx2Err = 2.5e-7f;         // ex2.approx.ftz.f32 relative error bound (+ margin)

// |fl32(maha) - maha_exact| bound from the rounding of mean offsets (A.z, A.w carry
// |mean - rect origin| + |mean - block origin|), L, dx, dy, p, q.
__device__ __forceinline__ float maha_err_bound(const float4& A, const float4& B, const Eval& e) {
    const float ddx = kEps * (A.z + fabsf(e.dx));
    const float ddy = kEps * (A.w + fabsf(e.dy));
    const float a = fabsf(B.x * e.dx), b = fabsf(B.y * e.dy);
    const float dp = kEps * (a + 2.f * b + fabsf(e.p)) + fabsf(B.x) * ddx + fabsf(B.y) * ddy;
    const float dq = 2.f * kEps * fabsf(e.q) + fabsf(B.z) * ddy;
    return 2.f * fabsf(e.p) * dp + 2.f * fabsf(e.q) * dq + kEps * (e.q * e.q + e.maha);
}

// Stage a record's mean relative to the block origin: (rect origin - block origin)
// is an exact small integer, so one rounding is added; its size enters the
// error scale used by maha_err_bound.
__device__ __forceinline__ float4 stage_A(const float4& a, float ox, float oy) {
    const float mx = __fadd_rn(__fsub_rn(a.x, ox), a.z);
    const float my = __fadd_rn(__fsub_rn(a.y, oy), a.w);
    return make_float4(mx, my, fabsf(a.z) + fabsf(mx), fabsf(a.w) + fabsf(my));
}

// One scan pass of the rank order: thread tid tests rank r (ascending or descending
// passes pass their own r); returns the number of covering ranks of the pass and this
// thread's position among them (rank order of the pass's threads), or -1.
template <int kThreads = 256>
__device__ __forceinline__ int scan_compact(bool cov, int* wsum, int& total) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned b = __ballot_sync(0xffffffffu, cov);
    if (lane == 0) wsum[warp] = __popc(b);
    __syncthreads();
    int off = __popc(b & ((1u << lane) - 1u)), tot = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        const int v = wsum[w];
        off += w < warp ? v : 0;
        tot += v;
    }
    total = tot;
    return cov ? off : -1;
}

// Warp reduce-scatter of 8 per-lane values: 9 shuffles instead of 40.  On
// return, lanes with (lane & 3) == 0 hold the warp sum of value index
// ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1).
__device__ __forceinline__ float reduce_scatter8(float v[8], int lane) {
    {
        const bool hi = lane & 16;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float send = hi ? v[i] : v[i + 4];
            const float keep = hi ? v[i + 4] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
    }
    {
        const bool hi = lane & 8;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const float send = hi ? v[i] : v[i + 2];
            const float keep = hi ? v[i + 2] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
    }
    {
        const bool hi = lane & 4;
        const float send = hi ? v[0] : v[1];
        const float keep = hi ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    float s = v[0];
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    return s;
}

}  // namespace tsb
