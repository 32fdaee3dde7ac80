// SSIM term of the trainer's image loss (losses.cpp:29-166, trainer.cpp:210-219):
//   loss_c = w_c [(1 - lambda) mse_c + lambda (1 - mean SSIM_c)]
// for every quad channel c of a rendered frame against its target raw frame.  The
// mse part is fused into the forward raster's epilogue (with w_c (1 - lambda));
// these kernels add lambda's part to the loss and to d_quad.
//
// SSIM uses an 11-tap Gaussian window (sigma 1.5), separable, zero padded, exactly
// as conv_same (losses.cpp:51-75).  One 32x8-pixel tile per block with a 5-pixel
// halo staged in shared memory; both passes and the per-pixel SSIM terms run in fp64
// (the reference is fp64; sigma^2 = E[x^2] - E[x]^2 cancels).
//   k_ssim_fwd: mu1, mu2, E[x^2], E[y^2], E[xy] -> S per pixel (block partial sums)
//               and the three gradient planes dS/dmu1 (all paths), dS/dE[x^2], dS/dE[xy];
//   k_ssim_bwd: the adjoint convolutions of those planes (the window is symmetric, so
//               conv_same is its own adjoint), d_quad += scale (c1 + 2 x c2 + y c3).
#include <cuda_runtime.h>

#include "tsb_internal.h"

namespace tsb {

namespace {
constexpr int kTW = 32, kTH = 8, kR = 5, kWin = 11;
constexpr int kSW = kTW + 2 * kR, kSH = kTH + 2 * kR;
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;

}  // namespace

__constant__ double c_ssim_win[kWin];

// x, y: planar [nch][H][W] (channel c at x + c * HW); g: [nch][3][H][W] fp64.
__global__ void __launch_bounds__(kTW* kTH) k_ssim_fwd(const float* __restrict__ x, int W, int H, SsimArgs a) {
    __shared__ double sx[kSH][kSW], sy[kSH][kSW];
    __shared__ double hq[5][kSH][kTW];
    __shared__ double red[kTW * kTH / 32];
    if (block_aborted(a.abort)) return;
    const float* __restrict__ y = a.fd->target;
    const int c = a.chans[blockIdx.z];
    double* __restrict__ g = a.g;
    double* __restrict__ part = a.part;
    const size_t HW = (size_t)W * H;
    const float* X = x + c * HW;
    const float* Y = y + c * HW;
    const int bx = blockIdx.x * kTW, by = blockIdx.y * kTH, tid = threadIdx.x;
    for (int i = tid; i < kSH * kSW; i += kTW * kTH) {
        const int ry = i / kSW, rx = i - ry * kSW;
        const int gx = bx + rx - kR, gy = by + ry - kR;
        const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
        sx[ry][rx] = in ? (double)X[(size_t)gy * W + gx] : 0.0;
        sy[ry][rx] = in ? (double)Y[(size_t)gy * W + gx] : 0.0;
    }
    __syncthreads();
    for (int i = tid; i < kSH * kTW; i += kTW * kTH) {  // horizontal pass
        const int ry = i / kTW, cx = i - ry * kTW;
        double a = 0, b = 0, aa = 0, bb = 0, ab = 0;
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            const double w = c_ssim_win[k], u = sx[ry][cx + k], v = sy[ry][cx + k];
            a += w * u;
            b += w * v;
            aa += w * (u * u);
            bb += w * (v * v);
            ab += w * (u * v);
        }
        hq[0][ry][cx] = a;
        hq[1][ry][cx] = b;
        hq[2][ry][cx] = aa;
        hq[3][ry][cx] = bb;
        hq[4][ry][cx] = ab;
    }
    __syncthreads();
    const int cx = tid % kTW, cy = tid / kTW;
    const int px = bx + cx, py = by + cy;
    double mu1 = 0, mu2 = 0, p11 = 0, p22 = 0, p12 = 0;
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
        const double w = c_ssim_win[k];
        mu1 += w * hq[0][cy + k][cx];
        mu2 += w * hq[1][cy + k][cx];
        p11 += w * hq[2][cy + k][cx];
        p22 += w * hq[3][cy + k][cx];
        p12 += w * hq[4][cy + k][cx];
    }
    double S = 0.0;
    if (px < W && py < H) {
        const double s1 = p11 - mu1 * mu1, s2 = p22 - mu2 * mu2, s12 = p12 - mu1 * mu2;
        const double A1 = 2.0 * mu1 * mu2 + kC1, A2 = 2.0 * s12 + kC2;
        const double B1 = mu1 * mu1 + mu2 * mu2 + kC1, B2 = s1 + s2 + kC2;
        S = (A1 * A2) / (B1 * B2);
        const double dS_dsig1 = -S / B2;
        const double dS_dsig12 = 2.0 * A1 / (B1 * B2);
        const double g_mu1 =
            2.0 * mu2 * A2 / (B1 * B2) - 2.0 * mu1 * S / B1 - 2.0 * mu1 * dS_dsig1 - mu2 * dS_dsig12;
        double* G = g + (size_t)blockIdx.z * 3 * HW + (size_t)py * W + px;
        G[0] = g_mu1;
        G[HW] = dS_dsig1;
        G[2 * HW] = dS_dsig12;
    }
    for (int m = 16; m > 0; m >>= 1) S += __shfl_xor_sync(0xffffffffu, S, m);
    if ((tid & 31) == 0) red[tid >> 5] = S;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int i = 0; i < kTW * kTH / 32; ++i) s += red[i];
        part[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s;
    }
}

// d_quad[c] += scale[c] * (conv(g_mu1) + 2 x conv(dS/dsig1) + y conv(dS/dsig12))
__global__ void __launch_bounds__(kTW* kTH) k_ssim_bwd(const float* __restrict__ x, int W, int H, SsimArgs a) {
    __shared__ double sg[3][kSH][kSW];
    __shared__ double hq[3][kSH][kTW];
    if (block_aborted(a.abort)) return;
    const float* __restrict__ y = a.fd->target;
    const int c = a.chans[blockIdx.z];
    const double* __restrict__ g = a.g;
    const size_t HW = (size_t)W * H;
    const double* G = g + (size_t)blockIdx.z * 3 * HW;
    const int bx = blockIdx.x * kTW, by = blockIdx.y * kTH, tid = threadIdx.x;
    for (int i = tid; i < kSH * kSW; i += kTW * kTH) {
        const int ry = i / kSW, rx = i - ry * kSW;
        const int gx = bx + rx - kR, gy = by + ry - kR;
        const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
        const size_t o = (size_t)gy * W + gx;
        sg[0][ry][rx] = in ? G[o] : 0.0;
        sg[1][ry][rx] = in ? G[HW + o] : 0.0;
        sg[2][ry][rx] = in ? G[2 * HW + o] : 0.0;
    }
    __syncthreads();
    for (int i = tid; i < kSH * kTW; i += kTW * kTH) {
        const int ry = i / kTW, cx = i - ry * kTW;
        double ha = 0, hb = 0, hd = 0;
#pragma unroll
        for (int k = 0; k < kWin; ++k) {
            const double w = c_ssim_win[k];
            ha += w * sg[0][ry][cx + k];
            hb += w * sg[1][ry][cx + k];
            hd += w * sg[2][ry][cx + k];
        }
        hq[0][ry][cx] = ha;
        hq[1][ry][cx] = hb;
        hq[2][ry][cx] = hd;
    }
    __syncthreads();
    const int cx = tid % kTW, cy = tid / kTW;
    const int px = bx + cx, py = by + cy;
    if (px >= W || py >= H) return;
    double ca = 0, cb = 0, cd = 0;
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
        const double w = c_ssim_win[k];
        ca += w * hq[0][cy + k][cx];
        cb += w * hq[1][cy + k][cx];
        cd += w * hq[2][cy + k][cx];
    }
    const size_t o = c * HW + (size_t)py * W + px;
    const double xv = x[o], yv = y[o];
    a.d_quad[o] += (float)(a.scale[blockIdx.z] * (ca + 2.0 * xv * cb + yv * cd));
}

// loss += sum_z lam_w[z] * (1 - sum_blocks(part[z]) / npx)
__global__ void k_ssim_loss(SsimArgs a, int nblocks, double npx) {
    __shared__ double s[256];
    if (block_aborted(a.abort)) return;
    double total = 0.0;
    for (int z = 0; z < a.nz; ++z) {
        double acc = 0.0;
        for (int i = threadIdx.x; i < nblocks; i += blockDim.x) acc += a.part[(size_t)z * nblocks + i];
        s[threadIdx.x] = acc;
        __syncthreads();
        for (int m = blockDim.x / 2; m > 0; m >>= 1) {
            if ((int)threadIdx.x < m) s[threadIdx.x] += s[threadIdx.x + m];
            __syncthreads();
        }
        total += a.lam_w[z] * (1.0 - s[0] / npx);
        __syncthreads();
    }
    if (threadIdx.x == 0) *a.loss += total;
}

void ssim_init() {
    static bool done = false;
    if (done) return;
    double w[kWin];
    double sum = 0.0;
    for (int i = 0; i < kWin; ++i) {
        const double d = i - kWin / 2;
        w[i] = exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += w[i];
    }
    for (double& v : w) v /= sum;
    cudaMemcpyToSymbol(c_ssim_win, w, sizeof w);
    done = true;
}

int ssim_blocks(int W, int H) { return ((W + kTW - 1) / kTW) * ((H + kTH - 1) / kTH); }

void launch_ssim(const float* x, int W, int H, const SsimArgs& a, cudaStream_t st) {
    if (a.nz <= 0) return;
    const dim3 grid((W + kTW - 1) / kTW, (H + kTH - 1) / kTH, a.nz);
    k_ssim_fwd<<<grid, kTW * kTH, 0, st>>>(x, W, H, a);
    k_ssim_bwd<<<grid, kTW * kTH, 0, st>>>(x, W, H, a);
    k_ssim_loss<<<1, 256, 0, st>>>(a, (int)(grid.x * grid.y), (double)W * H);
}

}  // namespace tsb
