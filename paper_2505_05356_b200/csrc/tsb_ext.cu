// Colour and flow channels of RenderPass (TSB_CH_COLOR / TSB_CH_FLOW):
//   forward   splat.cpp:273-294 (colour + motion accumulators), 301-334 (bg colour,
//             backprojection of the composited depth and reprojection of x + motion);
//   backward  splat.cpp:361-505 for the colour / motion upstreams;
//   chain     splat.cpp:560-571 (colour SH, clamp-gated, + the view-direction term).
//
// These channels ride beside the ToF hot path instead of inside it: the forward
// kernels of tsb_raster.cu keep their register budget, and the extra work is
// paid only by frames that ask for colour or flow.
//   k_ext_prep  per visible Gaussian: colour = clamp(color_sh^T b(view_dir)) in fp64;
//   k_ext_fwd   per pixel: re-walks the tile lists the forward walked (up to the
//               pixel's termination entry) with the forward's own decisions -- the
//               same fp32 evaluation bits for ordinary pixels, the fp64 records of
//               the fix-up for the pixels the fix-up recomposited -- and accumulates
//               w_k (colour, motion_fwd, motion_bwd); the flow projection reads the
//               final depth_raw / weight of the forward;
//   k_ext_bwd   per pixel, back to front: the upstreams are all T-weighted linear
//               channels, so they reduce to one scalar recursion
//                 d_alpha += Tk (v_k - B),  B <- alpha v_k + (1 - alpha) B,
//                 v_k = up_c . colour_k + up_mf . mf_k + up_mb . mb_k,  B_0 = up_c . bg_colour;
//               the d_alpha part is linear, so its screen-space gradients are added
//               to the ToF backward's (same buffer); the 9 per-entry terms w_k up
//               go to the extension's own screen buffer;
//   k_chain_ext per Gaussian: colour SH gradients (gated 0 < colour_raw < 1), the
//               view-direction term into the position (and keyframe) gradients, and
//               SceneGrads::d_motion_fwd / d_motion_bwd.
// Compiled with -fmad=false (fp64 colour and records round as the oracle does); the
// fp32 evaluation uses explicit-rounding intrinsics (tsb_raster.cuh), unaffected.
#include <cuda_runtime.h>

#include "tsb_fp64.cuh"
#include "tsb_raster.cuh"

namespace tsb {

namespace {

// color_raw = color_sh^T b(view_dir) (splat.cpp:163-173), fp64, same order as the oracle.
struct Color64 {
    double raw[3], view_dir[3], depth, b[16];
};

__device__ __forceinline__ float color_coef(const SceneK& S, int gi, int f) {
    const float4 v = S.color_sh[(size_t)(f >> 2) * S.n + gi];
    const int l = f & 3;
    return l == 0 ? v.x : (l == 1 ? v.y : (l == 2 ? v.z : v.w));
}

__device__ __forceinline__ void color64(const SceneK& S, const CamK& C, const FrameK& F, int gi, Color64& c) {
    double x[3], p[3];
    frame_mean(S, F, gi, x);
    const double* R = C.R;
    for (int i = 0; i < 3; ++i) p[i] = R[i * 3 + 0] * x[0] + R[i * 3 + 1] * x[1] + R[i * 3 + 2] * x[2] + C.t[i];
    c.depth = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
    for (int i = 0; i < 3; ++i) c.view_dir[i] = (x[i] - C.center[i]) / c.depth;
    sh_basis64(c.view_dir, S.sh_degree, c.b);
    for (int ch = 0; ch < 3; ++ch) {
        double cr = 0.0;
        if (S.color_sh)
            for (int k = 0; k < 16; ++k) cr += (double)color_coef(S, gi, 16 * ch + k) * c.b[k];
        c.raw[ch] = cr;
    }
}

__global__ void __launch_bounds__(256) k_ext_prep(SceneK S, CamK C, const FrameDev* __restrict__ fd,
                                                  const uint32_t* __restrict__ touched, float4* __restrict__ col,
                                                  const int32_t* __restrict__ abort) {
    const int gi = blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= S.n || *abort || touched[gi] == 0u) return;
    Color64 c;
    color64(S, C, fd->F, gi, c);
    col[gi] = make_float4((float)clampd(c.raw[0], 0.0, 1.0), (float)clampd(c.raw[1], 0.0, 1.0),
                          (float)clampd(c.raw[2], 0.0, 1.0), 0.f);
}

struct PixMap {
    int tile, x, y;
    bool active;
    float ox, oy, pcx, pcy;
    size_t HW, o;
};

__device__ __forceinline__ PixMap pix_map(const OptK& O, int W, int H) {
    PixMap m;
    const int nsub = O.sub * O.sub;
    m.tile = blockIdx.x / nsub;
    const int sb = blockIdx.x % nsub, tid = threadIdx.x;
    const int lx = (sb % O.sub) * kTile + (tid % kTile), ly = (sb / O.sub) * kTile + (tid / kTile);
    m.x = (m.tile % O.tiles_x) * O.ts + lx;
    m.y = (m.tile / O.tiles_x) * O.ts + ly;
    m.active = lx < O.ts && ly < O.ts && m.x < W && m.y < H;
    m.ox = (float)(m.x - (tid % kTile));
    m.oy = (float)(m.y - (tid / kTile));
    m.pcx = (float)(tid % kTile) + 0.5f;
    m.pcy = (float)(tid / kTile) + 0.5f;
    m.HW = (size_t)W * H;
    m.o = m.active ? (size_t)m.y * W + m.x : 0;
    return m;
}

__device__ __forceinline__ int block_max(int v, int* smax) {
    for (int m = 16; m > 0; m >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, m));
    if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = v;
    __syncthreads();
    int b = 0;
#pragma unroll
    for (int i = 0; i < kRasterThreads / 32; ++i) b = max(b, smax[i]);
    return b;
}

__device__ __forceinline__ float4 ld_or_zero(const float4* p, uint32_t i) {
    return p ? p[i] : make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void __launch_bounds__(kRasterThreads) k_ext_fwd(RecK rec, SceneK S, CamK C, OptK O,
                                                            const FrameDev* __restrict__ fd, ScanK sc, FixupK fx,
                                                            PixK px, int nf, ExtK E) {
    __shared__ float4 sA[kRasterThreads], sB[kRasterThreads];
    __shared__ float4 sC[kRasterThreads], sMf[kRasterThreads], sMb[kRasterThreads];
    __shared__ uint32_t sg[kRasterThreads];
    __shared__ int smax[kRasterThreads / 32];
    __shared__ int wsum[2][kRasterThreads / 32];
    if (block_aborted(px.abort)) return;
    const int W = C.W, H = C.H, tid = threadIdx.x;
    const PixMap m = pix_map(O, W, H);
    const int ttx = m.tile % O.tiles_x, tty = m.tile / O.tiles_x;
    int last = 0;
    bool fixed = false;
    if (m.active) {
        const int l = px.last[m.o];
        fixed = l < 0;
        last = l & kLastMask;
    }
    const int bmax = block_max(last, smax);
    const FrameK F = fd->F;
    const int stamp = fd->stamp;
    float T = 1.f;
    double Td = 1.0;
    double acc[9];  // fp64 sums: the motion channels are signed and cancel
#pragma unroll
    for (int c = 0; c < 9; ++c) acc[c] = 0.0;
    // the tile's list up to the block's furthest pixel: the rank order scanned upwards
    const ScanSeg seg = scan_seg(sc, ttx, tty);
    const int V = seg.n;
    int pass = 0;
    for (int r0 = 0, ebase = 0; r0 < V && ebase < bmax; r0 += kRasterThreads, ++pass) {
        const int rr = r0 + tid;
        const bool cov = rr < V && tile_covers(seg_rect(sc, seg, rr), ttx, tty);
        int total;
        const int pos = scan_compact(cov, wsum[pass & 1], total);  // (its barrier follows the last pass's reads)
        if (pos >= 0) {
            const uint32_t r = sc.ord[seg_rank(sc, seg, rr)];
            sg[pos] = r;
            sA[pos] = stage_A(rec.A[r], m.ox, m.oy);
            sB[pos] = rec.B[r];
            sC[pos] = ld_or_zero(E.col, r);
            sMf[pos] = ld_or_zero(E.mf, r);
            sMb[pos] = ld_or_zero(E.mb, r);
        }
        __syncthreads();
        {
            const int nb = total;
            const int jmax = min(nb, last - ebase);
            ebase += total;
            for (int j = 0; j < jmax; ++j) {
                double wd;
                double cx[3] = {0.0, 0.0, 0.0};
                if (!fixed) {  // the forward's fp32 decisions, bit for bit
                    const float4 A = sA[j], B = sB[j];
                    Eval ev;
                    eval_entry(A, B, m.pcx, m.pcy, ev);
                    if (ev.maha - O.cut2_f > 0.f) continue;
                    eval_alpha(B, ev);
                    if (ev.alpha - O.alpha_thr_f < 0.f) continue;
                    wd = ev.alpha * T;
                    T = T * (1.f - ev.alpha);
                } else {  // the fix-up's fp64 decisions (k_fixup, tsb_geom.cu)
                    const int g = (int)sg[j];
                    const Rec64 r = fx.stamp[g] == stamp ? fx.cache[g] : make_rec64(S, C, O, F, g);
                    if (m.x < r.rect.x || m.x >= r.rect.y || m.y < r.rect.z || m.y >= r.rect.w) continue;
                    const double dx = (m.x + 0.5) - r.m0.x, dy = (m.y + 0.5) - r.m0.y;
                    const double maha = r.m0.z * dx * dx + 2.0 * r.m0.w * dx * dy + r.m1.x * dy * dy;
                    if (maha > O.cut2 || maha < 0.0) continue;
                    const double alpha = r.m1.y * exp(-0.5 * maha);
                    if (alpha < O.alpha_thr) continue;
                    wd = alpha * Td;
                    if (!E.out64) wd = (double)(float)wd;
                    Td *= 1.0 - alpha;
                    if (E.out64 && E.col) {  // reference-exact mode: the fp64 clamped colour
                        Color64 c64;
                        color64(S, C, F, g, c64);
                        for (int ch = 0; ch < 3; ++ch) cx[ch] = clampd(c64.raw[ch], 0.0, 1.0);
                    }
                }
                const float4 cc = sC[j], mf = sMf[j], mb = sMb[j];
                const bool c64 = fixed && E.out64;
                acc[0] = fma(wd, c64 ? cx[0] : (double)cc.x, acc[0]);
                acc[1] = fma(wd, c64 ? cx[1] : (double)cc.y, acc[1]);
                acc[2] = fma(wd, c64 ? cx[2] : (double)cc.z, acc[2]);
                acc[3] = fma(wd, (double)mf.x, acc[3]);
                acc[4] = fma(wd, (double)mf.y, acc[4]);
                acc[5] = fma(wd, (double)mf.z, acc[5]);
                acc[6] = fma(wd, (double)mb.x, acc[6]);
                acc[7] = fma(wd, (double)mb.y, acc[7]);
                acc[8] = fma(wd, (double)mb.z, acc[8]);
            }
        }
    }
    if (!m.active) return;
    const size_t HW = m.HW, o = m.o;
    const double Tfin = px.out[ch_T(nf) * HW + o];
    for (int c = 0; c < 3; ++c) E.out[c * HW + o] = (float)(acc[c] + O.bg_color[c] * Tfin);
    for (int c = 3; c < 9; ++c) E.out[c * HW + o] = (float)acc[c];
    if (E.out64) {  // reference-exact mode: fp64 planes, with the fix-up's fp64 T_N
        const double T64 = fixed ? Td : Tfin;
        for (int c = 0; c < 3; ++c) E.out64[c * HW + o] = acc[c] + O.bg_color[c] * T64;
        for (int c = 3; c < 9; ++c) E.out64[c * HW + o] = acc[c];
    }
    for (int c = 9; c < kExtPlanes; ++c) E.out[c * HW + o] = 0.f;
    if (!E.flow) return;
    const double SW = px.out[ch_weight(nf) * HW + o];
    if (!(SW > O.cov_eps)) return;
    // cam.backproject (camera.hpp:34-43): optical centre + dist * normalize(R^T d_cam)
    const double SD = px.out[ch_depth_raw(nf) * HW + o];
    const double dist = SD / SW;
    const double pcx = m.x + 0.5, pcy = m.y + 0.5;
    const double dc[3] = {(pcx - C.cx) / C.fx, (pcy - C.cy) / C.fy, 1.0};
    const double* R = C.R;
    double dir[3];
    for (int a = 0; a < 3; ++a) dir[a] = R[0 * 3 + a] * dc[0] + R[1 * 3 + a] * dc[1] + R[2 * 3 + a] * dc[2];
    const double dn = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
    double xd[3];
    for (int a = 0; a < 3; ++a) xd[a] = C.center[a] + dist * (dir[a] / dn);
    for (int k = 0; k < 2; ++k) {
        double q[3], p[3];
        for (int a = 0; a < 3; ++a) q[a] = xd[a] + acc[3 + 3 * k + a];
        for (int i = 0; i < 3; ++i) p[i] = R[i * 3 + 0] * q[0] + R[i * 3 + 1] * q[1] + R[i * 3 + 2] * q[2] + C.t[i];
        if (p[2] > 0.0) {
            E.out[(9 + 2 * k) * HW + o] = (float)(C.fx * p[0] / p[2] + C.cx - pcx);
            E.out[(10 + 2 * k) * HW + o] = (float)(C.fy * p[1] / p[2] + C.cy - pcy);
            E.out[(13 + k) * HW + o] = 1.f;
        }
    }
}

constexpr int kExtSub = 16;  // entries per slot round: 8 warps x 16 entries x 16 floats

__global__ void __launch_bounds__(kRasterThreads) k_ext_bwd(RecK rec, OptK O, int W, int H, int nf, ScanK sc,
                                                            PixK px, UpK up, ExtK E, double* __restrict__ screen,
                                                            int scap) {
    __shared__ float4 sA[kRasterThreads], sB[kRasterThreads];
    __shared__ float4 sC[kRasterThreads], sMf[kRasterThreads], sMb[kRasterThreads];
    __shared__ uint32_t srank[kRasterThreads];
    __shared__ float slot[kRasterThreads / 32][kExtSub][16];  // per warp, per entry: its reduced gradients
    __shared__ int smax[kRasterThreads / 32];
    __shared__ int wsum[2][kRasterThreads / 32];
    __shared__ float sbg[kRasterThreads / 32][3];
    if (block_aborted(px.abort)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const PixMap m = pix_map(O, W, H);
    const int ttx = m.tile % O.tiles_x, tty = m.tile / O.tiles_x;
    const size_t HW = m.HW, o = m.o;
    int last = 0;
    float Tnext = 0.f, Bx = 0.f;
    float u[9], bgc[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 0; c < 9; ++c) u[c] = 0.f;
    if (m.active) {
        last = px.last[o] & kLastMask;
        Tnext = px.T_pre[o];
        const float Tf = px.out[ch_T(nf) * HW + o];
        for (int c = 0; c < 3; ++c) {
            if (up.color) {
                u[c] = up.color[c * HW + o];
                Bx = fmaf(u[c], (float)O.bg_color[c], Bx);
                bgc[c] = u[c] * Tf;  // d_bg_color (splat.cpp:427-428)
            }
            if (up.mf) u[3 + c] = up.mf[c * HW + o];
            if (up.mb) u[6 + c] = up.mb[c * HW + o];
        }
    }
    for (int c = 0; c < 3; ++c) {
        float v = bgc[c];
        for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
        if (lane == 0) sbg[tid >> 5][c] = v;
    }
    int wmax = last;
    for (int s = 16; s > 0; s >>= 1) wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, s));
    if (lane == 0) smax[tid >> 5] = wmax;
    __syncthreads();
    int bmax = 0;
#pragma unroll
    for (int i = 0; i < kRasterThreads / 32; ++i) bmax = max(bmax, smax[i]);
    if (tid < 3) {
        double s = 0.0;
        for (int i = 0; i < kRasterThreads / 32; ++i) s += sbg[i][tid];
        E.bg_part[(size_t)blockIdx.x * 3 + tid] = s;
    }
    bool first = true;
    const float cut2 = O.cut2_f, thr = O.alpha_thr_f;
    // the tile's list back to front: the rank order scanned downwards from where the forward stopped
    const int2 bt = sc.blk_term[blockIdx.x];
    const ScanSeg seg = scan_seg(sc, ttx, tty);
    const uint32_t wbit = 1u << warp;
    int pass = 0;
    for (int r_hi = bt.x, e_top = bt.y; bmax > 0 && r_hi > 0 && e_top > 0; r_hi -= kRasterThreads, ++pass) {
        const int rr = r_hi - 1 - tid;
        const bool cov = rr >= 0 && tile_covers(seg_rect(sc, seg, rr), ttx, tty);
        int total;
        const int pos = scan_compact(cov, wsum[pass & 1], total);  // descending rank order
        const int e_lo = e_top - total;
        if (pos >= 0) {
            const int j = total - 1 - pos;  // ascending
            const uint32_t r = sc.ord[seg_rank(sc, seg, rr)];
            srank[j] = r;
            sA[j] = stage_A(rec.A[r], m.ox, m.oy);
            sB[j] = rec.B[r];
            sC[j] = ld_or_zero(E.col, r);
            sMf[j] = ld_or_zero(E.mf, r);
            sMb[j] = ld_or_zero(E.mb, r);
        }
        e_top = e_lo;
        __syncthreads();
        for (int hi = total; hi > 0; hi -= kExtSub) {
            const int lo = max(0, hi - kExtSub);
            for (int k = tid; k < (kRasterThreads / 32) * kExtSub * 16; k += kRasterThreads) (&slot[0][0][0])[k] = 0.f;
            __syncthreads();
            const int jtop = min(hi, wmax - e_lo);
            for (int j = jtop - 1; j >= lo; --j) {
                const int el = e_lo + j;
                (void)wbit;
                bool contrib = false;
                float ga[8], gb[8];
                if (el < last) {
                    const float4 Aa = sA[j], Bb = sB[j];
                    Eval ev;
                    eval_entry(Aa, Bb, m.pcx, m.pcy, ev);
                    if (!(ev.maha - cut2 > 0.f)) {
                        eval_alpha(Bb, ev);
                        if (!(ev.alpha - thr < 0.f)) {
                            contrib = true;
                            const float om = 1.f - ev.alpha;
                            // T before this entry, back from the last contributor's (correctly rounded:
                            // these channels are T-weighted like the ones of k_raster_bwd<EXTRA>)
                            const float Tk = first ? Tnext : __fdiv_rn(Tnext, om);
                            first = false;
                            Tnext = Tk;
                            const float4 cc = sC[j], mf = sMf[j], mb = sMb[j];
                            float v = u[0] * cc.x;
                            v = fmaf(u[1], cc.y, v);
                            v = fmaf(u[2], cc.z, v);
                            v = fmaf(u[3], mf.x, v);
                            v = fmaf(u[4], mf.y, v);
                            v = fmaf(u[5], mf.z, v);
                            v = fmaf(u[6], mb.x, v);
                            v = fmaf(u[7], mb.y, v);
                            v = fmaf(u[8], mb.z, v);
                            const float d_alpha = Tk * (v - Bx);
                            Bx = fmaf(ev.alpha, v, om * Bx);
                            const float dpow = ev.alpha * d_alpha;
                            const float w = ev.alpha * Tk;
                            ga[0] = dpow * (Bb.x * ev.p);
                            ga[1] = dpow * (Bb.y * ev.p + Bb.z * ev.q);
                            ga[2] = -0.5f * ev.dx * ev.dx * dpow;
                            ga[3] = -ev.dx * ev.dy * dpow;
                            ga[4] = -0.5f * ev.dy * ev.dy * dpow;
                            ga[5] = ev.g * d_alpha;
                            ga[6] = w * u[0];
                            ga[7] = w * u[1];
#pragma unroll
                            for (int k = 0; k < 7; ++k) gb[k] = w * u[2 + k];
                            gb[7] = 0.f;
                        }
                    }
                }
                if (__any_sync(0xffffffffu, contrib)) {
                    if (!contrib) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) ga[k] = gb[k] = 0.f;
                    }
                    const float s1 = reduce_scatter8(ga, lane);
                    const float s2 = reduce_scatter8(gb, lane);
                    if ((lane & 3) == 0) {
                        const int vi = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
                        slot[warp][j - lo][vi] = s1;
                        slot[warp][j - lo][8 + vi] = s2;
                    }
                }
            }
            __syncthreads();
            // fixed-order sum over the warps; 15 values per entry (d_alpha part + colour / motion w up)
            for (int k = tid; k < (hi - lo) * 15; k += kRasterThreads) {
                const int je = k / 15, c = k - je * 15;
                float v = 0.f;
#pragma unroll
                for (int w = 0; w < kRasterThreads / 32; ++w) v += slot[w][je][c];
                if (v != 0.f) {
                    const uint32_t r = srank[lo + je];
                    if (c < 6) atomicAdd(&screen[(size_t)c * scap + r], (double)v);
                    else atomicAdd(&E.screen[(size_t)(c - 6) * scap + r], v);
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(128) k_chain_ext(SceneK S, CamK C, FrameK F, const uint32_t* __restrict__ touched,
                                                   ExtK E, float4* __restrict__ grads) {
    const int gi = blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= S.n || touched[gi] == 0u) return;
    const size_t n = (size_t)S.n;
    float g[9];
    bool any = false;
    for (int c = 0; c < 9; ++c) {
        g[c] = E.screen[c * n + gi];
        any |= g[c] != 0.f;
    }
    if (!any) return;
    for (int c = 0; c < 9; ++c) E.screen[c * n + gi] = 0.f;
    if (E.d_motion) {  // SceneGrads::d_motion_fwd / d_motion_bwd (splat.cpp:646-647)
        float4 a = E.d_motion[gi], b = E.d_motion[n + gi];
        a.x += g[3]; a.y += g[4]; a.z += g[5];
        b.x += g[6]; b.y += g[7]; b.z += g[8];
        E.d_motion[gi] = a;
        E.d_motion[n + gi] = b;
    }
    if (!S.color_sh || (g[0] == 0.f && g[1] == 0.f && g[2] == 0.f)) return;
    Color64 c;
    color64(S, C, F, gi, c);
    double dcol[3];
    for (int ch = 0; ch < 3; ++ch) dcol[ch] = (c.raw[ch] > 0.0 && c.raw[ch] < 1.0) ? (double)g[ch] : 0.0;
    // d_color_sh[k][c] = b_k dcol_c  (flat 16 c + k)
    float4* gc = grads + (S.color_sh - S.pos_op) + gi;
    for (int a = 0; a < kColorArrays; ++a) {
        float d[4];
        for (int l = 0; l < 4; ++l) {
            const int f = 4 * a + l;
            d[l] = (float)(c.b[f & 15] * dcol[f >> 4]);
        }
        float4 v = gc[(size_t)a * n];
        v.x += d[0]; v.y += d[1]; v.z += d[2]; v.w += d[3];
        gc[(size_t)a * n] = v;
    }
    if (S.sh_degree == 0) return;  // the basis is constant: no view-direction term
    // d_dir = Jb^T (color_sh dcol); view_dir = (x - C) / |x - C| feeds the position
    double Jb[16][3];
    sh_jacobian64(c.view_dir, S.sh_degree, Jb);
    double d_dir[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < 16; ++k) {
        double t = 0.0;
        for (int ch = 0; ch < 3; ++ch) t += (double)color_coef(S, gi, 16 * ch + k) * dcol[ch];
        for (int a = 0; a < 3; ++a) d_dir[a] += Jb[k][a] * t;
    }
    const double vd = c.view_dir[0] * d_dir[0] + c.view_dir[1] * d_dir[1] + c.view_dir[2] * d_dir[2];
    double dpos[3];
    for (int a = 0; a < 3; ++a) dpos[a] = (d_dir[a] - c.view_dir[a] * vd) / c.depth;
    float4 g0 = grads[gi];
    g0.x += (float)dpos[0]; g0.y += (float)dpos[1]; g0.z += (float)dpos[2];
    grads[gi] = g0;
    if (S.nk > 0) {
        const double wa = 1.0 - F.w, wb = F.w;
        float4* gm = grads + (size_t)(3 + F.key) * n + gi;
        float4 a = *gm;
        a.x += (float)(wa * dpos[0]); a.y += (float)(wa * dpos[1]); a.z += (float)(wa * dpos[2]);
        *gm = a;
        float4* gm2 = grads + (size_t)(3 + F.key + 1) * n + gi;
        float4 b = *gm2;
        b.x += (float)(wb * dpos[0]); b.y += (float)(wb * dpos[1]); b.z += (float)(wb * dpos[2]);
        *gm2 = b;
    }
}

// ---- flow loss (losses.cpp:168-251) -------------------------------------------
// Per pixel and direction: valid = target.valid > 0.5 and flow_valid > 0.5; residual of the
// rendered flow; the unscaled pull-back 2 r through the projection at the frozen
// backprojected point (camera.hpp:34-43) + the motion accumulator; block partial sums of the
// squared error and of the valid count.  The scale 1 / (count used) needs the totals, so it
// is applied by k_flow_scale after k_flow_reduce.
__global__ void __launch_bounds__(256) k_flow_loss(CamK C, int nf, const float* __restrict__ out_tof,
                                                   const float* __restrict__ ext, FlowK F) {
    __shared__ double red[4][8];
    const int W = C.W, H = C.H;
    const size_t HW = (size_t)W * H;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double v[4] = {0.0, 0.0, 0.0, 0.0};  // sse_fwd, count_fwd, sse_bwd, count_bwd
    if (i < (int)HW && !*F.abort) {
        const int x = i % W, y = i / W;
        const double pcx = x + 0.5, pcy = y + 0.5;
        for (int k = 0; k < 2; ++k) {
            const float* tgt = F.target[k];
            float* d = F.d_macc + (size_t)3 * k * HW;
            if (!tgt) continue;
            const bool valid = tgt[2 * HW + i] > 0.5f && ext[(13 + k) * HW + i] > 0.5f;
            if (!valid) {
                d[i] = d[HW + i] = d[2 * HW + i] = 0.f;
                continue;
            }
            const double ru = (double)ext[(9 + 2 * k) * HW + i] - (double)tgt[i];
            const double rv = (double)ext[(10 + 2 * k) * HW + i] - (double)tgt[HW + i];
            v[2 * k] = ru * ru + rv * rv;
            v[2 * k + 1] = 1.0;
            const double du = 2.0 * ru, dv = 2.0 * rv;
            const double depth = out_tof[ch_depth(nf) * HW + i];
            const double dc[3] = {(pcx - C.cx) / C.fx, (pcy - C.cy) / C.fy, 1.0};
            const double* R = C.R;
            double dir[3];
            for (int a = 0; a < 3; ++a) dir[a] = R[0 * 3 + a] * dc[0] + R[1 * 3 + a] * dc[1] + R[2 * 3 + a] * dc[2];
            const double dn = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
            double q[3], pc[3];
            for (int a = 0; a < 3; ++a)
                q[a] = C.center[a] + depth * (dir[a] / dn) + (double)ext[(3 + 3 * k + a) * HW + i];
            for (int r = 0; r < 3; ++r) pc[r] = R[r * 3 + 0] * q[0] + R[r * 3 + 1] * q[1] + R[r * 3 + 2] * q[2] + C.t[r];
            const double z = pc[2], z2 = z * z;
            const double dp[3] = {C.fx * du / z, C.fy * dv / z, -(C.fx * pc[0] * du + C.fy * pc[1] * dv) / z2};
            for (int a = 0; a < 3; ++a)
                d[(size_t)a * HW + i] = (float)(R[0 * 3 + a] * dp[0] + R[1 * 3 + a] * dp[1] + R[2 * 3 + a] * dp[2]);
        }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int c = 0; c < 4; ++c) {
        double t = v[c];
        for (int m = 16; m > 0; m >>= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
        if (lane == 0) red[c][w] = t;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double t = 0.0;
        for (int j = 0; j < 8; ++j) t += red[threadIdx.x][j];
        F.part[(size_t)blockIdx.x * 4 + threadIdx.x] = t;
    }
}

// res: [0] value, [1] valid pixels, [2] / [3] gradient scale per direction (0: no gradient).
__global__ void k_flow_reduce(FlowK F, int nparts, double weight) {
    __shared__ double s[4][256];
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = threadIdx.x; i < nparts; i += blockDim.x)
        for (int c = 0; c < 4; ++c) a[c] += F.part[(size_t)i * 4 + c];
    for (int c = 0; c < 4; ++c) s[c][threadIdx.x] = a[c];
    __syncthreads();
    for (int m = blockDim.x / 2; m > 0; m >>= 1) {
        if ((int)threadIdx.x < m)
            for (int c = 0; c < 4; ++c) s[c][threadIdx.x] += s[c][threadIdx.x + m];
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    int used = 0;
    double value = 0.0, count = 0.0;
    for (int k = 0; k < 2; ++k) {
        if (!F.target[k] || s[2 * k + 1][0] == 0.0) continue;
        value += s[2 * k][0] / s[2 * k + 1][0];
        count += s[2 * k + 1][0];
        ++used;
    }
    F.res[0] = used ? value / used : 0.0;
    F.res[1] = count;
    for (int k = 0; k < 2; ++k)
        F.res[2 + k] = (used && F.target[k] && s[2 * k + 1][0] > 0.0) ? weight / (s[2 * k + 1][0] * used) : 0.0;
}

__global__ void __launch_bounds__(256) k_flow_scale(FlowK F, int npx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npx) return;
    for (int k = 0; k < 2; ++k) {
        if (!F.target[k]) continue;
        const float sc = (float)F.res[2 + k];
        float* d = F.d_macc + (size_t)3 * k * npx;
        for (int a = 0; a < 3; ++a) d[(size_t)a * npx + i] *= sc;
    }
}

// write_render_stacks' derived planes (eval.cpp:96-121, 20-34): mean depth gated at
// coverage weight > 0.5 (NaN elsewhere) and d_ToF decoded from the rendered quad of the
// first frequency (tof.hpp:64-71: phase of (q90 - q270, q0 - q180) in [0, 2 pi), NaN
// where both differences vanish).
__global__ void __launch_bounds__(256) k_stack_planes(const float* __restrict__ out, int nf, int npx, double freq,
                                                      double c, float* __restrict__ dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npx) return;
    const size_t n = (size_t)npx;
    const float nanf = __int_as_float(0x7fc00000);
    dst[i] = out[ch_weight(nf) * n + i] > 0.5f ? out[ch_depth(nf) * n + i] : nanf;
    const double re = (double)out[n + i] - (double)out[3 * n + i];
    const double im = (double)out[i] - (double)out[2 * n + i];
    float d = nanf;
    if (!(re == 0.0 && im == 0.0)) {
        double psi = atan2(im, re);
        if (psi < 0.0) psi += 2.0 * M_PI;
        d = (float)(psi * c / (4.0 * M_PI * freq));
    }
    dst[n + i] = d;
}

}  // namespace

void launch_stack_planes(const float* out, int nf, int npx, double freq, double c, float* dst, cudaStream_t st) {
    if (npx > 0) k_stack_planes<<<(npx + 255) / 256, 256, 0, st>>>(out, nf, npx, freq, c, dst);
}

int flow_loss_parts(int npx) { return (npx + 255) / 256; }

void launch_flow_loss(const CamK& C, int nf, const float* out_tof, const float* ext, const FlowK& F, double weight,
                      cudaStream_t st) {
    const int npx = C.W * C.H, nb = flow_loss_parts(npx);
    k_flow_loss<<<nb, 256, 0, st>>>(C, nf, out_tof, ext, F);
    k_flow_reduce<<<1, 256, 0, st>>>(F, nb, weight);
    k_flow_scale<<<nb, 256, 0, st>>>(F, npx);
}

void launch_ext_prep(const SceneK& S, const CamK& C, const FrameDev* fd, const uint32_t* touched, const ExtK& E,
                     const int32_t* abort, cudaStream_t st) {
    if (S.n <= 0 || !E.col) return;
    k_ext_prep<<<(S.n + 255) / 256, 256, 0, st>>>(S, C, fd, touched, E.col, abort);
}

void launch_ext_fwd(const RecK& rec, const SceneK& S, const CamK& C, const OptK& O, const FrameDev* fd,
                    const ScanK& sc, const FixupK& fx, const PixK& px, int nf, const ExtK& E, cudaStream_t st) {
    const int grid = O.tiles_x * O.tiles_y * O.sub * O.sub;
    k_ext_fwd<<<grid, kRasterThreads, 0, st>>>(rec, S, C, O, fd, sc, fx, px, nf, E);
}

void launch_ext_bwd(const RecK& rec, const OptK& O, int W, int H, int nf, const ScanK& sc, const PixK& px,
                    const UpK& up, const ExtK& E, double* screen, int scap, cudaStream_t st) {
    const int grid = O.tiles_x * O.tiles_y * O.sub * O.sub;
    k_ext_bwd<<<grid, kRasterThreads, 0, st>>>(rec, O, W, H, nf, sc, px, up, E, screen, scap);
}

void launch_chain_ext(const SceneK& S, const CamK& C, const FrameK& F, const uint32_t* touched, const ExtK& E,
                      float4* grads, cudaStream_t st) {
    if (S.n <= 0) return;
    k_chain_ext<<<(S.n + 127) / 128, 128, 0, st>>>(S, C, F, touched, E, grads);
}

}  // namespace tsb
