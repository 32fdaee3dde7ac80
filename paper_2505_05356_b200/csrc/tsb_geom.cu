// fp64 per-Gaussian kernels: preprocess, fp64 pixel fix-up, parameter chain.
// Compiled with -fmad=false (see tsb_fp64.cuh).
#include <cuda_runtime.h>

#include <cstdlib>

#include "tsb_fp64.cuh"
#include "tsb_ties.cuh"

#ifndef TSB_PRE_CTAS
#define TSB_PRE_CTAS 6
#endif

namespace tsb {

// ---------------------------------------------------------------------------
// k_preprocess: RenderPassImpl::prepare (splat.cpp:105-177), one thread per
// Gaussian.  Writes the fp64 depth sort key (bits of the positive double, so
// unsigned order == numeric order; culled -> ~0), tile rect, tiles touched and
// the fp32 raster record (indexed by Gaussian; the duplicate kernel gathers it
// into rank order).
// ---------------------------------------------------------------------------
// sin/cos of the ToF phase for the fp32 record: exact fp64 reduction modulo 2 pi
// (phases here are < ~1e3 rad), then fp32 sincosf of the reduced angle -- within
// 2 ulp of the fp64 result rounded to fp32, for a fraction of the fp64 cost.
__device__ __forceinline__ void sincos_phase32(double psi, float& sn, float& cs) {
    constexpr double kTwoPiHi = 6.283185307179586232;     // 2 pi rounded to double
    constexpr double kTwoPiLo = 2.4492935982947064e-16;   // 2 pi - kTwoPiHi
    const double k = rint(psi * 0.15915494309189535);
    const double r = fma(-k, kTwoPiLo, fma(-k, kTwoPiHi, psi));
    sincosf((float)r, &sn, &cs);
}

// The per-Gaussian values the binning / raster / tie resolution read: fp64 depth,
// tile rect and the fp32 raster record.
__device__ __forceinline__ void write_records(const SceneK& S, const Prep64& s, int gi, double* __restrict__ depth64,
                                              uint2* __restrict__ rect, const RecK& rec) {
    depth64[gi] = s.depth;
    rect[gi] = make_uint2((uint32_t)s.x0 | ((uint32_t)s.x1 << 16), (uint32_t)s.y0 | ((uint32_t)s.y1 << 16));
    // factored conic (Cholesky of [[a, b], [b, c]]) in fp64, rounded once
    const double l11 = sqrt(s.ca);
    const double l12 = s.cb * rcp64(l11);
    const double l22 = rsqrt(s.c11);
    rec.A[gi] = make_float4((float)s.x0, (float)s.y0, (float)(s.mean[0] - (double)s.x0),
                            (float)(s.mean[1] - (double)s.y0));
    rec.B[gi] = make_float4((float)l11, (float)l12, (float)l22, (float)s.opacity);
    float sn, cs;
    sincos_phase32(phase_of_depth(s.depth, S.freq[0], S.c), sn, cs);
    rec.C[gi] = make_float4((float)s.coef, (float)s.depth, sn, cs);
    if (S.nf > 1) {
        sincos_phase32(phase_of_depth(s.depth, S.freq[1], S.c), sn, cs);
        rec.D[gi] = make_float4(sn, cs, 0.f, 0.f);
    }
}

// Visibility and fp64 depth of one Gaussian for a lean frame (below), without the fp64
// EWA projection.  The depth (sort key) and the near / opacity culls are computed with
// the same expressions as prep64, so they are bit-identical.  The rect only decides
// visibility here: with a = mean - r, b = mean + r, the clamped rect of prep64 is
// non-empty iff b > -1 and a < W (per axis) and det > 0.  The projected covariance runs
// in fp32 next to a bound of its magnitudes (|M| |Sigma| |M|^T); a decision within 1e-4
// of those magnitudes of its threshold (fp32 errors are ~1e-6 of them) is left to the
// exact fp64 prep64.  The discriminant uses the cancellation-free form
// ((c0 - c3) / 2)^2 + c1^2 (equal to mid^2 - det).  Returns 0 culled, 1 visible,
// 2 undecided.
__device__ __forceinline__ int lean_visible(const SceneK& S, const CamK& C, const OptK& O, const FrameK& F, int gi,
                                            double& depth) {
    // every load of the test up front (one memory round trip instead of three: the culls
    // below would otherwise hold the opacity and covariance loads behind them)
    const size_t n = (size_t)S.n;
    const bool cached = S.opac && S.cov6f;
    double op = 0.0;
    float c00 = 0.f, c01 = 0.f, c02 = 0.f, c11 = 0.f, c12 = 0.f, c22 = 0.f;
    if (cached) {
        op = S.opac[gi];
        c00 = S.cov6f[gi]; c01 = S.cov6f[n + gi]; c02 = S.cov6f[2 * n + gi];
        c11 = S.cov6f[3 * n + gi]; c12 = S.cov6f[4 * n + gi]; c22 = S.cov6f[5 * n + gi];
    }
    double x[3];
    frame_mean(S, F, gi, x);
    const double* R = C.R;
    double p[3];
    for (int i = 0; i < 3; ++i) p[i] = R[i * 3 + 0] * x[0] + R[i * 3 + 1] * x[1] + R[i * 3 + 2] * x[2] + C.t[i];
    if (p[2] < C.near_plane) return 0;
    depth = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
    if (!cached) op = S.opac ? S.opac[gi] : opacity64(S, gi);
    if (op < O.alpha_thr) return 0;
    if (!S.cov6) return 2;
    // the bound in fp32 from the fp64 camera-space mean (its errors, ~1e-7 relative, sit far
    // inside the tolerances below); camera constants are host-rounded fp32 copies
    const float pf0 = (float)p[0], pf1 = (float)p[1], izf = 1.f / (float)p[2];
    const float mx = C.fxf * (pf0 * izf) + C.cxf, my = C.fyf * (pf1 * izf) + C.cyf;
    const float limx = C.limxf, limy = C.limyf;
    const float txz = fminf(fmaxf(pf0 * izf, -limx), limx);  // clamped tx / z
    const float tyz = fminf(fmaxf(pf1 * izf, -limy), limy);
    const float fxz = C.fxf * izf, fyz = C.fyf * izf;
    // M = J W (2 x 3), J = [[fx/z, 0, -fx tx/z^2], [0, fy/z, -fy ty/z^2]]
    float M[6], Ma[6];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const float r0 = C.Rf[0 * 3 + j], r1 = C.Rf[1 * 3 + j], r2 = C.Rf[2 * 3 + j];
        M[j] = fxz * (r0 - txz * r2);
        M[3 + j] = fyz * (r1 - tyz * r2);
        Ma[j] = fabsf(fxz) * (fabsf(r0) + fabsf(txz * r2));
        Ma[3 + j] = fabsf(fyz) * (fabsf(r1) + fabsf(tyz * r2));
    }
    if (!cached) {  // (the fp32 cache, 24 B instead of 48, was loaded above)
        c00 = (float)S.cov6[gi]; c01 = (float)S.cov6[n + gi]; c02 = (float)S.cov6[2 * n + gi];
        c11 = (float)S.cov6[3 * n + gi]; c12 = (float)S.cov6[4 * n + gi]; c22 = (float)S.cov6[5 * n + gi];
    }
    const float V[9] = {c00, c01, c02, c01, c11, c12, c02, c12, c22};
    float T[6], Ta[6];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            T[i * 3 + j] = M[i * 3 + 0] * V[j] + M[i * 3 + 1] * V[3 + j] + M[i * 3 + 2] * V[6 + j];
            Ta[i * 3 + j] = Ma[i * 3 + 0] * fabsf(V[j]) + Ma[i * 3 + 1] * fabsf(V[3 + j]) + Ma[i * 3 + 2] * fabsf(V[6 + j]);
        }
    const float dil = O.dilation_f;
    const float a0 = T[0] * M[0] + T[1] * M[1] + T[2] * M[2] + dil;
    const float a1 = T[0] * M[3] + T[1] * M[4] + T[2] * M[5];
    const float a3 = T[3] * M[3] + T[4] * M[4] + T[5] * M[5] + dil;
    const float b0 = Ta[0] * Ma[0] + Ta[1] * Ma[1] + Ta[2] * Ma[2] + fabsf(dil);
    const float b1 = Ta[0] * Ma[3] + Ta[1] * Ma[4] + Ta[2] * Ma[5];
    const float b3 = Ta[3] * Ma[3] + Ta[4] * Ma[4] + Ta[5] * Ma[5] + fabsf(dil);
    const float det = a0 * a3 - a1 * a1;
    const float dtol = 1e-4f * (b0 * b3 + b1 * b1);
    if (!(fabsf(det) > dtol)) return 2;  // also NaN
    if (det < 0.f) return 0;
    const float h = 0.5f * (a0 - a3);
    const float disc = h * h + a1 * a1;
    const float lam = 0.5f * (a0 + a3) + sqrtf(fmaxf(disc, 0.1f));
    const float r = O.sigma_cutoff_f * sqrtf(lam);
    const float tol = 1e-4f * (r * fmaxf(1.f, (b0 + b3) / lam) + fabsf(mx) + fabsf(my) + 1.f);
    // huge or non-finite: prep64.  Its rect bounds go through x86 int conversion (INT_MIN
    // past 2^31), which culls splats the plain geometric test keeps, so anything whose
    // mean +- radius gets anywhere near 2^31 px is decided exactly.
    if (!(tol < 1e8f && fabsf(mx) + r < 1e9f && fabsf(my) + r < 1e9f)) return 2;
    const float bx = mx + r + 1.f, ax = C.Wf - (mx - r);
    const float by = my + r + 1.f, ay = C.Hf - (my - r);
    if (fabsf(bx) <= tol || fabsf(ax) <= tol || fabsf(by) <= tol || fabsf(ay) <= tol) return 2;
    return (bx > 0.f && ax > 0.f && by > 0.f && ay > 0.f) ? 1 : 0;
}

// The exact fp64 decision for the rare undecided Gaussians, out of line: inlined, its
// registers made the lean path spill (7 local-memory accesses per Gaussian at 40 registers).
// (The kernel's parameter structs are __grid_constant__, so passing them by reference does
// not copy them to the stack.)
// Returns the depth of a visible Gaussian, -1 for a culled one (by value: no stack slot).
__device__ __noinline__ double lean_exact(const SceneK& S, const CamK& C, const OptK& O, const FrameK& F, int gi) {
    Prep64 s;
    return prep64<false>(S, C, O, F, gi, s) ? s.depth : -1.0;
}

// LEAN (prefix-sorted frames): only the sort key, tiles touched and the visible
// count / key range; the records of the Gaussians the frame reads -- its sorted
// prefix -- are written after the sort by k_records.
template <bool LEAN>
__global__ void __launch_bounds__(256, LEAN ? TSB_PRE_CTAS : 5) k_preprocess(const __grid_constant__ SceneK S,
                                                    const __grid_constant__ CamK C,
                                                    const __grid_constant__ OptK O, const FrameDev* __restrict__ fd,
                                                    uint32_t* __restrict__ depth_key,
                                                    double* __restrict__ depth64,
                                                    uint32_t* __restrict__ gidx,
                                                    uint32_t* __restrict__ touched,
                                                    uint2* __restrict__ rect, RecK rec,
                                                    int32_t* __restrict__ n_visible,
                                                    uint32_t* __restrict__ key_range) {
    uint32_t kmine = 0xffffffffu, kmaxe = 0u;
    const int gi = blockIdx.x * blockDim.x + threadIdx.x;
    const FrameK F = fd->F;
    bool vis = false;
    if (gi < S.n && LEAN) {
        // only visibility and the key: touched is a visibility flag for its readers
        double depth = 0.0;
        int v = lean_visible(S, C, O, F, gi, depth);
        if (v == 2) {
            depth = lean_exact(S, C, O, F, gi);
            v = depth >= 0.0 ? 1 : 0;
        }
        vis = v == 1;
        if (vis) {
            depth_key[gi] = __float_as_uint((float)depth);
            kmine = kmaxe = depth_key[gi];
            touched[gi] = 1u;
        } else {
            depth_key[gi] = 0xffffffffu;
            touched[gi] = 0u;
        }
    } else if (gi < S.n) {
        Prep64 s;
        vis = prep64<false>(S, C, O, F, gi, s);
        if (!LEAN) gidx[gi] = (uint32_t)gi;
        if (vis) {
            // fp32 rounding is monotone, so this 32-bit key orders like the fp64
            // depth except inside runs of equal keys (resolved where read, tsb_ties.cuh).
            depth_key[gi] = __float_as_uint((float)s.depth);
            kmine = kmaxe = depth_key[gi];
            const int ts = O.ts;
            const int tx0 = s.x0 / ts, tx1 = (s.x1 - 1) / ts;
            const int ty0 = s.y0 / ts, ty1 = (s.y1 - 1) / ts;
            touched[gi] = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
            if (!LEAN) write_records(S, s, gi, depth64, rect, rec);
        } else {
            depth_key[gi] = 0xffffffffu;
            touched[gi] = 0u;
        }
    }
    // block-level reduction, then one atomic per block for each of count / min / max
    __shared__ uint32_t s_cnt[8], s_min[8], s_max[8];
    const unsigned m = __ballot_sync(0xffffffffu, vis);
    kmine = __reduce_min_sync(0xffffffffu, kmine);
    kmaxe = __reduce_max_sync(0xffffffffu, kmaxe);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_cnt[w] = __popc(m);
        s_min[w] = kmine;
        s_max[w] = kmaxe;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t c = 0, lo = 0xffffffffu, hi = 0u;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            c += s_cnt[i];
            lo = min(lo, s_min[i]);
            hi = max(hi, s_max[i]);
        }
        if (c) {
            atomicAdd(n_visible, (int)c);
            atomicMin(&key_range[0], lo);
            atomicMax(&key_range[1], hi);
        }
    }
}

// Time-independent per-Gaussian cache (SceneK::cov6 / opac), after every parameter change.
__global__ void __launch_bounds__(256) k_param_cache(SceneK S, double* __restrict__ cov6, double* __restrict__ opac,
                                                     float* __restrict__ cov6f) {
    const int gi = blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= S.n) return;
    double c[9];
    cov3d64(S, gi, c);
    const size_t n = (size_t)S.n;
    cov6[gi] = c[0];
    cov6[n + gi] = c[1];
    cov6[2 * n + gi] = c[2];
    cov6[3 * n + gi] = c[4];
    cov6[4 * n + gi] = c[5];
    cov6[5 * n + gi] = c[8];
    const int pl[6] = {0, 1, 2, 4, 5, 8};
#pragma unroll
    for (int k = 0; k < 6; ++k) cov6f[k * n + gi] = (float)c[pl[k]];
    opac[gi] = opacity64(S, gi);
}

void launch_param_cache(const SceneK& S, double* cov6, double* opac, float* cov6f, cudaStream_t st) {
    if (S.n <= 0) return;
    SceneK raw = S;
    raw.cov6 = nullptr;
    raw.opac = nullptr;
    raw.cov6f = nullptr;
    k_param_cache<<<(S.n + 255) / 256, 256, 0, st>>>(raw, cov6, opac, cov6f);
}

void launch_preprocess(const SceneK& S, const CamK& C, const OptK& O, const FrameDev* F,
                       uint32_t* depth_key, double* depth64, uint32_t* gidx, uint32_t* touched, uint2* rect,
                       RecK rec, int32_t* n_visible, uint32_t* key_range, bool lean, cudaStream_t st) {
    if (S.n <= 0) return;
    const int bs = 256;
    if (lean)
        k_preprocess<true><<<(S.n + bs - 1) / bs, bs, 0, st>>>(S, C, O, F, depth_key, depth64, gidx, touched, rect,
                                                               rec, n_visible, key_range);
    else
        k_preprocess<false><<<(S.n + bs - 1) / bs, bs, 0, st>>>(S, C, O, F, depth_key, depth64, gidx, touched, rect,
                                                                rec, n_visible, key_range);
}

// Records of a lean-preprocessed frame: the Gaussians list[0, *count) (its sorted
// prefix), or with list == null every visible Gaussian (then also the identity
// order the full sort starts from).  Same prep64 on the same inputs as k_preprocess.
__global__ void __launch_bounds__(256, 5) k_records(SceneK S, CamK C, OptK O, const FrameDev* __restrict__ fd,
                                                 const uint32_t* __restrict__ list, const int32_t* __restrict__ count,
                                                 int n, const uint32_t* __restrict__ depth_key,
                                                 double* __restrict__ depth64, uint32_t* __restrict__ gidx,
                                                 uint2* __restrict__ rect, RecK rec, int32_t* __restrict__ abort) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (list ? *count : n)) return;
    const int gi = list ? (int)list[i] : i;
    if (!list) {
        gidx[gi] = (uint32_t)gi;
        if (depth_key[gi] == 0xffffffffu) return;
    }
    const FrameK F = fd->F;
    // prep64 reads the opacity, covariance and reflectivity behind its culls (each a
    // dependent round trip); this Gaussian is known visible, so start them all into L2 now
    {
        const size_t n = (size_t)S.n;
        if (S.opac) asm volatile("prefetch.global.L2 [%0];" ::"l"(S.opac + gi));
        if (S.cov6)
            for (int c = 0; c < 6; ++c) asm volatile("prefetch.global.L2 [%0];" ::"l"(S.cov6 + c * n + gi));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(S.scale_amp + gi));
    }
    Prep64 s;
    // The lean preprocess kept this Gaussian; the exact test must agree.  If it does
    // not, the frame is redone from the exact (non-lean) preprocess (abort bit 16).
    if (!prep64<false>(S, C, O, F, gi, s)) {
        atomicOr(abort, 16);
        return;
    }
    write_records(S, s, gi, depth64, rect, rec);
}

int launch_records(const SceneK& S, const CamK& C, const OptK& O, const FrameDev* F, const uint32_t* list,
                   const int32_t* count, int n, const uint32_t* depth_key, double* depth64, uint32_t* gidx,
                   uint2* rect, RecK rec, int32_t* abort, cudaStream_t st) {
    if (n <= 0) return 0;
    k_records<<<(n + 255) / 256, 256, 0, st>>>(S, C, O, F, list, count, n, depth_key, depth64, gidx, rect, rec,
                                               abort);
    return 1;
}

// ---------------------------------------------------------------------------
// k_fixup: fp64 re-composite of the pixels the fp32 raster flagged as having a
// decision (maha <= cutoff^2, alpha >= threshold, T < floor) inside its error
// band.  One warp per flagged pixel: lanes recompute the fp64 records of 32
// list entries in parallel (the same prep64 the preprocess used), then the warp
// walks them in order exactly as splat.cpp:260-297 does.
// ---------------------------------------------------------------------------
struct FixupAcc {
    double T, SW, SD, Tpre, Tpre_le, accQ[8];  // Tpre_le: T before the entry that made T exactly 0
    double dref, SDs, SD2s;  // distortion moments about the first contributor's depth
    int nc, processed, last_eff;
    bool done;
};

// The raster block (tile, 16 x 16 sub-block) a pixel belongs to: its forward recorded the
// tile list it consumed (ScanK::blk_list) and where its scan of the order stopped.
__device__ __forceinline__ int raster_block(const OptK& O, int x, int y) {
    const int tile = (y / O.ts) * O.tiles_x + x / O.ts;
    const int sb = ((y % O.ts) / kTile) * O.sub + (x % O.ts) / kTile;
    return tile * O.sub * O.sub + sb;
}
__device__ __forceinline__ const uint32_t* block_list(const ScanK& sc, int rb) {
    return sc.blk_list + (size_t)rb * kBlkListCap;
}

// Mark the Gaussians the flagged pixels will visit (their tile lists up to the
// fp32 termination point + a margin) and queue each once for the record cache.
__global__ void __launch_bounds__(128) k_fixup_mark(OptK O, FixupK fx, PixK px, int W, const FrameDev* __restrict__ fd) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int count = block_aborted(fx.overflow) ? 0 : *px.n_flagged;
    const int stamp = fd->stamp;
    for (int i = warp; i < count; i += nwarps) {
        const int pix = px.flagged[i] & 0xffffff;
        const int x = pix % W, y = pix / W;
        const int tx = x / O.ts, ty = y / O.ts;
        const ScanSeg seg = scan_seg(fx.sc, tx, ty);
        const int V = seg.n;
        const int limit = (px.last[pix] & kLastMask) + 64;
        int e = 0, r_from = 0;
        const int rb = raster_block(O, x, y);
        const int2 bt = fx.sc.blk_term[rb];
        if (bt.y <= kBlkListCap) {  // the block's recorded list, then the order past its scan
            const uint32_t* bl = block_list(fx.sc, rb);
            for (int k = lane; k < min(bt.y, limit); k += 32) {
                const uint32_t g = fx.sc.ord[bl[k]];
                if (atomicExch(&fx.stamp[g], stamp) != stamp) {
                    const int slot = atomicAdd(fx.work_n, 1);
                    fx.work[slot] = (int)g;
                }
            }
            e = bt.y;
            r_from = bt.x;
        }
        for (int r0 = r_from; r0 < V && e < limit; r0 += 32) {
            const int r = r0 + lane;
            const bool cov = r < V && tile_covers(seg_rect(fx.sc, seg, r), tx, ty);
            const unsigned m = __ballot_sync(0xffffffffu, cov);
            if (cov && e + __popc(m & ((1u << lane) - 1u)) < limit) {
                const uint32_t g = fx.sc.ord[seg_rank(fx.sc, seg, r)];
                if (atomicExch(&fx.stamp[g], stamp) != stamp) {
                    const int slot = atomicAdd(fx.work_n, 1);
                    fx.work[slot] = (int)g;
                }
            }
            e += __popc(m);
        }
    }
}

__global__ void __launch_bounds__(128) k_fixup_records(SceneK S, CamK C, OptK O, const FrameDev* __restrict__ fd,
                                                       FixupK fx) {
    const int n = *fx.work_n;
    const FrameK F = fd->F;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int g = fx.work[i];
        fx.cache[g] = make_rec64(S, C, O, F, g);
    }
}

// Per warp: evaluate up to 32 candidate entries in parallel (lane j: entry j).
// Only the transmittance product T *= (1 - alpha) and the termination test are
// inherently sequential (they decide the integers); lane 0 runs that chain over
// the batch's contributors from shared memory, then every lane adds its own
// weighted terms and the warp reduces them (fp64; summation order differs from
// the reference only at the 1e-16 level).
struct FixSlot {
    double om;     // 1 - alpha (contributors)
    double Tpre;   // T before this entry (written by lane 0)
    int contrib;
};

__device__ __forceinline__ double warp_sum(double v) {
    for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}

__device__ __forceinline__ void fixup_batch(const SceneK& S, const CamK& C, const OptK& O, const FrameK& F,
                                            const FixupK& fx, int stamp, int nf, int x, int y, bool is_entry, int g,
                                            int entry_idx, FixSlot* slot, FixupAcc& a, int lane) {
    const double pcx = x + 0.5, pcy = y + 0.5;
    bool inc = false;
    double alpha = 0.0, coef = 0.0, depth = 0.0;
    if (is_entry) {
        const Rec64 r = fx.stamp[g] == stamp ? fx.cache[g] : make_rec64(S, C, O, F, g);
        if (!(x < r.rect.x || x >= r.rect.y || y < r.rect.z || y >= r.rect.w)) {
            const double dx = pcx - r.m0.x, dy = pcy - r.m0.y;
            const double maha = r.m0.z * dx * dx + 2.0 * r.m0.w * dx * dy + r.m1.x * dy * dy;
            if (!(maha > O.cut2 || maha < 0.0)) {
                const double gg = exp(-0.5 * maha);
                alpha = r.m1.y * gg;
                if (!(alpha < O.alpha_thr)) {
                    inc = true;
                    coef = r.m1.z;
                    depth = r.m1.w;
                }
            }
        }
    }
    slot[lane].contrib = inc ? 1 : 0;
    slot[lane].om = 1.0 - alpha;
    __syncwarp();
    int jterm = 32, le = -1;
    if (lane == 0) {
        double T = a.T;
        for (int j = 0; j < 32; ++j) {
            if (!slot[j].contrib) continue;
            slot[j].Tpre = T;
            T *= slot[j].om;
            if (T == 0.0 && le < 0) le = j;
            if (T < O.floor_T) {
                jterm = j;
                break;
            }
        }
        a.T = T;
    }
    __syncwarp();
    jterm = __shfl_sync(0xffffffffu, jterm, 0);
    le = __shfl_sync(0xffffffffu, le, 0);
    a.T = __shfl_sync(0xffffffffu, a.T, 0);
    const bool mine = inc && lane <= jterm;
    double w = 0.0, w2 = 0.0, q[8];
    for (int c = 0; c < 8; ++c) q[c] = 0.0;
    if (mine) {
        const double Tk = slot[lane].Tpre;
        w = alpha * Tk;
        w2 = alpha * Tk * Tk;
        const double cq = coef * w2;
        #pragma unroll
        for (int f = 0; f < 2; ++f) {
            if (f >= nf) break;
            double sn, cs;
            sincos(phase_of_depth(depth, S.freq[f], S.c), &sn, &cs);
            q[4 * f + 0] = cq * sn;
            q[4 * f + 1] = cq * cs;
        }
    }
    const unsigned mm = __ballot_sync(0xffffffffu, mine);
    if (mm) {
        #pragma unroll
        for (int f = 0; f < 2; ++f) {
            if (f >= nf) break;
            const double s0 = warp_sum(q[4 * f + 0]), s1 = warp_sum(q[4 * f + 1]);
            a.accQ[4 * f + 0] += s0;
            a.accQ[4 * f + 1] += s1;
            a.accQ[4 * f + 2] -= s0;
            a.accQ[4 * f + 3] -= s1;
        }
        a.SW += warp_sum(w);
        a.SD += warp_sum(w * depth);
        if (a.nc == 0) a.dref = (double)(float)__shfl_sync(0xffffffffu, depth, __ffs(mm) - 1);  // = record depth
        const double dd = depth - a.dref;
        a.SDs += warp_sum(w * dd);
        a.SD2s += warp_sum(w * dd * dd);
        a.nc += __popc(mm);
        const int last_lane = 31 - __clz(mm);
        a.Tpre = __shfl_sync(0xffffffffu, mine ? slot[lane].Tpre : 0.0, last_lane);
    }
    if (le >= 0 && a.last_eff < 0) {
        a.last_eff = __shfl_sync(0xffffffffu, entry_idx, le) + 1;
        a.Tpre_le = slot[le].Tpre;
    }
    if (jterm < 32) {
        a.processed = __shfl_sync(0xffffffffu, entry_idx, jterm) + 1;
        a.done = true;
    }
    __syncwarp();
}

// A warp's scan of the rank order for one pixel's tile: kScanRanks ranks per step (lane
// j tests ranks r0 + 32 k + j), covering ranks appended in rank order (ascending or
// descending scan) to the warp's queue, so the expensive per-entry fp64 work always runs
// on full batches of 32 entries (a tile list holds ~1-7 % of the ranks).
constexpr int kScanK = 4;                    // rank groups of 32 per step
constexpr int kQueue = 32 + 32 * kScanK;     // entries a queue can hold after a step
// Scan positions index the tile's super-tile list (ScanSeg); qr receives the position
// (pos_out) or the rank.
__device__ __forceinline__ void queue_step(const ScanK& sc, const ScanSeg& seg, int r0, bool descending, int tx,
                                           int ty, int* qg, int* qr, int& qn, int lane, bool pos_out,
                                           int r_min = 0) {
    const uint32_t below = (1u << lane) - 1u;
    const int V = seg.n;
#pragma unroll
    for (int k = 0; k < kScanK; ++k) {
        const int r = descending ? r0 - 1 - (32 * k + lane) : r0 + 32 * k + lane;
        const bool cov = r >= r_min && r < V && tile_covers(seg_rect(sc, seg, r), tx, ty);
        const unsigned m = __ballot_sync(0xffffffffu, cov);
        if (cov) {
            const uint32_t rk = seg_rank(sc, seg, r);
            qg[qn + __popc(m & below)] = (int)sc.ord[rk];
            qr[qn + __popc(m & below)] = pos_out ? r : (int)rk;
        }
        qn += __popc(m);
    }
    __syncwarp();
}
// drop the first 32 queued entries
__device__ __forceinline__ void queue_pop32(int* qg, int* qr, int& qn, int lane) {
    int g[kQueue / 32 - 1], r[kQueue / 32 - 1];
#pragma unroll
    for (int k = 0; k < kQueue / 32 - 1; ++k) {
        const int i = 32 + 32 * k + lane;
        g[k] = i < qn ? qg[i] : 0;
        r[k] = i < qn ? qr[i] : 0;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kQueue / 32 - 1; ++k) {
        const int i = 32 * k + lane;
        if (i + 32 < qn) {
            qg[i] = g[k];
            qr[i] = r[k];
        }
    }
    qn = max(qn - 32, 0);
    __syncwarp();
}

__global__ void __launch_bounds__(128) k_fixup(SceneK S, CamK C, OptK O, const FrameDev* __restrict__ fd, FixupK fx,
                                               PixK px, int nf) {
    __shared__ FixSlot slots[4][32];
    __shared__ int queue_g[4][kQueue], queue_r[4][kQueue];
    const FrameK F = fd->F;
    const int stamp = fd->stamp;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    FixSlot* slot = slots[threadIdx.x >> 5];
    const int count = block_aborted(fx.overflow) ? 0 : *px.n_flagged;
    const int W = C.W;
    const size_t HW = (size_t)W * C.H;
    const int V_all = *fx.sc.n_rank;
    const uint32_t lanes_below = (1u << lane) - 1u;
    for (int i = warp; i < count; i += nwarps) {
        const int pix = px.flagged[i] & 0xffffff;
        const int x = pix % W, y = pix / W;
        const int tx = x / O.ts, ty = y / O.ts;
        const ScanSeg seg = scan_seg(fx.sc, tx, ty);
        const int V = seg.n;
        FixupAcc a;
        a.T = 1.0; a.SW = 0.0; a.SD = 0.0; a.Tpre = 1.0; a.Tpre_le = 1.0;
        a.dref = 0.0; a.SDs = 0.0; a.SD2s = 0.0;
        for (int c = 0; c < 8; ++c) a.accQ[c] = 0.0;
        a.nc = 0; a.processed = 0; a.last_eff = -1; a.done = false;
        // the tile's list, 32 entries at a time: the entries its raster block recorded, then
        // (rank order from where that block's scan stopped) the ranks covering the tile
        int* qg = queue_g[threadIdx.x >> 5];
        int* qr = queue_r[threadIdx.x >> 5];
        int qn = 0, r_end = V, r_from = 0;
        {
            const int rb = raster_block(O, x, y);
            const int2 bt = fx.sc.blk_term[rb];
            if (bt.y <= kBlkListCap) {
                const uint32_t* bl = block_list(fx.sc, rb);
                for (int e0 = 0; e0 < bt.y && !a.done; e0 += 32) {
                    const bool is_e = e0 + lane < bt.y;
                    const int rk = is_e ? (int)bl[e0 + lane] : 0;
                    fixup_batch(S, C, O, F, fx, stamp, nf, x, y, is_e, is_e ? (int)fx.sc.ord[rk] : 0, e0 + lane, slot,
                                a, lane);
                    if (!a.done) a.processed = min(bt.y, e0 + 32);
                    else r_end = bt.x;  // ended inside the list: the backward walks only the list
                }
                r_from = bt.x;
            }
        }
        for (int r0 = r_from; !a.done && (r0 < V || qn > 0); r0 += 32 * kScanK) {
            if (r0 < V) queue_step(fx.sc, seg, r0, false, tx, ty, qg, qr, qn, lane, true);
            const bool flush = r0 + 32 * kScanK >= V;  // no more ranks: run the partial batch
            while (!a.done && (qn >= 32 || (flush && qn > 0))) {
                const bool is_e = lane < qn;
                const int e0 = a.processed;
                fixup_batch(S, C, O, F, fx, stamp, nf, x, y, is_e, is_e ? qg[lane] : 0, e0 + lane, slot, a, lane);
                if (!a.done) a.processed = e0 + min(qn, 32);
                else r_end = qr[a.processed - 1 - e0] + 1;  // position after the terminating entry
                queue_pop32(qg, qr, qn, lane);
            }
        }
        // the prefix order ended with the pixel alive: the frame is redone with the full order
        if (!a.done && lane == 0 && V_all < *fx.sc.n_all) atomicOr(fx.overflow, 8);
        if (lane == 0) {
            const size_t o = (size_t)y * W + x;
            #pragma unroll
            for (int c = 0; c < 8; ++c)
                if (c < 4 * nf) px.out[c * HW + o] = (float)(a.accQ[c] + O.bg_quad[c] * a.T * a.T);
            px.out[ch_depth_raw(nf) * HW + o] = (float)a.SD;
            px.out[ch_depth(nf) * HW + o] = a.SW > O.cov_eps ? (float)(a.SD / a.SW) : __int_as_float(0x7fc00000);
            px.out[ch_weight(nf) * HW + o] = (float)a.SW;
            px.out[ch_T(nf) * HW + o] = (float)a.T;
            #pragma unroll
            for (int f = 0; f < 2; ++f) {
                if (f >= nf) break;
                px.out[(ch_phasor(nf) + 2 * f + 0) * HW + o] =
                    (float)(2.0 * a.accQ[4 * f + 1] + O.bg_phasor[2 * f + 0] * a.T * a.T);
                px.out[(ch_phasor(nf) + 2 * f + 1) * HW + o] =
                    (float)(2.0 * a.accQ[4 * f + 0] + O.bg_phasor[2 * f + 1] * a.T * a.T);
            }
            if (px.dist3) {
                px.out[ch_distortion(nf) * HW + o] = (float)(2.0 * (a.SW * a.SD2s - a.SDs * a.SDs));
                px.dist3[o] = a.dref;
                px.dist3[HW + o] = a.SDs;
                px.dist3[2 * HW + o] = a.SD2s;
            }
            if (px.out64) {  // reference-exact mode: the same planes in fp64
                double* q = px.out64;
                for (int c = 0; c < 4 * nf; ++c) q[c * HW + o] = a.accQ[c] + O.bg_quad[c] * a.T * a.T;
                q[ch_depth_raw(nf) * HW + o] = a.SD;
                q[ch_depth(nf) * HW + o] = a.SW > O.cov_eps ? a.SD / a.SW : __longlong_as_double(0x7ff8000000000000ll);
                q[ch_weight(nf) * HW + o] = a.SW;
                q[ch_T(nf) * HW + o] = a.T;
                for (int f = 0; f < nf; ++f) {
                    q[(ch_phasor(nf) + 2 * f + 0) * HW + o] = 2.0 * a.accQ[4 * f + 1] + O.bg_phasor[2 * f + 0] * a.T * a.T;
                    q[(ch_phasor(nf) + 2 * f + 1) * HW + o] = 2.0 * a.accQ[4 * f + 0] + O.bg_phasor[2 * f + 1] * a.T * a.T;
                }
                q[ch_distortion(nf) * HW + o] = 2.0 * (a.SW * a.SD2s - a.SDs * a.SDs);
            }
            if (px.n_contrib) px.n_contrib[o] = a.nc;
            if (px.n_processed) px.n_processed[o] = a.processed;
            const int le = a.last_eff >= 0 ? a.last_eff : a.processed;
            const double Tpre = a.last_eff >= 0 ? a.Tpre_le : a.Tpre;
            // the fp64 backward replays this walk back to front from where it stopped
            const bool bwd64 = i < fx.state_cap;
            if (bwd64) {
                FixState f;
                f.T = a.T; f.Tpre = Tpre; f.SW = a.SW;
                f.dref = a.dref; f.SDs = a.SDs; f.SD2s = a.SD2s;
                f.r_end = r_end;
                f.e_end = a.processed;
                fx.state[i] = f;
                fx.fix_idx[o] = i;
            }
            px.last[o] = le | kLastFixed | (bwd64 ? kLastBwd64 : 0);
            px.T_pre[o] = (float)Tpre;
        }
    }
}

int launch_fixup(const SceneK& S, const CamK& C, const OptK& O, const FrameDev* fd, const FixupK& fx,
                 const PixK& px, int nf, cudaStream_t st) {
    // The record cache (mark + records: each Gaussian's fp64 record computed once per frame
    // for all the pixels that visit it) -- A/B switch TSB_FIXUP_CACHE=0: records inline.
    static const bool cache = [] {
        const char* e = std::getenv("TSB_FIXUP_CACHE");
        return !e || std::atoi(e) != 0;
    }();
    if (cache) {
        cudaMemsetAsync(fx.work_n, 0, sizeof(int), st);
        k_fixup_mark<<<148, 128, 0, st>>>(O, fx, px, C.W, fd);
        k_fixup_records<<<148, 128, 0, st>>>(S, C, O, fd, fx);
    }
    k_fixup<<<148, 128, 0, st>>>(S, C, O, fd, fx, px, nf);
    return cache ? 3 : 1;
}

// ---------------------------------------------------------------------------
// k_fixup_bwd: fp64 backward of the pixels k_fixup recomposited (splat.cpp:374-519,
// every ToF upstream of BufferGrads), so their gradients follow the fp64 decisions
// and transmittances of their fp64 forward (SURVEY H1 for the backward; the fp32
// raster backward skips them).  One warp per pixel walks its entries back to front,
// 32 at a time (lane j = the j-th entry from the back), each lane evaluating its
// entry's fp64 record exactly as k_fixup did.  The reverse sweep's recursions are
// warp scans instead of a serial loop:
//   T before entry k      T_k = T_{k+1} / (1 - alpha_k)         (product scan; the
//                         pixel's last contributor starts from its stored T before it)
//   T^2-weighted channels A_k = alpha_{k+1} U_{k+1} + (1 - alpha_{k+1})^2 A_{k+1}
//   T-weighted channels   B_k = alpha_{k+1} v_{k+1} + (1 - alpha_{k+1}) B_{k+1}
//   transmittance         R_k = prod_{j > k} (1 - alpha_j)
// (A and B are affine maps composed across lanes), with
//   d alpha_k = T_k^2 (U_k + 2 (alpha_k - 1) A_k) + T_k (v_k - B_k) - up_T T_k R_k,
//   U_k = coef_k (upQ . basis_k + 2 upP . (cos, sin)_k),
//   v_k = up_draw d_k + up_w + up_dd phi_k,  phi_k = 2 sum_j w_j (d_j - d_k)^2.
// ---------------------------------------------------------------------------
namespace {
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double scan_mul_incl(double v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_up_sync(kFull, v, d);
        if (lane >= d) v *= o;
    }
    return v;
}

// inclusive composition in lane order of x -> a x + b: lane j ends with f_j o ... o f_0
__device__ __forceinline__ void scan_affine_incl(double& a, double& b, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double ao = __shfl_up_sync(kFull, a, d), bo = __shfl_up_sync(kFull, b, d);
        if (lane >= d) {
            b = fma(a, bo, b);
            a *= ao;
        }
    }
}

struct BwdPix {
    double us[2], uc[2], dpsi[2];  // per frequency: upstream weights of (sin, cos); d psi / d depth
    double uDraw, uW, uDD, uT;
    double SW, dref, SDs, SD2s;
    double Tnext, A, B, R;          // carried across batches (back to front)
    bool first;                     // the pixel's last contributor not reached yet
};

// Where a recomposited pixel's per-entry gradients go: added atomically to the pass's
// screen-space gradients, or (deterministic mode) to the (rank, tile, sub-block) slot the
// raster backward filled, by the one warp that owns that raster block.
struct AtomicOut {
    double* screen;
    int scap;
    __device__ __forceinline__ void add(int c, int g, int r, double v) const {
        (void)r;
        atomicAdd(&screen[(size_t)c * scap + g], v);
    }
};
struct DetOut {
    ScanK sc;
    int tx, ty, sb;
    __device__ __forceinline__ void add(int c, int g, int r, double v) const {
        (void)g;
        float* p = &sc.det_part[det_slot(sc, r, sc.trect[r], tx, ty, sb) * 8 + c];
        *p = (float)((double)*p + v);
    }
};

template <class Out>
__device__ __forceinline__ void fixbwd_batch(const SceneK& S, const CamK& C, const OptK& O, const FrameK& F,
                                             const FixupK& fx, int stamp, int nf, int x, int y, bool is_entry, int g,
                                             int rk, BwdPix& b, const Out& out, int lane) {
    bool inc = false;
    double alpha = 0.0, G = 0.0, dx = 0.0, dy = 0.0, coef = 0.0, depth = 0.0;
    Rec64 r;
    if (is_entry) {  // k_fixup's decisions, same expressions
        r = fx.stamp[g] == stamp ? fx.cache[g] : make_rec64(S, C, O, F, g);
        if (!(x < r.rect.x || x >= r.rect.y || y < r.rect.z || y >= r.rect.w)) {
            dx = (x + 0.5) - r.m0.x;
            dy = (y + 0.5) - r.m0.y;
            const double maha = r.m0.z * dx * dx + 2.0 * r.m0.w * dx * dy + r.m1.x * dy * dy;
            if (!(maha > O.cut2 || maha < 0.0)) {
                G = exp(-0.5 * maha);
                alpha = r.m1.y * G;
                if (!(alpha < O.alpha_thr)) {
                    inc = true;
                    coef = r.m1.z;
                    depth = r.m1.w;
                }
            }
        }
    }
    const unsigned cm = __ballot_sync(kFull, inc);
    if (!cm) return;
    const double om = inc ? 1.0 - alpha : 1.0;
    // T before each contributor, back from the pixel's last one (its T is stored, alpha may be 1)
    const int j0 = b.first ? __ffs(cm) - 1 : -1;
    const double P = scan_mul_incl(lane == j0 ? 1.0 : om, lane);
    const double Tk = b.Tnext / P;
    double su = 0.0, sd = 0.0;
    if (inc) {
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            if (f >= nf) break;
            double sn, cs;
            sincos(phase_of_depth(depth, S.freq[f], S.c), &sn, &cs);
            su += b.us[f] * sn + b.uc[f] * cs;
            sd += b.dpsi[f] * (b.us[f] * cs - b.uc[f] * sn);
        }
    }
    const double e = b.dref - depth;
    const double phi = 2.0 * (b.SD2s + 2.0 * e * b.SDs + e * e * b.SW);
    const double U = coef * su;
    const double v = b.uDraw * depth + b.uW + b.uDD * phi;
    // accumulators behind each entry: exclusive scans of the composed maps
    double aA = inc ? om * om : 1.0, bA = inc ? alpha * U : 0.0;
    double aB = inc ? om : 1.0, bB = inc ? alpha * v : 0.0;
    scan_affine_incl(aA, bA, lane);
    scan_affine_incl(aB, bB, lane);
    const double Rin = scan_mul_incl(om, lane);
    double Aex = __shfl_up_sync(kFull, fma(aA, b.A, bA), 1);
    double Bex = __shfl_up_sync(kFull, fma(aB, b.B, bB), 1);
    double Rex = __shfl_up_sync(kFull, Rin, 1) * b.R;
    if (lane == 0) {
        Aex = b.A;
        Bex = b.B;
        Rex = b.R;
    }
    if (inc) {
        const double d_alpha = Tk * Tk * (U + 2.0 * (alpha - 1.0) * Aex) + Tk * (v - Bex) - b.uT * Tk * Rex;
        const double w = alpha * Tk, w2 = w * Tk;
        const double dpow = alpha * d_alpha;
        const double g8[8] = {dpow * (r.m0.z * dx + r.m0.w * dy),
                              dpow * (r.m0.w * dx + r.m1.x * dy),
                              -0.5 * dx * dx * dpow,
                              -dx * dy * dpow,
                              -0.5 * dy * dy * dpow,
                              G * d_alpha,
                              w2 * su,
                              w2 * coef * sd + b.uDraw * w + b.uDD * 4.0 * w * (b.SW * (depth - b.dref) - b.SDs)};
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if (g8[c] != 0.0) out.add(c, g, rk, g8[c]);
    }
    // carry to the next batch (the entries in front): values after lane 31
    b.Tnext = __shfl_sync(kFull, Tk, 31);
    b.A = __shfl_sync(kFull, fma(aA, b.A, bA), 31);
    b.B = __shfl_sync(kFull, fma(aB, b.B, bB), 31);
    b.R *= __shfl_sync(kFull, Rin, 31);
    b.first = false;
}
}  // namespace

// One recomposited pixel's fp64 backward: k_fixup's walk, back to front.
template <class Out>
__device__ void fixbwd_pixel(const SceneK& S, const CamK& C, const OptK& O, const FrameK& F, const FixupK& fx,
                             const PixK& px, const UpK& up, int nf, int stamp, int i, int pix, int* qg, int* qr,
                             const Out& out, int lane) {
    const int W = C.W;
    const size_t HW = (size_t)W * C.H;
    const int last = px.last[pix] & kLastMask;
    const FixState st = fx.state[i];
    const int x = pix % W, y = pix / W;
    const int tx = x / O.ts, ty = y / O.ts;
    const ScanSeg seg = scan_seg(fx.sc, tx, ty);
    const size_t o = (size_t)pix;
    BwdPix b;
    b.A = 0.0;
    for (int f = 0; f < 2; ++f) {
        b.us[f] = b.uc[f] = 0.0;
        b.dpsi[f] = f < nf ? 4.0 * M_PI * S.freq[f] / S.c : 0.0;
        if (f >= nf) continue;
        if (up.quad) {
            double q[4];
            for (int c = 0; c < 4; ++c) {
                q[c] = up.quad[(4 * f + c) * HW + o];
                b.A += q[c] * O.bg_quad[4 * f + c];
            }
            b.us[f] = q[0] - q[2];
            b.uc[f] = q[1] - q[3];
        }
        if (up.phasor) {
            const double p0 = up.phasor[(2 * f + 0) * HW + o], p1 = up.phasor[(2 * f + 1) * HW + o];
            b.A += p0 * O.bg_phasor[2 * f + 0] + p1 * O.bg_phasor[2 * f + 1];
            b.us[f] += 2.0 * p1;
            b.uc[f] += 2.0 * p0;
        }
    }
    b.uDraw = up.depth_raw ? (double)up.depth_raw[o] : 0.0;
    b.uW = up.weight ? (double)up.weight[o] : 0.0;
    b.uDD = up.distortion ? (double)up.distortion[o] : 0.0;
    b.uT = up.transm ? (double)up.transm[o] : 0.0;
    b.SW = st.SW; b.dref = st.dref; b.SDs = st.SDs; b.SD2s = st.SD2s;
    b.Tnext = st.Tpre;
    b.B = 0.0;
    b.R = 1.0;
    b.first = true;
    // the walk of k_fixup back to front: the ranks past the raster block's recorded list
    // downwards from where the walk stopped (covering ranks queued in descending order, so
    // lane j of a batch holds the j-th entry from the back), then the recorded list reversed
    const int rb = raster_block(O, x, y);
    const int2 bt = fx.sc.blk_term[rb];
    const bool listed = bt.y <= kBlkListCap;
    const int r_lo = listed ? bt.x : 0;  // the rank scan covers [r_lo, r_end)
    int qn = 0, e_hi = st.e_end;
    for (int r_hi = st.r_end; e_hi > 0 && (r_hi > r_lo || qn > 0); r_hi -= 32 * kScanK) {
        if (r_hi > r_lo) queue_step(fx.sc, seg, r_hi, true, tx, ty, qg, qr, qn, lane, false, r_lo);
        const bool flush = r_hi - 32 * kScanK <= r_lo;
        while (e_hi > 0 && (qn >= 32 || (flush && qn > 0))) {
            const int e = e_hi - 1 - lane;  // queued entries in descending list order
            const bool is_q = lane < qn && e >= 0;
            fixbwd_batch(S, C, O, F, fx, stamp, nf, x, y, is_q && e < last, is_q ? qg[lane] : 0, is_q ? qr[lane] : 0,
                         b, out, lane);
            e_hi -= min(qn, 32);
            queue_pop32(qg, qr, qn, lane);
        }
    }
    if (listed) {
        const uint32_t* bl = block_list(fx.sc, rb);
        for (; e_hi > 0; e_hi -= 32) {
            const int e = e_hi - 1 - lane;
            const bool is_q = e >= 0;
            const int rk = is_q ? (int)bl[e] : 0;
            fixbwd_batch(S, C, O, F, fx, stamp, nf, x, y, is_q && e < last, is_q ? (int)fx.sc.ord[rk] : 0, rk, b, out,
                         lane);
        }
    }
}

__global__ void __launch_bounds__(128) k_fixup_bwd(SceneK S, CamK C, OptK O, const FrameDev* __restrict__ fd,
                                                   FixupK fx, PixK px, UpK up, int nf, double* __restrict__ screen,
                                                   int scap) {
    __shared__ int queue_g[4][kQueue], queue_r[4][kQueue];
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int count = block_aborted(fx.overflow) ? 0 : min(*px.n_flagged, fx.state_cap);
    const AtomicOut out{screen, scap};
    for (int i = warp; i < count; i += nwarps) {
        const int pix = px.flagged[i] & 0xffffff;
        if (!(px.last[pix] & kLastBwd64)) continue;
        fixbwd_pixel(S, C, O, fd->F, fx, px, up, nf, fd->stamp, i, pix, queue_g[threadIdx.x >> 5],
                     queue_r[threadIdx.x >> 5], out, lane);
    }
}

// Deterministic: warp w owns raster block (tile, sub-block) rb and processes its recomposited
// pixels in pixel order, adding into that block's own slots after the raster backward.
__global__ void __launch_bounds__(128) k_fixup_bwd_det(SceneK S, CamK C, OptK O, const FrameDev* __restrict__ fd,
                                                       FixupK fx, PixK px, UpK up, int nf) {
    __shared__ int queue_g[4][kQueue], queue_r[4][kQueue];
    if (block_aborted(fx.overflow)) return;
    const int lane = threadIdx.x & 31;
    const int rb = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nsub2 = O.sub * O.sub;
    if (rb >= O.tiles_x * O.tiles_y * nsub2) return;
    const int tile = rb / nsub2, sb = rb % nsub2;
    const int tx = tile % O.tiles_x, ty = tile / O.tiles_x;
    const DetOut out{fx.sc, tx, ty, sb};
    for (int k = 0; k < kTile * kTile; k += 32) {
        const int q = k + lane;
        const int lx = (sb % O.sub) * kTile + (q % kTile), ly = (sb / O.sub) * kTile + q / kTile;
        const int x = tx * O.ts + lx, y = ty * O.ts + ly;
        const bool valid = lx < O.ts && ly < O.ts && x < C.W && y < C.H;
        const int pix = valid ? y * C.W + x : 0;
        unsigned m = __ballot_sync(0xffffffffu, valid && (px.last[pix] & kLastBwd64));
        while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1u;
            const int p = __shfl_sync(0xffffffffu, pix, j);
            fixbwd_pixel(S, C, O, fd->F, fx, px, up, nf, fd->stamp, fx.fix_idx[p], p, queue_g[threadIdx.x >> 5],
                         queue_r[threadIdx.x >> 5], out, lane);
        }
    }
}

void launch_fixup_bwd(const SceneK& S, const CamK& C, const OptK& O, const FrameDev* fd, const FixupK& fx,
                      const PixK& px, const UpK& up, int nf, double* screen, int scap, cudaStream_t st) {
    k_fixup_bwd<<<148, 128, 0, st>>>(S, C, O, fd, fx, px, up, nf, screen, scap);
}

void launch_fixup_bwd_det(const SceneK& S, const CamK& C, const OptK& O, const FrameDev* fd, const FixupK& fx,
                          const PixK& px, const UpK& up, int nf, cudaStream_t st) {
    const int nrb = O.tiles_x * O.tiles_y * O.sub * O.sub;
    k_fixup_bwd_det<<<(nrb + 3) / 4, 128, 0, st>>>(S, C, O, fd, fx, px, up, nf);
}

// Intermediates the chain needs, recomputed in fp64 with reciprocals instead of
// divisions (values agree with prep64 to a few ulp; the chain has no decisions
// except the frustum-clamp flags and the 0 < r < 1 gate, which use the same
// comparisons as prep64 on the same inputs).
struct Chain64 {
    double p[3], depth, opacity, refl_raw, M[6], cov3d[9], tx, ty, ca, cb, cc, Rq[9], uq[4], sv[3], qn;
    double view_dir[3];
    bool clx, cly;
};

__device__ __forceinline__ void chain_prep(const SceneK& S, const CamK& C, const OptK& O, const FrameK& F, int gi,
                                           Chain64& s) {
    double x[3];
    frame_mean(S, F, gi, x);
    const double* R = C.R;
    for (int i = 0; i < 3; ++i) s.p[i] = R[i * 3 + 0] * x[0] + R[i * 3 + 1] * x[1] + R[i * 3 + 2] * x[2] + C.t[i];
    s.depth = sqrt(s.p[0] * s.p[0] + s.p[1] * s.p[1] + s.p[2] * s.p[2]);
    const float4 po = S.pos_op[gi];
    s.opacity = 1.0 / (1.0 + exp(-(double)po.w));
    const double z = s.p[2], iz = 1.0 / z;
    const float4 qf = S.quat[gi];
    const double q[4] = {(double)qf.x, (double)qf.y, (double)qf.z, (double)qf.w};
    const double qq = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
    s.qn = sqrt(qq);
    const double iq = qq > 0.0 ? 1.0 / s.qn : 1.0;
    for (int i = 0; i < 4; ++i) s.uq[i] = q[i] * iq;
    {
        const double w = s.uq[0], xx = s.uq[1], y = s.uq[2], zz = s.uq[3];
        s.Rq[0] = 1 - 2 * (y * y + zz * zz); s.Rq[1] = 2 * (xx * y - w * zz);     s.Rq[2] = 2 * (xx * zz + w * y);
        s.Rq[3] = 2 * (xx * y + w * zz);     s.Rq[4] = 1 - 2 * (xx * xx + zz * zz); s.Rq[5] = 2 * (y * zz - w * xx);
        s.Rq[6] = 2 * (xx * zz - w * y);     s.Rq[7] = 2 * (y * zz + w * xx);     s.Rq[8] = 1 - 2 * (xx * xx + y * y);
    }
    const float4 sa = S.scale_amp[gi];
    s.sv[0] = exp((double)sa.x);
    s.sv[1] = exp((double)sa.y);
    s.sv[2] = exp((double)sa.z);
    double M3[9];
    for (int r = 0; r < 3; ++r)
        for (int j = 0; j < 3; ++j) M3[r * 3 + j] = s.Rq[r * 3 + j] * s.sv[j];
    for (int i = 0; i < 3; ++i)
        for (int j = i; j < 3; ++j) {
            s.cov3d[i * 3 + j] = M3[i * 3 + 0] * M3[j * 3 + 0] + M3[i * 3 + 1] * M3[j * 3 + 1] +
                                 M3[i * 3 + 2] * M3[j * 3 + 2];
            s.cov3d[j * 3 + i] = s.cov3d[i * 3 + j];
        }
    // same comparisons as prep64 (splat.cpp:136-140) for the clamp routing
    const double rx = s.p[0] / z, ry = s.p[1] / z;
    s.clx = rx < -C.lim_x || rx > C.lim_x;
    s.cly = ry < -C.lim_y || ry > C.lim_y;
    s.tx = clampd(rx, -C.lim_x, C.lim_x) * z;
    s.ty = clampd(ry, -C.lim_y, C.lim_y) * z;
    const double J[6] = {C.fx * iz, 0.0, -C.fx * s.tx * iz * iz, 0.0, C.fy * iz, -C.fy * s.ty * iz * iz};
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            s.M[i * 3 + j] = J[i * 3 + 0] * R[0 * 3 + j] + J[i * 3 + 1] * R[1 * 3 + j] + J[i * 3 + 2] * R[2 * 3 + j];
    double T23[6];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            T23[i * 3 + j] = s.M[i * 3 + 0] * s.cov3d[0 * 3 + j] + s.M[i * 3 + 1] * s.cov3d[1 * 3 + j] +
                             s.M[i * 3 + 2] * s.cov3d[2 * 3 + j];
    double c2[4];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            c2[i * 2 + j] = T23[i * 3 + 0] * s.M[j * 3 + 0] + T23[i * 3 + 1] * s.M[j * 3 + 1] +
                            T23[i * 3 + 2] * s.M[j * 3 + 2];
    c2[0] += O.dilation;
    c2[3] += O.dilation;
    const double idet = 1.0 / (c2[0] * c2[3] - c2[1] * c2[1]);
    s.ca = c2[3] * idet;
    s.cb = -c2[1] * idet;
    s.cc = c2[0] * idet;
    // the gate 0 < r_raw < 1 must see prep64's exact value
    s.refl_raw = refl_raw64(S, C, gi, x, s.depth, s.view_dir);
}

// Reflectivity SH part of the chain for sh_degree > 0 (out of line so the common
// degree-0 path keeps its register budget): d_refl[k] = b_k d_r, accumulated into the
// SH gradient arrays (coefficients 1..15; coefficient 0 is the caller's), and the
// returned d_dir = Jb^T (refl_sh * d_r) (splat.cpp:579-583).  Arguments and result by
// value: arrays or references would live in the caller's local memory.
__device__ __noinline__ double3 sh_chain(const float4* scale_amp, const float4* sh, int n, int degree, int gi,
                                         double v0, double v1, double v2, double d_r, float4* gs) {
    const double view_dir[3] = {v0, v1, v2};
    double b[16], c[16], Jb[16][3];
    sh_basis64(view_dir, degree, b);
    refl_coeffs(scale_amp, sh, n, gi, c);
    sh_jacobian64(view_dir, degree, Jb);
    for (int a = 0; a < 4; ++a) {
        float4 v = gs[(size_t)a * n];
        const int k = 1 + 4 * a;
        v.x += (float)(b[k] * d_r);
        v.y += (float)(b[k + 1] * d_r);
        v.z += (float)(b[k + 2] * d_r);
        if (a < 3) v.w += (float)(b[k + 3] * d_r);
        gs[(size_t)a * n] = v;
    }
    double d[3];
    for (int a = 0; a < 3; ++a) {
        double t = 0.0;
        for (int k = 0; k < 16; ++k) t += Jb[k][a] * (c[k] * d_r);
        d[a] = t;
    }
    return make_double3(d[0], d[1], d[2]);
}

// ---------------------------------------------------------------------------
// k_chain: per visible Gaussian, chain the 8 screen-space gradients back to the
// parameters (splat.cpp:551-648) in fp64, then through the trajectory
// (trainer.cpp:313-314, 329-331), and accumulate into the scene gradient
// buffer (GroupGrads::add).  Clears the screen-gradient slots it consumed.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128, 4) k_chain(SceneK S, CamK C, OptK O, FrameK F,
                                               const uint32_t* __restrict__ touched,
                                               double* __restrict__ screen,
                                               float4* __restrict__ grads) {
    const int gi = blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= S.n || touched[gi] == 0u) return;
    double g8[8];
    bool any = false;
    for (int c = 0; c < 8; ++c) {
        g8[c] = screen[(size_t)c * S.n + gi];
        any |= g8[c] != 0.0;
    }
    // The chain is linear in the screen-space gradients: a splat no pixel reached
    // (e.g. behind every tile's termination point) contributes exactly nothing.
    if (!any) return;
    for (int c = 0; c < 8; ++c) screen[(size_t)c * S.n + gi] = 0.0;
    Chain64 s;
    chain_prep(S, C, O, F, gi, s);
    const double d_mean0 = g8[0], d_mean1 = g8[1], d_ca = g8[2], d_cb = g8[3], d_cc = g8[4];
    const double d_op = g8[5], d_coef = g8[6], d_dep = g8[7];
    const double* R = C.R;

    const double d_logit = d_op * s.opacity * (1.0 - s.opacity);
    const double r_cl = clampd(s.refl_raw, 0.0, 1.0);
    const double id = 1.0 / s.depth;
    const double id2 = id * id;
    const double d_depth = d_dep + d_coef * (-2.0 * S.s_int * r_cl * id2 * id);
    // reflectivity SH through coef = s_int * r / d^2 (splat.cpp:573-583), gated by 0 < r_raw < 1
    double d_dir[3] = {0.0, 0.0, 0.0};
    double d_amp = 0.0;
    const bool gated = s.refl_raw > 0.0 && s.refl_raw < 1.0;
    if (gated) {
        const double d_r = d_coef * S.s_int * id2;
        d_amp = 0.28209479177387814 * d_r;  // b_0 d_r
        if (S.sh_degree > 0) {
            const double3 dd = sh_chain(S.scale_amp, S.sh, S.n, S.sh_degree, gi, s.view_dir[0], s.view_dir[1],
                                        s.view_dir[2], d_r, grads + (size_t)(3 + S.nk) * S.n + gi);
            d_dir[0] = dd.x;
            d_dir[1] = dd.y;
            d_dir[2] = dd.z;
        }
    }

    const double Q[4] = {s.ca, s.cb, s.cb, s.cc};
    const double GQ[4] = {d_ca, 0.5 * d_cb, 0.5 * d_cb, d_cc};
    double QG[4], G2[4];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) QG[a * 2 + b] = Q[a * 2 + 0] * GQ[0 * 2 + b] + Q[a * 2 + 1] * GQ[1 * 2 + b];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) G2[a * 2 + b] = -(QG[a * 2 + 0] * Q[0 * 2 + b] + QG[a * 2 + 1] * Q[1 * 2 + b]);
    double GM[6], dM[6], MtG[6], G3[9];
    for (int a = 0; a < 2; ++a)
        for (int j = 0; j < 3; ++j) GM[a * 3 + j] = G2[a * 2 + 0] * s.M[0 * 3 + j] + G2[a * 2 + 1] * s.M[1 * 3 + j];
    for (int a = 0; a < 2; ++a)
        for (int j = 0; j < 3; ++j) {
            double t = 0;
            for (int k = 0; k < 3; ++k) t += (2.0 * GM[a * 3 + k]) * s.cov3d[k * 3 + j];
            dM[a * 3 + j] = t;
        }
    for (int i = 0; i < 3; ++i)
        for (int b = 0; b < 2; ++b) MtG[i * 2 + b] = s.M[0 * 3 + i] * G2[0 * 2 + b] + s.M[1 * 3 + i] * G2[1 * 2 + b];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) G3[i * 3 + j] = MtG[i * 2 + 0] * s.M[0 * 3 + j] + MtG[i * 2 + 1] * s.M[1 * 3 + j];
    double dJ[6];
    for (int a = 0; a < 2; ++a)
        for (int j = 0; j < 3; ++j)
            dJ[a * 3 + j] = dM[a * 3 + 0] * R[j * 3 + 0] + dM[a * 3 + 1] * R[j * 3 + 1] + dM[a * 3 + 2] * R[j * 3 + 2];
    const double z = s.p[2], iz = 1.0 / z, iz2 = iz * iz, iz3 = iz2 * iz;
    double dp[3] = {0, 0, 0};
    const double dtx = dJ[2] * (-C.fx * iz2);
    const double dty = dJ[5] * (-C.fy * iz2);
    dp[2] += dJ[0] * (-C.fx * iz2) + dJ[4] * (-C.fy * iz2) + dJ[2] * (2.0 * C.fx * s.tx * iz3) +
             dJ[5] * (2.0 * C.fy * s.ty * iz3);
    if (s.clx) dp[2] += dtx * (s.tx * iz); else dp[0] += dtx;
    if (s.cly) dp[2] += dty * (s.ty * iz); else dp[1] += dty;
    dp[0] += d_mean0 * C.fx * iz;
    dp[2] += d_mean0 * (-C.fx * s.p[0] * iz2);
    dp[1] += d_mean1 * C.fy * iz;
    dp[2] += d_mean1 * (-C.fy * s.p[1] * iz2);
    for (int a = 0; a < 3; ++a) dp[a] += d_depth * (s.p[a] * id);
    // view_dir = (x - C)/|x - C| feeds the world position directly (splat.cpp:619-622)
    const double vd = s.view_dir[0] * d_dir[0] + s.view_dir[1] * d_dir[1] + s.view_dir[2] * d_dir[2];
    double dpos[3];
    for (int a = 0; a < 3; ++a)
        dpos[a] = (d_dir[a] - s.view_dir[a] * vd) * id + R[0 * 3 + a] * dp[0] + R[1 * 3 + a] * dp[1] +
                  R[2 * 3 + a] * dp[2];

    // cov3d = M3 M3^T, M3 = R(q) diag(exp(log_scale))
    double M3[9], dM3[9];
    for (int rr = 0; rr < 3; ++rr)
        for (int j = 0; j < 3; ++j) M3[rr * 3 + j] = s.Rq[rr * 3 + j] * s.sv[j];
    for (int rr = 0; rr < 3; ++rr)
        for (int j = 0; j < 3; ++j) {
            double t = 0;
            for (int k = 0; k < 3; ++k) t += (2.0 * G3[rr * 3 + k]) * M3[k * 3 + j];
            dM3[rr * 3 + j] = t;
        }
    double dls[3];
    for (int j = 0; j < 3; ++j) {
        double ds = 0;
        for (int rr = 0; rr < 3; ++rr) ds += s.Rq[rr * 3 + j] * dM3[rr * 3 + j];
        dls[j] = ds * s.sv[j];
    }
    double dRq[9];
    for (int rr = 0; rr < 3; ++rr)
        for (int j = 0; j < 3; ++j) dRq[rr * 3 + j] = dM3[rr * 3 + j] * s.sv[j];
    const double w = s.uq[0], x = s.uq[1], y = s.uq[2], zq = s.uq[3];
    const double dR[4][9] = {{0, -zq, y, zq, 0, -x, -y, x, 0},
                             {0, y, zq, y, -2 * x, -w, zq, w, -2 * x},
                             {-2 * y, x, w, x, 0, zq, -w, zq, -2 * y},
                             {-2 * zq, -w, x, w, -2 * zq, y, x, y, 0}};
    double duq[4];
    for (int c = 0; c < 4; ++c) {
        double t = 0;
        for (int k = 0; k < 9; ++k) t += dRq[k] * dR[c][k];
        duq[c] = 2.0 * t;
    }
    const double ud = s.uq[0] * duq[0] + s.uq[1] * duq[1] + s.uq[2] * duq[2] + s.uq[3] * duq[3];
    const double iqn = 1.0 / s.qn;
    double dq[4];
    for (int c = 0; c < 4; ++c) dq[c] = (duq[c] - s.uq[c] * ud) * iqn;

    // accumulate (GroupGrads::add; canonical += dXi + dXip1 == dP)
    const int n = S.n;
    float4 g0 = grads[gi];
    g0.x += (float)dpos[0]; g0.y += (float)dpos[1]; g0.z += (float)dpos[2]; g0.w += (float)d_logit;
    grads[gi] = g0;
    float4 g1 = grads[n + gi];
    g1.x += (float)dls[0]; g1.y += (float)dls[1]; g1.z += (float)dls[2]; g1.w += (float)d_amp;
    grads[n + gi] = g1;
    float4 g2 = grads[2 * n + gi];
    g2.x += (float)dq[0]; g2.y += (float)dq[1]; g2.z += (float)dq[2]; g2.w += (float)dq[3];
    grads[2 * n + gi] = g2;
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

void launch_chain(const SceneK& S, const CamK& C, const OptK& O, const FrameK& F,
                  const uint32_t* touched, double* screen, float4* grads, cudaStream_t st) {
    if (S.n <= 0) return;
    const int bs = 128;
    k_chain<<<(S.n + bs - 1) / bs, bs, 0, st>>>(S, C, O, F, touched, screen, grads);
}

}  // namespace tsb
