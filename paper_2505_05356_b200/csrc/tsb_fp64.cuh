// fp64 per-Gaussian preprocess shared by the preprocess, fp64 fix-up and chain
// kernels.  This TU family is compiled with -fmad=false so that every double
// operation rounds exactly as written, in the same order as the reference
// RenderPassImpl::prepare (proj/src/splat.cpp:105-177) and the CPU oracle
// (oracle/tofsplat_oracle.c prepare()).  Integer outcomes (cull, tile rect,
// global (depth, index) order) are therefore bit-identical to the oracle.
#pragma once

#include "tsb_internal.h"

namespace tsb {

// sh_basis (sh.hpp:26-50), same expressions and evaluation order as the oracle.
__device__ __forceinline__ void sh_basis64(const double* d, int degree, double* b) {
    const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
    const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                          0.5462742152960396};
    const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                          -0.4570457994644658, 1.445305721320277, -0.5900435899266435};
    const double x = d[0], y = d[1], z = d[2];
    for (int k = 0; k < 16; ++k) b[k] = 0.0;
    b[0] = C0;
    if (degree < 1) return;
    b[1] = -C1 * y;
    b[2] = C1 * z;
    b[3] = -C1 * x;
    if (degree < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    b[4] = C2[0] * x * y;
    b[5] = C2[1] * y * z;
    b[6] = C2[2] * (2.0 * zz - xx - yy);
    b[7] = C2[3] * x * z;
    b[8] = C2[4] * (xx - yy);
    if (degree < 3) return;
    b[9] = C3[0] * y * (3.0 * xx - yy);
    b[10] = C3[1] * x * y * z;
    b[11] = C3[2] * y * (4.0 * zz - xx - yy);
    b[12] = C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    b[13] = C3[4] * x * (4.0 * zz - xx - yy);
    b[14] = C3[5] * z * (xx - yy);
    b[15] = C3[6] * x * (xx - 3.0 * yy);
}

// sh_basis_jacobian (sh.hpp:53-79): J[k][a] = d b_k / d dir_a.
__device__ __forceinline__ void sh_jacobian64(const double* d, int degree, double J[16][3]) {
    const double C1 = 0.4886025119029199;
    const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                          0.5462742152960396};
    const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                          -0.4570457994644658, 1.445305721320277, -0.5900435899266435};
    const double x = d[0], y = d[1], z = d[2];
    for (int k = 0; k < 16; ++k) J[k][0] = J[k][1] = J[k][2] = 0.0;
    if (degree < 1) return;
    J[1][1] = -C1;
    J[2][2] = C1;
    J[3][0] = -C1;
    if (degree < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    J[4][0] = C2[0] * y; J[4][1] = C2[0] * x;
    J[5][1] = C2[1] * z; J[5][2] = C2[1] * y;
    J[6][0] = -2.0 * C2[2] * x; J[6][1] = -2.0 * C2[2] * y; J[6][2] = 4.0 * C2[2] * z;
    J[7][0] = C2[3] * z; J[7][2] = C2[3] * x;
    J[8][0] = 2.0 * C2[4] * x; J[8][1] = -2.0 * C2[4] * y;
    if (degree < 3) return;
    J[9][0] = C3[0] * 6.0 * x * y; J[9][1] = C3[0] * (3.0 * xx - 3.0 * yy);
    J[10][0] = C3[1] * y * z; J[10][1] = C3[1] * x * z; J[10][2] = C3[1] * x * y;
    J[11][0] = -2.0 * C3[2] * x * y; J[11][1] = C3[2] * (4.0 * zz - xx - 3.0 * yy); J[11][2] = 8.0 * C3[2] * y * z;
    J[12][0] = -6.0 * C3[3] * x * z; J[12][1] = -6.0 * C3[3] * y * z;
    J[12][2] = C3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
    J[13][0] = C3[4] * (4.0 * zz - 3.0 * xx - yy); J[13][1] = -2.0 * C3[4] * x * y; J[13][2] = 8.0 * C3[4] * x * z;
    J[14][0] = 2.0 * C3[5] * x * z; J[14][1] = -2.0 * C3[5] * y * z; J[14][2] = C3[5] * (xx - yy);
    J[15][0] = C3[6] * (3.0 * xx - 3.0 * yy); J[15][1] = -6.0 * C3[6] * x * y;
}

// The 16 reflectivity SH coefficients of Gaussian gi (coefficient 0 lives in scale_amp.w).
__device__ __forceinline__ void refl_coeffs(const float4* __restrict__ scale_amp, const float4* __restrict__ sh, int n,
                                            int gi, double* c) {
    c[0] = (double)scale_amp[gi].w;
    for (int a = 0; a < 4; ++a) {
        const float4 v = sh[(size_t)a * n + gi];
        const int k = 1 + 4 * a;
        c[k] = v.x;
        c[k + 1] = v.y;
        c[k + 2] = v.z;
        if (a < 3) c[k + 3] = v.w;
    }
}

// sum_k refl_sh[k] b_k(view_dir) for sh_degree > 0 (out of line: keeps the
// degree-0 kernels' register budget).  Scalar arguments only: a SceneK reference
// would make every caller copy the struct to its stack at entry.
static __device__ __noinline__ double refl_sh_eval(const float4* scale_amp, const float4* sh, int n, int degree,
                                                   int gi, double v0, double v1, double v2) {
    const double v[3] = {v0, v1, v2};
    double b[16], c[16];
    sh_basis64(v, degree, b);
    refl_coeffs(scale_amp, sh, n, gi, c);
    double rr = 0.0;
    for (int k = 0; k < 16; ++k) rr += c[k] * b[k];
    return rr;
}

// view_dir = (x - center) / depth and r_raw = sum_k refl_sh[k] b[k] (splat.cpp:163-165).
__device__ __forceinline__ double refl_raw64(const SceneK& S, const CamK& C, int gi, const double* x, double depth,
                                             double* view_dir) {
    if (S.sh_degree == 0) {  // view_dir does not enter (its chain term is multiplied by zero)
        view_dir[0] = view_dir[1] = view_dir[2] = 0.0;
        return (double)S.scale_amp[gi].w * 0.28209479177387814;
    }
    for (int i = 0; i < 3; ++i) view_dir[i] = (x[i] - C.center[i]) / depth;
    return refl_sh_eval(S.scale_amp, S.sh, S.n, S.sh_degree, gi, view_dir[0], view_dir[1], view_dir[2]);
}

struct Prep64 {
    double x[3];  // rendered world mean (trajectory-interpolated)
    double p[3];  // camera-space mean
    double depth; // Euclidean distance (splat.cpp:124)
    double opacity;
    double mean[2];
    double ca, cb, cc;
    double c11;  // dilated cov2d(1,1): l22 = 1/sqrt(c11)
    double coef;
    double refl_raw;
    double view_dir[3];
    double M[6];      // J W (2x3 row-major)
    double cov3d[9];  // row-major
    double tx, ty;
    bool clx, cly;
    int x0, x1, y0, y1;
};

__device__ __forceinline__ int d2i_like_x86(double v) {
    // static_cast<int>(std::floor(..)) on x86-64: out-of-range -> INT_MIN
    if (!(v >= -2147483648.0 && v < 2147483648.0)) return (int)0x80000000u;
    return (int)v;
}

// 1/x to a few ulps: hardware approximation + two Newton steps (no correctly rounded
// division and its slow path) -- only for values that end in an fp32 record.
__device__ __forceinline__ double rcp64(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    return fma(r, fma(-x, r, 1.0), r);
}

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

// Rendered mean at the frame (trainer.cpp:259-279): Xi = x + d_k, Xip1 = x + d_{k+1},
// P = (w == 0) ? Xi : (1 - w) Xi + w Xip1.
__device__ __forceinline__ void frame_mean(const SceneK& S, const FrameK& F, int gi, double* x) {
    const float4 po = S.pos_op[gi];
    const double c[3] = {(double)po.x, (double)po.y, (double)po.z};
    if (S.nk == 0) {
        x[0] = c[0]; x[1] = c[1]; x[2] = c[2];
        return;
    }
    const float4 da = S.motion[(size_t)F.key * S.n + gi];
    const float4 db = S.motion[(size_t)(F.key + 1) * S.n + gi];
    const double a[3] = {(double)da.x, (double)da.y, (double)da.z};
    const double b[3] = {(double)db.x, (double)db.y, (double)db.z};
    for (int i = 0; i < 3; ++i) {
        const double Xi = c[i] + a[i];
        const double Xip1 = c[i] + b[i];
        x[i] = (F.w == 0.0) ? Xi : (1.0 - F.w) * Xi + F.w * Xip1;
    }
}

// quat_to_rotation (scene.cpp:10-18) with Eigen::normalized semantics.
__device__ __forceinline__ void quat_rot(const double* q, double* u, double* R) {
    const double z = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
    if (z > 0.0) {
        const double n = sqrt(z);
        for (int i = 0; i < 4; ++i) u[i] = q[i] / n;
    } else {
        for (int i = 0; i < 4; ++i) u[i] = q[i];
    }
    const double w = u[0], x = u[1], y = u[2], zz = u[3];
    R[0] = 1 - 2 * (y * y + zz * zz); R[1] = 2 * (x * y - w * zz);    R[2] = 2 * (x * zz + w * y);
    R[3] = 2 * (x * y + w * zz);     R[4] = 1 - 2 * (x * x + zz * zz); R[5] = 2 * (y * zz - w * x);
    R[6] = 2 * (x * zz - w * y);     R[7] = 2 * (y * zz + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

// opacity = sigmoid(logit) (scene.hpp:14-15)
__device__ __forceinline__ double opacity64(const SceneK& S, int gi) {
    return 1.0 / (1.0 + exp(-(double)S.pos_op[gi].w));
}

// cov3d = M3 M3^T, M3 = R(q) diag(exp(log_scale)) (scene.cpp:20-33), row-major 3x3.
__device__ __forceinline__ void cov3d64(const SceneK& S, int gi, double* cov3d) {
    const float4 qf = S.quat[gi];
    const double q[4] = {(double)qf.x, (double)qf.y, (double)qf.z, (double)qf.w};
    double u[4], Rq[9];
    quat_rot(q, u, Rq);
    const float4 sa = S.scale_amp[gi];
    const double sv[3] = {exp((double)sa.x), exp((double)sa.y), exp((double)sa.z)};
    double M3[9];
    for (int r = 0; r < 3; ++r)
        for (int j = 0; j < 3; ++j) M3[r * 3 + j] = Rq[r * 3 + j] * sv[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            cov3d[i * 3 + j] = M3[i * 3 + 0] * M3[j * 3 + 0] + M3[i * 3 + 1] * M3[j * 3 + 1] +
                               M3[i * 3 + 2] * M3[j * 3 + 2];
}

// RenderPassImpl::prepare for one Gaussian (splat.cpp:114-176).  Returns true when
// the splat survives culling.  EXACT: every value rounds as the reference's (the fp64
// fix-up decides with them).  !EXACT (the preprocess): the values that only feed the
// fp32 raster record -- the conic and coef -- come from one reciprocal of det and of
// depth^2 instead of four correctly rounded divisions (a few fp64 ulps, far below the
// fp32 rounding of the record); cc is not formed.  Every decision (culls, clamps, rect,
// depth order) still uses exactly rounded values.
template <bool EXACT = true>
__device__ __forceinline__ bool prep64(const SceneK& S, const CamK& C, const OptK& O,
                                       const FrameK& F, int gi, Prep64& s) {
    frame_mean(S, F, gi, s.x);
    const double* R = C.R;
    for (int i = 0; i < 3; ++i)
        s.p[i] = R[i * 3 + 0] * s.x[0] + R[i * 3 + 1] * s.x[1] + R[i * 3 + 2] * s.x[2] + C.t[i];
    if (s.p[2] < C.near_plane) return false;
    s.depth = sqrt(s.p[0] * s.p[0] + s.p[1] * s.p[1] + s.p[2] * s.p[2]);
    s.opacity = S.opac ? S.opac[gi] : opacity64(S, gi);
    if (s.opacity < O.alpha_thr) return false;

    const double z = s.p[2];
    s.mean[0] = C.fx * s.p[0] / z + C.cx;
    s.mean[1] = C.fy * s.p[1] / z + C.cy;

    if (S.cov6) {
        const size_t n = (size_t)S.n;
        const double c00 = S.cov6[gi], c01 = S.cov6[n + gi], c02 = S.cov6[2 * n + gi];
        const double c11 = S.cov6[3 * n + gi], c12 = S.cov6[4 * n + gi], c22 = S.cov6[5 * n + gi];
        s.cov3d[0] = c00; s.cov3d[1] = c01; s.cov3d[2] = c02;
        s.cov3d[3] = c01; s.cov3d[4] = c11; s.cov3d[5] = c12;
        s.cov3d[6] = c02; s.cov3d[7] = c12; s.cov3d[8] = c22;
    } else {
        cov3d64(S, gi, s.cov3d);
    }
    const double rx = s.p[0] / z, ry = s.p[1] / z;
    s.clx = rx < -C.lim_x || rx > C.lim_x;
    s.cly = ry < -C.lim_y || ry > C.lim_y;
    s.tx = clampd(rx, -C.lim_x, C.lim_x) * z;
    s.ty = clampd(ry, -C.lim_y, C.lim_y) * z;
    double J[6];
    J[0] = C.fx / z; J[1] = 0.0; J[2] = -C.fx * s.tx / (z * z);
    J[3] = 0.0; J[4] = C.fy / z; J[5] = -C.fy * s.ty / (z * z);
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
    const double det = c2[0] * c2[3] - c2[1] * c2[1];
    if (!(det > 0.0)) return false;
    if (EXACT) {
        s.ca = c2[3] / det;
        s.cb = -c2[1] / det;
        s.cc = c2[0] / det;
    } else {
        const double idet = rcp64(det);
        s.ca = c2[3] * idet;
        s.cb = -c2[1] * idet;
        s.cc = 0.0;
    }
    s.c11 = c2[3];
    const double mid = 0.5 * (c2[0] + c2[3]);
    const double disc = mid * mid - det;
    const double lam_max = mid + sqrt(disc > 0.1 ? disc : 0.1);
    const double radius = O.sigma_cutoff * sqrt(lam_max);
    int v;
    v = d2i_like_x86(floor(s.mean[0] - radius)); s.x0 = v > 0 ? v : 0;
    v = d2i_like_x86(ceil(s.mean[0] + radius)) + 1; s.x1 = v < C.W ? v : C.W;
    v = d2i_like_x86(floor(s.mean[1] - radius)); s.y0 = v > 0 ? v : 0;
    v = d2i_like_x86(ceil(s.mean[1] + radius)) + 1; s.y1 = v < C.H ? v : C.H;
    if (s.x0 >= s.x1 || s.y0 >= s.y1) return false;

    // view-dependent reflectivity (sh.hpp:26-50; splat.cpp:163-167)
    s.refl_raw = refl_raw64(S, C, gi, s.x, s.depth, s.view_dir);
    const double r = clampd(s.refl_raw, 0.0, 1.0);
    s.coef = EXACT ? S.s_int * r / (s.depth * s.depth) : S.s_int * r * rcp64(s.depth * s.depth);
    return true;
}

// phase_of_depth (tof.hpp:41-43) and its derivative (splat.cpp:171).
__device__ __forceinline__ double phase_of_depth(double depth, double f, double c) {
    return 4.0 * M_PI * depth * f / c;
}

// fp64 record of a visible Gaussian for the pixel fix-up (tsb_geom.cu) and the
// fp64-fixed pixels of the colour / flow channels (tsb_ext.cu).
__device__ __forceinline__ Rec64 make_rec64(const SceneK& S, const CamK& C, const OptK& O, const FrameK& F, int g) {
    Prep64 s;
    prep64(S, C, O, F, g, s);  // visible by construction
    Rec64 r;
    r.m0 = make_double4(s.mean[0], s.mean[1], s.ca, s.cb);
    r.m1 = make_double4(s.cc, s.opacity, s.coef, s.depth);
    r.rect = make_int4(s.x0, s.x1, s.y0, s.y1);
    return r;
}

}  // namespace tsb
