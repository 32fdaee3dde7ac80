/*
 * tofsplat_oracle.c -- TEST INFRASTRUCTURE: double-precision CPU restatement of
 * the reference's render/optimise hot path.  See tofsplat_oracle.h for scope
 * and for the rule that only tests/, smoke() and bench.py's CPU legs use it.
 *
 * Built with -ffp-contract=off so every double operation rounds exactly as
 * written; the B200 fp64 preprocess (paper_2505_05356_b200/csrc/tsb_fp64.cuh)
 * is compiled without FMA contraction and follows the same operation order,
 * which is what makes tile rects / sort order / tile lists comparable bit for bit.
 * Eigen's internal reduction order for the reference's 3x3 products may differ
 * from the sequential order used here by one ulp; that only
 * moves integer outcomes in measure-zero cases.
 */
#include "tofsplat_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define SHN 16

static __thread char g_err[256];
static void set_err(const char* m) { snprintf(g_err, sizeof g_err, "%s", m); }
const char* orc_last_error(void) { return g_err; }

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ---- L1 math: sh.hpp:13-79, scene.cpp:10-27 ---------------------------- */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

void orc_sh_basis(const double* d, int degree, double* b) {
    const double x = d[0], y = d[1], z = d[2];
    memset(b, 0, sizeof(double) * SHN);
    b[0] = SH_C0;
    if (degree < 1) return;
    b[1] = -SH_C1 * y;
    b[2] = SH_C1 * z;
    b[3] = -SH_C1 * x;
    if (degree < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    b[4] = SH_C2[0] * x * y;
    b[5] = SH_C2[1] * y * z;
    b[6] = SH_C2[2] * (2.0 * zz - xx - yy);
    b[7] = SH_C2[3] * x * z;
    b[8] = SH_C2[4] * (xx - yy);
    if (degree < 3) return;
    b[9] = SH_C3[0] * y * (3.0 * xx - yy);
    b[10] = SH_C3[1] * x * y * z;
    b[11] = SH_C3[2] * y * (4.0 * zz - xx - yy);
    b[12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    b[13] = SH_C3[4] * x * (4.0 * zz - xx - yy);
    b[14] = SH_C3[5] * z * (xx - yy);
    b[15] = SH_C3[6] * x * (xx - 3.0 * yy);
}

void orc_sh_basis_jacobian(const double* d, int degree, double* J) {
    const double x = d[0], y = d[1], z = d[2];
    memset(J, 0, sizeof(double) * SHN * 3);
#define JS(r, a, b, c) (J[(r) * 3 + 0] = (a), J[(r) * 3 + 1] = (b), J[(r) * 3 + 2] = (c))
    if (degree < 1) return;
    J[1 * 3 + 1] = -SH_C1;
    J[2 * 3 + 2] = SH_C1;
    J[3 * 3 + 0] = -SH_C1;
    if (degree < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    JS(4, SH_C2[0] * y, SH_C2[0] * x, 0.0);
    JS(5, 0.0, SH_C2[1] * z, SH_C2[1] * y);
    JS(6, -2.0 * SH_C2[2] * x, -2.0 * SH_C2[2] * y, 4.0 * SH_C2[2] * z);
    JS(7, SH_C2[3] * z, 0.0, SH_C2[3] * x);
    JS(8, 2.0 * SH_C2[4] * x, -2.0 * SH_C2[4] * y, 0.0);
    if (degree < 3) return;
    JS(9, SH_C3[0] * 6.0 * x * y, SH_C3[0] * (3.0 * xx - 3.0 * yy), 0.0);
    JS(10, SH_C3[1] * y * z, SH_C3[1] * x * z, SH_C3[1] * x * y);
    JS(11, -2.0 * SH_C3[2] * x * y, SH_C3[2] * (4.0 * zz - xx - 3.0 * yy), 8.0 * SH_C3[2] * y * z);
    JS(12, -6.0 * SH_C3[3] * x * z, -6.0 * SH_C3[3] * y * z,
       SH_C3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy));
    JS(13, SH_C3[4] * (4.0 * zz - 3.0 * xx - yy), -2.0 * SH_C3[4] * x * y, 8.0 * SH_C3[4] * x * z);
    JS(14, 2.0 * SH_C3[5] * x * z, -2.0 * SH_C3[5] * y * z, SH_C3[5] * (xx - yy));
    JS(15, SH_C3[6] * (3.0 * xx - 3.0 * yy), -6.0 * SH_C3[6] * x * y, 0.0);
#undef JS
}

/* Vector4 squaredNorm, evaluated left to right. */
static double sqnorm4(const double* q) { return q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]; }

static void normalize4(const double* q, double* u) {
    const double z = sqnorm4(q);
    if (z > 0.0) {
        const double n = sqrt(z);
        for (int i = 0; i < 4; ++i) u[i] = q[i] / n;
    } else {
        for (int i = 0; i < 4; ++i) u[i] = q[i];
    }
}

void orc_quat_to_rotation(const double* q, double* R) {
    double u[4];
    normalize4(q, u);
    const double w = u[0], x = u[1], y = u[2], z = u[3];
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

/* quat_rotation_jacobian (scene.cpp:20-27), dR[c] row-major. */
static void quat_rot_jac(const double* uq, double dR[4][9]) {
    const double w = uq[0], x = uq[1], y = uq[2], z = uq[3];
    const double a[4][9] = {{0, -z, y, z, 0, -x, -y, x, 0},
                            {0, y, z, y, -2 * x, -w, z, w, -2 * x},
                            {-2 * y, x, w, x, 0, z, -w, z, -2 * y},
                            {-2 * z, -w, x, w, -2 * z, y, x, y, 0}};
    for (int c = 0; c < 4; ++c)
        for (int k = 0; k < 9; ++k) dR[c][k] = a[c][k] * 2.0;
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* ---- Prepared (splat.cpp:32-55) ---------------------------------------- */
typedef struct {
    int gidx;
    double p_cam[3];
    double depth;
    double mean2d[2];
    double conic_a, conic_b, conic_c;
    double opacity, coef, sin_psi, cos_psi, dpsi_dd;
    int x0, x1, y0, y1;
    double M[6];     /* 2x3 row-major */
    double cov3d[9]; /* row-major */
    double tx, ty;
    int clamp_x, clamp_y;
    double view_dir[3];
    double refl_raw;
    double sh_b[SHN];
    double color_raw[3], color[3];  /* splat.cpp:172-173 */
    double mf[3], mb[3];            /* splat.cpp:174-175 */
} Prepared;

struct orc_pass {
    orc_scene scene;
    orc_camera cam;
    orc_options opt;
    Prepared* prep;
    int nvis;
    int tiles_x, tiles_y;
    int64_t* tile_off; /* ntiles+1 */
    int32_t* tile_ids;
};

static int cmp_prepared(const void* a, const void* b) {
    const Prepared* x = (const Prepared*)a;
    const Prepared* y = (const Prepared*)b;
    /* splat.cpp:181-184: depth ascending, index breaks exact ties */
    if (x->depth != y->depth) return x->depth < y->depth ? -1 : 1;
    return (x->gidx > y->gidx) - (x->gidx < y->gidx);
}

static int cam_valid(const orc_camera* c) {
    return c->fx > 0 && c->fy > 0 && c->width > 0 && c->height > 0 && c->near_plane > 0 &&
           c->far_plane > c->near_plane;
}

/* Double -> int the way x86-64 cvttsd2si behaves for the reference's
 * static_cast<int>(std::floor(...)) (out-of-range -> INT_MIN). */
static int to_int(double v) {
    if (!(v >= -2147483648.0 && v < 2147483648.0)) return (int)0x80000000u;
    return (int)v;
}

/* RenderPassImpl::prepare (splat.cpp:105-185) */
static void prepare(orc_pass* P) {
    const orc_scene* sc = &P->scene;
    const orc_camera* cam = &P->cam;
    const orc_options* opt = &P->opt;
    const double* R = cam->R;
    const double lim_x = 1.3 * (0.5 * cam->width / cam->fx);
    const double lim_y = 1.3 * (0.5 * cam->height / cam->fy);
    /* optical_center = -(R^T t) */
    double center[3];
    for (int i = 0; i < 3; ++i)
        center[i] = -(R[0 * 3 + i] * cam->t[0] + R[1 * 3 + i] * cam->t[1] + R[2 * 3 + i] * cam->t[2]);

    P->prep = (Prepared*)malloc(sizeof(Prepared) * (sc->n > 0 ? sc->n : 1));
    int nv = 0;
    for (int gi = 0; gi < sc->n; ++gi) {
        const double* x = sc->position + 3 * gi;
        double p[3];
        for (int i = 0; i < 3; ++i)
            p[i] = R[i * 3 + 0] * x[0] + R[i * 3 + 1] * x[1] + R[i * 3 + 2] * x[2] + cam->t[i];
        if (p[2] < cam->near_plane) continue;

        Prepared s;
        memset(&s, 0, sizeof s);
        s.gidx = gi;
        memcpy(s.p_cam, p, sizeof p);
        s.depth = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
        s.opacity = 1.0 / (1.0 + exp(-sc->opacity_logit[gi]));
        if (s.opacity < opt->alpha_threshold) continue;

        const double z = p[2];
        s.mean2d[0] = cam->fx * p[0] / z + cam->cx;
        s.mean2d[1] = cam->fy * p[1] / z + cam->cy;

        double Rq[9];
        orc_quat_to_rotation(sc->rotation + 4 * gi, Rq);
        double sv[3];
        for (int j = 0; j < 3; ++j) sv[j] = exp(sc->log_scale[3 * gi + j]);
        double M3[9];
        for (int r = 0; r < 3; ++r)
            for (int j = 0; j < 3; ++j) M3[r * 3 + j] = Rq[r * 3 + j] * sv[j];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                s.cov3d[i * 3 + j] =
                    M3[i * 3 + 0] * M3[j * 3 + 0] + M3[i * 3 + 1] * M3[j * 3 + 1] + M3[i * 3 + 2] * M3[j * 3 + 2];
        const double rx = p[0] / z, ry = p[1] / z;
        s.clamp_x = rx < -lim_x || rx > lim_x;
        s.clamp_y = ry < -lim_y || ry > lim_y;
        s.tx = clampd(rx, -lim_x, lim_x) * z;
        s.ty = clampd(ry, -lim_y, lim_y) * z;
        double J[6];
        J[0] = cam->fx / z; J[1] = 0.0; J[2] = -cam->fx * s.tx / (z * z);
        J[3] = 0.0; J[4] = cam->fy / z; J[5] = -cam->fy * s.ty / (z * z);
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 3; ++j)
                s.M[i * 3 + j] = J[i * 3 + 0] * R[0 * 3 + j] + J[i * 3 + 1] * R[1 * 3 + j] + J[i * 3 + 2] * R[2 * 3 + j];
        /* cov2d = (M cov3d) M^T */
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
        c2[0] += opt->dilation;
        c2[3] += opt->dilation;
        const double det = c2[0] * c2[3] - c2[1] * c2[1];
        if (!(det > 0.0)) continue;
        s.conic_a = c2[3] / det;
        s.conic_b = -c2[1] / det;
        s.conic_c = c2[0] / det;

        const double mid = 0.5 * (c2[0] + c2[3]);
        const double disc = mid * mid - det;
        const double lam_max = mid + sqrt(disc > 0.1 ? disc : 0.1);
        const double radius = opt->sigma_cutoff * sqrt(lam_max);
        int v;
        v = to_int(floor(s.mean2d[0] - radius)); s.x0 = v > 0 ? v : 0;
        v = to_int(ceil(s.mean2d[0] + radius)) + 1; s.x1 = v < cam->width ? v : cam->width;
        v = to_int(floor(s.mean2d[1] - radius)); s.y0 = v > 0 ? v : 0;
        v = to_int(ceil(s.mean2d[1] + radius)) + 1; s.y1 = v < cam->height ? v : cam->height;
        if (s.x0 >= s.x1 || s.y0 >= s.y1) continue;

        for (int i = 0; i < 3; ++i) s.view_dir[i] = (x[i] - center[i]) / s.depth;
        orc_sh_basis(s.view_dir, sc->sh_degree, s.sh_b);
        double rr = 0.0;
        for (int k = 0; k < SHN; ++k) rr += sc->refl_sh[SHN * gi + k] * s.sh_b[k];
        s.refl_raw = rr;
        const double r = clampd(rr, 0.0, 1.0);
        s.coef = sc->source_intensity * r / (s.depth * s.depth);
        const double psi = 4.0 * M_PI * s.depth * sc->modulation_frequency / sc->speed_of_light;
        s.sin_psi = sin(psi);
        s.cos_psi = cos(psi);
        s.dpsi_dd = 4.0 * M_PI * sc->modulation_frequency / sc->speed_of_light;
        for (int c = 0; c < 3; ++c) {  /* color_raw = color_sh^T sh_b, clamped to [0, 1] */
            double cr = 0.0;
            if (sc->color_sh)
                for (int k = 0; k < SHN; ++k) cr += sc->color_sh[48 * (size_t)gi + SHN * c + k] * s.sh_b[k];
            s.color_raw[c] = cr;
            s.color[c] = clampd(cr, 0.0, 1.0);
            s.mf[c] = sc->motion_fwd ? sc->motion_fwd[3 * gi + c] : 0.0;
            s.mb[c] = sc->motion_bwd ? sc->motion_bwd[3 * gi + c] : 0.0;
        }
        P->prep[nv++] = s;
    }
    P->nvis = nv;
    qsort(P->prep, (size_t)nv, sizeof(Prepared), cmp_prepared);
}

/* build_tiles (splat.cpp:187-200), CSR instead of vector<vector<int>>. */
static void build_tiles(orc_pass* P) {
    const int ts = P->opt.tile_size > 1 ? P->opt.tile_size : 1;
    P->tiles_x = (P->cam.width + ts - 1) / ts;
    P->tiles_y = (P->cam.height + ts - 1) / ts;
    const int nt = P->tiles_x * P->tiles_y;
    P->tile_off = (int64_t*)calloc((size_t)nt + 1, sizeof(int64_t));
    for (int i = 0; i < P->nvis; ++i) {
        const Prepared* s = &P->prep[i];
        const int tx0 = s->x0 / ts, tx1 = (s->x1 - 1) / ts;
        const int ty0 = s->y0 / ts, ty1 = (s->y1 - 1) / ts;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) P->tile_off[ty * P->tiles_x + tx + 1]++;
    }
    for (int t = 0; t < nt; ++t) P->tile_off[t + 1] += P->tile_off[t];
    P->tile_ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(P->tile_off[nt] > 0 ? P->tile_off[nt] : 1));
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nt > 0 ? nt : 1));
    memcpy(cur, P->tile_off, sizeof(int64_t) * (size_t)nt);
    for (int i = 0; i < P->nvis; ++i) {
        const Prepared* s = &P->prep[i];
        const int tx0 = s->x0 / ts, tx1 = (s->x1 - 1) / ts;
        const int ty0 = s->y0 / ts, ty1 = (s->y1 - 1) / ts;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) P->tile_ids[cur[ty * P->tiles_x + tx]++] = i;
    }
    free(cur);
}

orc_pass* orc_pass_create(const orc_scene* scene, const orc_camera* cam, const orc_options* opt) {
    if (!scene || !cam) { set_err("render: scene and camera required"); return NULL; }
    if (!cam_valid(cam)) { set_err("render: invalid camera"); return NULL; }
    orc_pass* P = (orc_pass*)calloc(1, sizeof(orc_pass));
    P->scene = *scene;
    P->cam = *cam;
    P->opt = *opt;
    prepare(P);
    build_tiles(P);
    return P;
}

void orc_pass_destroy(orc_pass* P) {
    if (!P) return;
    free(P->prep);
    free(P->tile_off);
    free(P->tile_ids);
    free(P);
}

int32_t orc_pass_visible_count(const orc_pass* P) { return P->nvis; }
void orc_pass_tiles(const orc_pass* P, int32_t* tx, int32_t* ty) { *tx = P->tiles_x; *ty = P->tiles_y; }
int64_t orc_pass_num_keys(const orc_pass* P) { return P->tile_off[P->tiles_x * P->tiles_y]; }

void orc_pass_prepared(const orc_pass* P, int32_t* gidx, int32_t* rect, double* rec) {
    for (int i = 0; i < P->nvis; ++i) {
        const Prepared* s = &P->prep[i];
        if (gidx) gidx[i] = s->gidx;
        if (rect) { rect[4 * i] = s->x0; rect[4 * i + 1] = s->x1; rect[4 * i + 2] = s->y0; rect[4 * i + 3] = s->y1; }
        if (rec) {
            double* r = rec + 10 * i;
            r[0] = s->mean2d[0]; r[1] = s->mean2d[1];
            r[2] = s->conic_a; r[3] = s->conic_b; r[4] = s->conic_c;
            r[5] = s->opacity; r[6] = s->coef; r[7] = s->sin_psi; r[8] = s->cos_psi; r[9] = s->depth;
        }
    }
}

void orc_pass_tile_lists(const orc_pass* P, int64_t* offsets, int32_t* ids) {
    const int nt = P->tiles_x * P->tiles_y;
    if (offsets) memcpy(offsets, P->tile_off, sizeof(int64_t) * ((size_t)nt + 1));
    if (ids) memcpy(ids, P->tile_ids, sizeof(int32_t) * (size_t)P->tile_off[nt]);
}

/* ---- forward (splat.cpp:209-339) ---------------------------------------- */
void orc_pass_forward(const orc_pass* P, double* quad, double* phasor, double* depth_raw,
                      double* depth, double* weight, double* transmittance, double* distortion,
                      int32_t* n_contrib, int32_t* n_processed) {
    const int W = P->cam.width, H = P->cam.height;
    const size_t HW = (size_t)W * H;
    const orc_options* opt = &P->opt;
    const double cutoff2 = opt->sigma_cutoff * opt->sigma_cutoff;
    const int ts = opt->tile_size > 1 ? opt->tile_size : 1;
    const int ntiles = P->tiles_x * P->tiles_y;
    const double nan = NAN;

#pragma omp parallel for schedule(static)
    for (int tile = 0; tile < ntiles; ++tile) {
        const int32_t* ids = P->tile_ids + P->tile_off[tile];
        const int64_t nids = P->tile_off[tile + 1] - P->tile_off[tile];
        const int px0 = (tile % P->tiles_x) * ts, px1 = px0 + ts < W ? px0 + ts : W;
        const int py0 = (tile / P->tiles_x) * ts, py1 = py0 + ts < H ? py0 + ts : H;
        for (int y = py0; y < py1; ++y) {
            for (int x = px0; x < px1; ++x) {
                const double pcx = x + 0.5, pcy = y + 0.5;
                double T = 1.0;
                double accQ[4] = {0, 0, 0, 0}, accP[2] = {0, 0};
                double SW = 0, SD = 0, SD2 = 0;
                int nc = 0;
                int64_t e = 0;
                for (; e < nids; ++e) {
                    const Prepared* s = &P->prep[ids[e]];
                    if (x < s->x0 || x >= s->x1 || y < s->y0 || y >= s->y1) continue;
                    const double dx = pcx - s->mean2d[0], dy = pcy - s->mean2d[1];
                    const double maha = s->conic_a * dx * dx + 2.0 * s->conic_b * dx * dy + s->conic_c * dy * dy;
                    if (maha > cutoff2 || maha < 0.0) continue;
                    const double g = exp(-0.5 * maha);
                    const double alpha = s->opacity * g;
                    if (alpha < opt->alpha_threshold) continue;
                    ++nc;
                    const double w = alpha * T;
                    const double w2 = alpha * T * T;
                    const double cq = s->coef * w2;
                    accQ[0] += cq * s->sin_psi;
                    accQ[1] += cq * s->cos_psi;
                    accQ[2] -= cq * s->sin_psi;
                    accQ[3] -= cq * s->cos_psi;
                    const double cp = 2.0 * s->coef * w2;
                    accP[0] += cp * s->cos_psi;
                    accP[1] += cp * s->sin_psi;
                    SW += w;
                    SD += w * s->depth;
                    SD2 += w * s->depth * s->depth;
                    T *= 1.0 - alpha;
                    if (T < opt->transmittance_floor) { ++e; break; }
                }
                const size_t o = (size_t)y * W + x;
                if (transmittance) transmittance[o] = T;
                if (weight) weight[o] = SW;
                if (quad)
                    for (int c = 0; c < 4; ++c) quad[c * HW + o] = accQ[c] + opt->bg_quad[c] * T * T;
                if (phasor)
                    for (int c = 0; c < 2; ++c) phasor[c * HW + o] = accP[c] + opt->bg_phasor[c] * T * T;
                if (depth_raw) depth_raw[o] = SD;
                if (depth) depth[o] = SW > opt->coverage_eps ? SD / SW : nan;
                if (distortion) distortion[o] = 2.0 * (SW * SD2 - SD * SD);
                if (n_contrib) n_contrib[o] = nc;
                if (n_processed) n_processed[o] = (int32_t)e;
            }
        }
    }
}

/* ---- colour and flow channels (splat.cpp:273-294, 301-334) ------------------ */
void orc_pass_forward_ext(const orc_pass* P, double* color, double* mf_acc, double* mb_acc, double* flow_fwd,
                          double* flow_bwd, double* flow_valid) {
    const orc_camera* cam = &P->cam;
    const int W = cam->width, H = cam->height;
    const size_t HW = (size_t)W * H;
    const orc_options* opt = &P->opt;
    const double cutoff2 = opt->sigma_cutoff * opt->sigma_cutoff;
    const int ts = opt->tile_size > 1 ? opt->tile_size : 1;
    const int ntiles = P->tiles_x * P->tiles_y;
    const double* R = cam->R;
#pragma omp parallel for schedule(static)
    for (int tile = 0; tile < ntiles; ++tile) {
        const int32_t* ids = P->tile_ids + P->tile_off[tile];
        const int64_t nids = P->tile_off[tile + 1] - P->tile_off[tile];
        const int px0 = (tile % P->tiles_x) * ts, px1 = px0 + ts < W ? px0 + ts : W;
        const int py0 = (tile / P->tiles_x) * ts, py1 = py0 + ts < H ? py0 + ts : H;
        for (int y = py0; y < py1; ++y) {
            for (int x = px0; x < px1; ++x) {
                const double pcx = x + 0.5, pcy = y + 0.5;
                double T = 1.0, SW = 0, SD = 0;
                double accC[3] = {0, 0, 0}, accMf[3] = {0, 0, 0}, accMb[3] = {0, 0, 0};
                for (int64_t e = 0; e < nids; ++e) {
                    const Prepared* s = &P->prep[ids[e]];
                    if (x < s->x0 || x >= s->x1 || y < s->y0 || y >= s->y1) continue;
                    const double dx = pcx - s->mean2d[0], dy = pcy - s->mean2d[1];
                    const double maha = s->conic_a * dx * dx + 2.0 * s->conic_b * dx * dy + s->conic_c * dy * dy;
                    if (maha > cutoff2 || maha < 0.0) continue;
                    const double alpha = s->opacity * exp(-0.5 * maha);
                    if (alpha < opt->alpha_threshold) continue;
                    const double w = alpha * T;
                    for (int c = 0; c < 3; ++c) {
                        accC[c] += w * s->color[c];
                        accMf[c] += w * s->mf[c];
                        accMb[c] += w * s->mb[c];
                    }
                    SW += w;
                    SD += w * s->depth;
                    T *= 1.0 - alpha;
                    if (T < opt->transmittance_floor) break;
                }
                const size_t o = (size_t)y * W + x;
                for (int c = 0; c < 3; ++c) {
                    if (color) color[c * HW + o] = accC[c] + opt->bg_color[c] * T;
                    if (mf_acc) mf_acc[c * HW + o] = accMf[c];
                    if (mb_acc) mb_acc[c * HW + o] = accMb[c];
                }
                for (int c = 0; c < 2; ++c) {
                    if (flow_fwd) flow_fwd[c * HW + o] = 0.0;
                    if (flow_bwd) flow_bwd[c * HW + o] = 0.0;
                    if (flow_valid) flow_valid[c * HW + o] = 0.0;
                }
                if (SW > opt->coverage_eps) {
                    /* cam.backproject (camera.hpp:34-43): optical_center + dist * normalize(R^T d_cam),
                     * d_cam = ((px - cx) / fx, (py - cy) / fy, 1), dist = SD / SW (radial depth) */
                    const double dist = SD / SW;
                    const double dc[3] = {(pcx - cam->cx) / cam->fx, (pcy - cam->cy) / cam->fy, 1.0};
                    double dir[3], center[3];
                    for (int a = 0; a < 3; ++a) {
                        dir[a] = R[0 * 3 + a] * dc[0] + R[1 * 3 + a] * dc[1] + R[2 * 3 + a] * dc[2];
                        center[a] = -(R[0 * 3 + a] * cam->t[0] + R[1 * 3 + a] * cam->t[1] + R[2 * 3 + a] * cam->t[2]);
                    }
                    const double dn = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
                    double xd[3];
                    for (int a = 0; a < 3; ++a) xd[a] = center[a] + dist * (dir[a] / dn);
                    for (int k = 0; k < 2; ++k) {
                        const double* mo = k == 0 ? accMf : accMb;
                        double* fl = k == 0 ? flow_fwd : flow_bwd;
                        double q[3], p[3];
                        for (int a = 0; a < 3; ++a) q[a] = xd[a] + mo[a];
                        for (int i = 0; i < 3; ++i)
                            p[i] = R[i * 3 + 0] * q[0] + R[i * 3 + 1] * q[1] + R[i * 3 + 2] * q[2] + cam->t[i];
                        if (p[2] > 0.0) {
                            if (fl) {
                                fl[o] = cam->fx * p[0] / p[2] + cam->cx - pcx;
                                fl[HW + o] = cam->fy * p[1] / p[2] + cam->cy - pcy;
                            }
                            if (flow_valid) flow_valid[k * HW + o] = 1.0;
                        }
                    }
                }
            }
        }
    }
}

/* ---- backward (splat.cpp:347-650) --------------------------------------- */
typedef struct {
    double d_mean2d[2];
    double d_conic_a, d_conic_b, d_conic_c;
    double d_opacity, d_coef, d_depth;
    double d_color[3], d_mf[3], d_mb[3];
} SplatGrad;

typedef struct {
    int idx;
    double alpha, gval, T, dx, dy;
} Entry;

void orc_pass_backward(const orc_pass* P, const double* d_quad, const double* d_phasor,
                       const double* d_depth_raw, const double* d_weight,
                       const double* d_distortion, const double* d_transmittance,
                       double* d_position, double* d_log_scale, double* d_rotation,
                       double* d_opacity_logit, double* d_refl_sh, double* d_bg_quad,
                       double* d_bg_phasor, double* screen) {
    orc_pass_backward_ext(P, d_quad, d_phasor, d_depth_raw, d_weight, d_distortion, d_transmittance, NULL, NULL, NULL,
                          d_position, d_log_scale, d_rotation, d_opacity_logit, d_refl_sh, d_bg_quad, d_bg_phasor,
                          NULL, NULL, NULL, NULL, screen);
}

void orc_pass_backward_ext(const orc_pass* P, const double* d_quad, const double* d_phasor,
                           const double* d_depth_raw, const double* d_weight, const double* d_distortion,
                           const double* d_transmittance, const double* d_color, const double* d_mf_acc,
                           const double* d_mb_acc, double* d_position, double* d_log_scale, double* d_rotation,
                           double* d_opacity_logit, double* d_refl_sh, double* d_bg_quad, double* d_bg_phasor,
                           double* d_color_sh, double* d_motion_fwd, double* d_motion_bwd, double* d_bg_color,
                           double* screen) {
    const orc_scene* sc = &P->scene;
    const orc_camera* cam = &P->cam;
    const orc_options* opt = &P->opt;
    const int W = cam->width, H = cam->height;
    const size_t HW = (size_t)W * H;
    const double cutoff2 = opt->sigma_cutoff * opt->sigma_cutoff;
    const int ts = opt->tile_size > 1 ? opt->tile_size : 1;
    const int ntiles = P->tiles_x * P->tiles_y;
    const int nvis = P->nvis;
    const int n = sc->n;

    const int nthreads = orc_num_threads();
    SplatGrad* tl = (SplatGrad*)calloc((size_t)nthreads * (nvis > 0 ? nvis : 1), sizeof(SplatGrad));
    double* tl_bg = (double*)calloc((size_t)nthreads * 9, sizeof(double));

#pragma omp parallel
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        SplatGrad* sg = tl + (size_t)tid * (nvis > 0 ? nvis : 1);
        double* bgg = tl_bg + 9 * tid;
        size_t cap = 256;
        Entry* entries = (Entry*)malloc(sizeof(Entry) * cap);
#pragma omp for schedule(static)
        for (int tile = 0; tile < ntiles; ++tile) {
            const int32_t* ids = P->tile_ids + P->tile_off[tile];
            const int64_t nids = P->tile_off[tile + 1] - P->tile_off[tile];
            const int px0 = (tile % P->tiles_x) * ts, px1 = px0 + ts < W ? px0 + ts : W;
            const int py0 = (tile / P->tiles_x) * ts, py1 = py0 + ts < H ? py0 + ts : H;
            for (int y = py0; y < py1; ++y) {
                for (int x = px0; x < px1; ++x) {
                    const double pcx = x + 0.5, pcy = y + 0.5;
                    size_t ne = 0;
                    double T = 1.0, SW = 0, SD = 0, SD2 = 0;
                    for (int64_t e = 0; e < nids; ++e) {
                        const int idx = ids[e];
                        const Prepared* s = &P->prep[idx];
                        if (x < s->x0 || x >= s->x1 || y < s->y0 || y >= s->y1) continue;
                        const double dx = pcx - s->mean2d[0], dy = pcy - s->mean2d[1];
                        const double maha = s->conic_a * dx * dx + 2.0 * s->conic_b * dx * dy + s->conic_c * dy * dy;
                        if (maha > cutoff2 || maha < 0.0) continue;
                        const double g = exp(-0.5 * maha);
                        const double alpha = s->opacity * g;
                        if (alpha < opt->alpha_threshold) continue;
                        if (ne == cap) { cap *= 2; entries = (Entry*)realloc(entries, sizeof(Entry) * cap); }
                        entries[ne].idx = idx; entries[ne].alpha = alpha; entries[ne].gval = g;
                        entries[ne].T = T; entries[ne].dx = dx; entries[ne].dy = dy;
                        ++ne;
                        const double w = alpha * T;
                        SW += w;
                        SD += w * s->depth;
                        SD2 += w * s->depth * s->depth;
                        T *= 1.0 - alpha;
                        if (T < opt->transmittance_floor) break;
                    }
                    const double T_final = T;
                    const size_t o = (size_t)y * W + x;
                    double upQ[4] = {0, 0, 0, 0}, upP[2] = {0, 0};
                    double upDraw = 0, upW = 0, upDD = 0, upT = 0;
                    double upC[3] = {0, 0, 0}, upMf[3] = {0, 0, 0}, upMb[3] = {0, 0, 0};
                    if (d_color) for (int c = 0; c < 3; ++c) upC[c] = d_color[c * HW + o];
                    if (d_mf_acc) for (int c = 0; c < 3; ++c) upMf[c] = d_mf_acc[c * HW + o];
                    if (d_mb_acc) for (int c = 0; c < 3; ++c) upMb[c] = d_mb_acc[c * HW + o];
                    if (d_color) for (int c = 0; c < 3; ++c) bgg[6 + c] += upC[c] * T_final;
                    if (d_quad) for (int c = 0; c < 4; ++c) upQ[c] = d_quad[c * HW + o];
                    if (d_phasor) for (int c = 0; c < 2; ++c) upP[c] = d_phasor[c * HW + o];
                    if (d_depth_raw) upDraw = d_depth_raw[o];
                    if (d_weight) upW = d_weight[o];
                    if (d_distortion) upDD = d_distortion[o];
                    if (d_transmittance) upT = d_transmittance[o];
                    if (d_quad) for (int c = 0; c < 4; ++c) bgg[c] += upQ[c] * T_final * T_final;
                    if (d_phasor) for (int c = 0; c < 2; ++c) bgg[4 + c] += upP[c] * T_final * T_final;
                    if (ne == 0) continue;

                    double accQ[4], accP[2];
                    for (int c = 0; c < 4; ++c) accQ[c] = opt->bg_quad[c];
                    for (int c = 0; c < 2; ++c) accP[c] = opt->bg_phasor[c];
                    double accD = 0, accW = 0, accPhi = 0, Rsuf = 1.0;
                    double accC[3], accMf[3] = {0, 0, 0}, accMb[3] = {0, 0, 0};
                    for (int c = 0; c < 3; ++c) accC[c] = opt->bg_color[c];
                    for (long e = (long)ne - 1; e >= 0; --e) {
                        const Entry* en = &entries[e];
                        const Prepared* s = &P->prep[en->idx];
                        SplatGrad* ga = &sg[en->idx];
                        const double alpha = en->alpha, Tk = en->T, one_m = 1.0 - alpha;
                        const double w = alpha * Tk, w2 = alpha * Tk * Tk, Tk2 = Tk * Tk;
                        double d_alpha = 0;
                        if (d_color) {
                            double t = 0;
                            for (int c = 0; c < 3; ++c) t += upC[c] * (Tk * (s->color[c] - accC[c]));
                            d_alpha += t;
                            for (int c = 0; c < 3; ++c) ga->d_color[c] += upC[c] * w;
                            for (int c = 0; c < 3; ++c) accC[c] = alpha * s->color[c] + one_m * accC[c];
                        }
                        if (d_quad) {
                            const double basis[4] = {s->sin_psi, s->cos_psi, -s->sin_psi, -s->cos_psi};
                            double qk[4], t1 = 0, t2 = 0, t3 = 0;
                            for (int c = 0; c < 4; ++c) qk[c] = s->coef * basis[c];
                            for (int c = 0; c < 4; ++c) t1 += upQ[c] * (Tk2 * (qk[c] + 2.0 * (alpha - 1.0) * accQ[c]));
                            d_alpha += t1;
                            for (int c = 0; c < 4; ++c) t2 += upQ[c] * basis[c];
                            ga->d_coef += w2 * t2;
                            const double db[4] = {s->cos_psi, -s->sin_psi, -s->cos_psi, s->sin_psi};
                            for (int c = 0; c < 4; ++c) t3 += upQ[c] * db[c];
                            ga->d_depth += w2 * s->coef * s->dpsi_dd * t3;
                            for (int c = 0; c < 4; ++c) accQ[c] = alpha * qk[c] + one_m * one_m * accQ[c];
                        }
                        if (d_phasor) {
                            const double pb[2] = {s->cos_psi, s->sin_psi};
                            double pk[2], t1 = 0, t2 = 0, t3 = 0;
                            for (int c = 0; c < 2; ++c) pk[c] = 2.0 * s->coef * pb[c];
                            for (int c = 0; c < 2; ++c) t1 += upP[c] * (Tk2 * (pk[c] + 2.0 * (alpha - 1.0) * accP[c]));
                            d_alpha += t1;
                            for (int c = 0; c < 2; ++c) t2 += upP[c] * pb[c];
                            ga->d_coef += w2 * 2.0 * t2;
                            const double dpb[2] = {-s->sin_psi, s->cos_psi};
                            for (int c = 0; c < 2; ++c) t3 += upP[c] * dpb[c];
                            ga->d_depth += w2 * 2.0 * s->coef * s->dpsi_dd * t3;
                            for (int c = 0; c < 2; ++c) accP[c] = alpha * pk[c] + one_m * one_m * accP[c];
                        }
                        if (d_depth_raw) {
                            d_alpha += upDraw * Tk * (s->depth - accD);
                            ga->d_depth += upDraw * w;
                            accD = alpha * s->depth + one_m * accD;
                        }
                        if (d_weight) {
                            d_alpha += upW * Tk * (1.0 - accW);
                            accW = alpha + one_m * accW;
                        }
                        if (d_distortion) {
                            const double phi = 2.0 * SD2 + 2.0 * SW * s->depth * s->depth - 4.0 * SD * s->depth;
                            d_alpha += upDD * Tk * (phi - accPhi);
                            ga->d_depth += upDD * 4.0 * w * (SW * s->depth - SD);
                            accPhi = alpha * phi + one_m * accPhi;
                        }
                        if (d_mf_acc) {
                            double t = 0;
                            for (int c = 0; c < 3; ++c) t += upMf[c] * (Tk * (s->mf[c] - accMf[c]));
                            d_alpha += t;
                            for (int c = 0; c < 3; ++c) ga->d_mf[c] += upMf[c] * w;
                            for (int c = 0; c < 3; ++c) accMf[c] = alpha * s->mf[c] + one_m * accMf[c];
                        }
                        if (d_mb_acc) {
                            double t = 0;
                            for (int c = 0; c < 3; ++c) t += upMb[c] * (Tk * (s->mb[c] - accMb[c]));
                            d_alpha += t;
                            for (int c = 0; c < 3; ++c) ga->d_mb[c] += upMb[c] * w;
                            for (int c = 0; c < 3; ++c) accMb[c] = alpha * s->mb[c] + one_m * accMb[c];
                        }
                        if (d_transmittance) d_alpha -= upT * Tk * Rsuf;
                        Rsuf *= one_m;

                        ga->d_opacity += en->gval * d_alpha;
                        const double d_power = alpha * d_alpha;
                        ga->d_mean2d[0] += d_power * (s->conic_a * en->dx + s->conic_b * en->dy);
                        ga->d_mean2d[1] += d_power * (s->conic_b * en->dx + s->conic_c * en->dy);
                        ga->d_conic_a += -0.5 * en->dx * en->dx * d_power;
                        ga->d_conic_b += -en->dx * en->dy * d_power;
                        ga->d_conic_c += -0.5 * en->dy * en->dy * d_power;
                    }
                }
            }
        }
        free(entries);
    }

    /* fixed-order reduction (splat.cpp:521-543) */
    SplatGrad* acc = tl;
    double bg[9];
    memcpy(bg, tl_bg, sizeof bg);
    for (int t = 1; t < nthreads; ++t) {
        const SplatGrad* a = tl + (size_t)t * (nvis > 0 ? nvis : 1);
        for (int i = 0; i < nvis; ++i) {
            SplatGrad* b = &acc[i];
            b->d_mean2d[0] += a[i].d_mean2d[0];
            b->d_mean2d[1] += a[i].d_mean2d[1];
            b->d_conic_a += a[i].d_conic_a;
            b->d_conic_b += a[i].d_conic_b;
            b->d_conic_c += a[i].d_conic_c;
            b->d_opacity += a[i].d_opacity;
            b->d_coef += a[i].d_coef;
            b->d_depth += a[i].d_depth;
            for (int c = 0; c < 3; ++c) {
                b->d_color[c] += a[i].d_color[c];
                b->d_mf[c] += a[i].d_mf[c];
                b->d_mb[c] += a[i].d_mb[c];
            }
        }
        for (int c = 0; c < 9; ++c) bg[c] += tl_bg[9 * t + c];
    }
    if (d_bg_quad) for (int c = 0; c < 4; ++c) d_bg_quad[c] = bg[c];
    if (d_bg_phasor) for (int c = 0; c < 2; ++c) d_bg_phasor[c] = bg[4 + c];
    if (d_bg_color) for (int c = 0; c < 3; ++c) d_bg_color[c] = bg[6 + c];
    if (d_color_sh) memset(d_color_sh, 0, sizeof(double) * 48 * (size_t)n);
    if (d_motion_fwd) memset(d_motion_fwd, 0, sizeof(double) * 3 * (size_t)n);
    if (d_motion_bwd) memset(d_motion_bwd, 0, sizeof(double) * 3 * (size_t)n);

    if (d_position) memset(d_position, 0, sizeof(double) * 3 * (size_t)n);
    if (d_log_scale) memset(d_log_scale, 0, sizeof(double) * 3 * (size_t)n);
    if (d_rotation) memset(d_rotation, 0, sizeof(double) * 4 * (size_t)n);
    if (d_opacity_logit) memset(d_opacity_logit, 0, sizeof(double) * (size_t)n);
    if (d_refl_sh) memset(d_refl_sh, 0, sizeof(double) * SHN * (size_t)n);

    const double* R = cam->R;
    for (int i = 0; i < nvis; ++i) {
        const Prepared* s = &P->prep[i];
        const SplatGrad* g = &acc[i];
        const int gi = s->gidx;
        if (screen) {
            double* o = screen + 8 * i;
            o[0] = g->d_mean2d[0]; o[1] = g->d_mean2d[1]; o[2] = g->d_conic_a; o[3] = g->d_conic_b;
            o[4] = g->d_conic_c; o[5] = g->d_opacity; o[6] = g->d_coef; o[7] = g->d_depth;
        }
        if (d_opacity_logit) d_opacity_logit[gi] += g->d_opacity * s->opacity * (1.0 - s->opacity);

        double d_dir[3] = {0, 0, 0};
        double Jb[SHN * 3];
        orc_sh_basis_jacobian(s->view_dir, sc->sh_degree, Jb);

        /* colour SH: the clamp gates each channel (splat.cpp:560-571) */
        if (g->d_color[0] != 0.0 || g->d_color[1] != 0.0 || g->d_color[2] != 0.0) {
            double dcol[3];
            for (int c = 0; c < 3; ++c)
                dcol[c] = (s->color_raw[c] > 0.0 && s->color_raw[c] < 1.0) ? g->d_color[c] : 0.0;
            if (d_color_sh)
                for (int c = 0; c < 3; ++c)
                    for (int k = 0; k < SHN; ++k) d_color_sh[48 * (size_t)gi + SHN * c + k] += s->sh_b[k] * dcol[c];
            if (sc->color_sh) /* d_dir += Jb^T (color_sh dcol) */
                for (int a = 0; a < 3; ++a) {
                    double acc_ = 0;
                    for (int k = 0; k < SHN; ++k) {
                        double cs = 0;
                        for (int c = 0; c < 3; ++c) cs += sc->color_sh[48 * (size_t)gi + SHN * c + k] * dcol[c];
                        acc_ += Jb[k * 3 + a] * cs;
                    }
                    d_dir[a] += acc_;
                }
        }
        for (int c = 0; c < 3; ++c) {
            if (d_motion_fwd) d_motion_fwd[3 * gi + c] += g->d_mf[c];
            if (d_motion_bwd) d_motion_bwd[3 * gi + c] += g->d_mb[c];
        }

        const double r_cl = clampd(s->refl_raw, 0.0, 1.0);
        const double d2 = s->depth * s->depth;
        const double d_depth = g->d_depth + g->d_coef * (-2.0 * sc->source_intensity * r_cl / (d2 * s->depth));
        if (s->refl_raw > 0.0 && s->refl_raw < 1.0) {
            const double d_r = g->d_coef * sc->source_intensity / d2;
            if (d_refl_sh) for (int k = 0; k < SHN; ++k) d_refl_sh[SHN * gi + k] += s->sh_b[k] * d_r;
            /* d_dir += Jb^T (refl_sh * d_r) */
            for (int a = 0; a < 3; ++a) {
                double acc_ = 0;
                for (int k = 0; k < SHN; ++k) acc_ += Jb[k * 3 + a] * (sc->refl_sh[SHN * gi + k] * d_r);
                d_dir[a] += acc_;
            }
        }

        /* conic -> cov2d: G2 = -Q GQ Q */
        const double Q[4] = {s->conic_a, s->conic_b, s->conic_b, s->conic_c};
        const double GQ[4] = {g->d_conic_a, 0.5 * g->d_conic_b, 0.5 * g->d_conic_b, g->d_conic_c};
        double QG[4], G2[4];
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) QG[a * 2 + b] = Q[a * 2 + 0] * GQ[0 * 2 + b] + Q[a * 2 + 1] * GQ[1 * 2 + b];
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) G2[a * 2 + b] = -(QG[a * 2 + 0] * Q[0 * 2 + b] + QG[a * 2 + 1] * Q[1 * 2 + b]);
        /* dM = 2 G2 M cov3d ; G3 = M^T G2 M */
        double GM[6], dM[6], G3[9], MtG[6];
        for (int a = 0; a < 2; ++a)
            for (int j = 0; j < 3; ++j) GM[a * 3 + j] = G2[a * 2 + 0] * s->M[0 * 3 + j] + G2[a * 2 + 1] * s->M[1 * 3 + j];
        for (int a = 0; a < 2; ++a)
            for (int j = 0; j < 3; ++j) {
                double t = 0;
                for (int k = 0; k < 3; ++k) t += (2.0 * GM[a * 3 + k]) * s->cov3d[k * 3 + j];
                dM[a * 3 + j] = t;
            }
        /* G3 = (M^T G2) M */
        for (int i2 = 0; i2 < 3; ++i2)
            for (int b = 0; b < 2; ++b) MtG[i2 * 2 + b] = s->M[0 * 3 + i2] * G2[0 * 2 + b] + s->M[1 * 3 + i2] * G2[1 * 2 + b];
        for (int i2 = 0; i2 < 3; ++i2)
            for (int j = 0; j < 3; ++j) G3[i2 * 3 + j] = MtG[i2 * 2 + 0] * s->M[0 * 3 + j] + MtG[i2 * 2 + 1] * s->M[1 * 3 + j];
        /* dJ = dM R^T */
        double dJ[6];
        for (int a = 0; a < 2; ++a)
            for (int j = 0; j < 3; ++j)
                dJ[a * 3 + j] = dM[a * 3 + 0] * R[j * 3 + 0] + dM[a * 3 + 1] * R[j * 3 + 1] + dM[a * 3 + 2] * R[j * 3 + 2];
        const double z = s->p_cam[2], z2 = z * z, z3 = z2 * z;
        double dp[3] = {0, 0, 0};
        const double dtx = dJ[2] * (-cam->fx / z2);
        const double dty = dJ[5] * (-cam->fy / z2);
        dp[2] += dJ[0] * (-cam->fx / z2) + dJ[4] * (-cam->fy / z2) + dJ[2] * (2.0 * cam->fx * s->tx / z3) +
                 dJ[5] * (2.0 * cam->fy * s->ty / z3);
        if (s->clamp_x) dp[2] += dtx * (s->tx / z); else dp[0] += dtx;
        if (s->clamp_y) dp[2] += dty * (s->ty / z); else dp[1] += dty;
        dp[0] += g->d_mean2d[0] * cam->fx / z;
        dp[2] += g->d_mean2d[0] * (-cam->fx * s->p_cam[0] / z2);
        dp[1] += g->d_mean2d[1] * cam->fy / z;
        dp[2] += g->d_mean2d[1] * (-cam->fy * s->p_cam[1] / z2);
        for (int a = 0; a < 3; ++a) dp[a] += d_depth * (s->p_cam[a] / s->depth);

        const double vd = s->view_dir[0] * d_dir[0] + s->view_dir[1] * d_dir[1] + s->view_dir[2] * d_dir[2];
        double dpos[3];
        for (int a = 0; a < 3; ++a) dpos[a] = (d_dir[a] - s->view_dir[a] * vd) / s->depth;
        for (int a = 0; a < 3; ++a) dpos[a] += R[0 * 3 + a] * dp[0] + R[1 * 3 + a] * dp[1] + R[2 * 3 + a] * dp[2];
        if (d_position) for (int a = 0; a < 3; ++a) d_position[3 * gi + a] += dpos[a];

        /* cov3d = M3 M3^T, M3 = R(q) diag(exp(ls)) */
        const double* q = sc->rotation + 4 * gi;
        double uq[4], Rq[9], sv[3], M3[9], dM3[9];
        normalize4(q, uq);
        orc_quat_to_rotation(q, Rq);
        for (int j = 0; j < 3; ++j) sv[j] = exp(sc->log_scale[3 * gi + j]);
        for (int r = 0; r < 3; ++r)
            for (int j = 0; j < 3; ++j) M3[r * 3 + j] = Rq[r * 3 + j] * sv[j];
        for (int r = 0; r < 3; ++r)
            for (int j = 0; j < 3; ++j) {
                double t = 0;
                for (int k = 0; k < 3; ++k) t += (2.0 * G3[r * 3 + k]) * M3[k * 3 + j];
                dM3[r * 3 + j] = t;
            }
        for (int j = 0; j < 3; ++j) {
            double ds = 0;
            for (int r = 0; r < 3; ++r) ds += Rq[r * 3 + j] * dM3[r * 3 + j];
            if (d_log_scale) d_log_scale[3 * gi + j] += ds * sv[j];
        }
        double dRq[9];
        for (int r = 0; r < 3; ++r)
            for (int j = 0; j < 3; ++j) dRq[r * 3 + j] = dM3[r * 3 + j] * sv[j];
        double dR[4][9];
        quat_rot_jac(uq, dR);
        double duq[4];
        for (int c = 0; c < 4; ++c) {
            double t = 0;
            for (int k = 0; k < 9; ++k) t += dRq[k] * dR[c][k];
            duq[c] = t;
        }
        const double qn = sqrt(sqnorm4(q));
        const double ud = uq[0] * duq[0] + uq[1] * duq[1] + uq[2] * duq[2] + uq[3] * duq[3];
        if (d_rotation) for (int c = 0; c < 4; ++c) d_rotation[4 * gi + c] += (duq[c] - uq[c] * ud) / qn;
    }
    free(tl);
    free(tl_bg);
}

/* ---- losses / optimiser ------------------------------------------------- */
double orc_mse(const double* pred, const double* target, size_t n, double* d_pred) {
    if (n == 0) return 0.0;
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double d = pred[i] - target[i];
        acc += d * d;
    }
    if (d_pred) {
        const double s = 2.0 / (double)n;
        for (size_t i = 0; i < n; ++i) d_pred[i] += s * (pred[i] - target[i]);
    }
    return acc / (double)n;
}

void orc_adam_step(double* p, const double* g, double* m, double* v, size_t n, int64_t t,
                   double lr, double b1, double b2, double eps) {
    const double bc1 = 1.0 - pow(b1, (double)t);
    const double bc2 = 1.0 - pow(b2, (double)t);
    for (size_t i = 0; i < n; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * g[i];
        v[i] = b2 * v[i] + (1.0 - b2) * (g[i] * g[i]);
        p[i] -= (lr / bc1) * (m[i] / (sqrt(v[i] / bc2) + eps));
    }
}

void orc_interp_positions(const double* x, const double* d_i, const double* d_ip1, double w,
                          size_t n, double* out) {
    for (size_t k = 0; k < 3 * n; ++k) {
        const double Xi = x[k] + d_i[k];
        const double Xip1 = x[k] + d_ip1[k];
        out[k] = (w == 0.0) ? Xi : (1.0 - w) * Xi + w * Xip1;
    }
}
