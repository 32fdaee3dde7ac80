/*
 * tofsplat_oracle.h -- CPU restatement of the reference C-ToF splat hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 kernels
 * (and the "port" CPU baseline in bench.py).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path (paper_2505_05356_b200, libtsb.so) never links or calls it.
 *
 * It restates, in double precision and without Eigen, the reference's
 *   RenderPassImpl::prepare / sort / build_tiles   proj/src/splat.cpp:105-200
 *   RenderPass::forward                            proj/src/splat.cpp:209-339
 *   RenderPass::backward (+ fixed-order reduce, chain)  proj/src/splat.cpp:347-650
 *   mse                                            proj/src/losses.cpp:9-25
 *   AdamState::step                                proj/src/trainer.cpp:18-31
 *   trajectory lerp / chain                        proj/src/trainer.cpp:259-331
 *   densify statistic                              proj/src/trainer.cpp:381-384
 * and additionally EXPORTS the integer intermediates the reference keeps
 * private (prepared order, tile rects, per-tile lists, per-pixel contributor
 * counts) so the GPU's integer work can be compared bit for bit.
 *
 * Parity pin: tests/test_oracle_kat.py checks this oracle against every
 * closed-form known-answer test of proj/tests/unit/test_splat.cpp,
 * test_tof.cpp, test_scene.cpp, test_camera_sh.cpp, test_trainer.cpp (Adam),
 * test_losses.cpp (mse), acceptance checks 3/6/7, and runs the reference's
 * finite-difference gradcheck (proj/src/gradcheck.cpp) against it.  The
 * reference itself cannot be built here (Eigen3 absent), so these KATs are the pin.
 *
 * Colour and flow channels (splat.cpp:172-175, 273-294,
 * 301-334, 419-504, 560-571, 645-646) are restated by orc_pass_forward_ext /
 * orc_pass_backward_ext.
 */
#ifndef TOFSPLAT_ORACLE_H
#define TOFSPLAT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* CameraModel (proj/include/tofsplat/camera.hpp:9-17); R row-major, p_cam = R p + t. */
typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double near_plane, far_plane;
    double R[9];
    double t[3];
} orc_camera;

/* RenderOptions + Backgrounds (proj/include/tofsplat/splat.hpp:22-37). */
typedef struct {
    double alpha_threshold;     /* 1/255 */
    double transmittance_floor; /* 1e-4 */
    double dilation;            /* 0.3 */
    double sigma_cutoff;        /* 3 */
    double coverage_eps;        /* 1e-12 */
    int32_t tile_size;          /* 16 */
    int32_t _pad;
    double bg_quad[4];
    double bg_phasor[2];
    double bg_color[3];         /* Backgrounds::color */
} orc_options;

/* CanonicalScene / Gaussian (proj/include/tofsplat/scene.hpp:23-52), SoA.
 * `position` is the rendered mean (RenderInput::positions override, splat.hpp:45). */
typedef struct {
    int32_t n, sh_degree;
    double modulation_frequency, source_intensity, speed_of_light;
    const double* position;      /* 3n */
    const double* log_scale;     /* 3n */
    const double* rotation;      /* 4n, (w,x,y,z) raw */
    const double* opacity_logit; /* n */
    const double* refl_sh;       /* 16n */
    const double* color_sh;      /* 48n, [16 c + k] (Gaussian::color_sh(k, c)); NULL: black */
    const double* motion_fwd;    /* 3n (RenderInput::motion_fwd); NULL: zero */
    const double* motion_bwd;    /* 3n */
} orc_scene;

typedef struct orc_pass orc_pass;

const char* orc_last_error(void);
int orc_num_threads(void);
void orc_set_num_threads(int n);

/* RenderPass ctor: prepare + global (depth, gidx) sort + build_tiles.  NULL on error. */
orc_pass* orc_pass_create(const orc_scene* scene, const orc_camera* cam, const orc_options* opt);
void orc_pass_destroy(orc_pass* p);
int32_t orc_pass_visible_count(const orc_pass* p);
void orc_pass_tiles(const orc_pass* p, int32_t* tiles_x, int32_t* tiles_y);
int64_t orc_pass_num_keys(const orc_pass* p);

/* Prepared records in sorted (rank) order.  rect: x0,x1,y0,y1 per rank.
 * rec: mean_x, mean_y, conic_a, conic_b, conic_c, opacity, coef, sin_psi, cos_psi, depth. */
void orc_pass_prepared(const orc_pass* p, int32_t* gidx, int32_t* rect, double* rec);
/* Per-tile index lists (indices into the prepared order == rank), CSR. */
void orc_pass_tile_lists(const orc_pass* p, int64_t* offsets, int32_t* ids);

/* Forward (splat.cpp:209-339).  Planar [C][H][W]; any output may be NULL.
 * n_contrib: entries that passed the maha/alpha tests; n_processed: list entries
 * visited before the T-floor break (or the list length). */
void orc_pass_forward(const orc_pass* p, double* quad, double* phasor, double* depth_raw,
                      double* depth, double* weight, double* transmittance, double* distortion,
                      int32_t* n_contrib, int32_t* n_processed);

/* Backward (splat.cpp:347-650).  Upstream images may be NULL (channel absent).
 * Outputs (N-sized, zero for culled) are overwritten.  screen (8 per rank:
 * d_mean2d x,y, d_conic a,b,c, d_opacity, d_coef, d_depth) may be NULL. */
void orc_pass_backward(const orc_pass* p, const double* d_quad, const double* d_phasor,
                       const double* d_depth_raw, const double* d_weight,
                       const double* d_distortion, const double* d_transmittance,
                       double* d_position, double* d_log_scale, double* d_rotation,
                       double* d_opacity_logit, double* d_refl_sh, double* d_bg_quad,
                       double* d_bg_phasor, double* screen);

/* Colour and flow channels of RenderPass::forward (splat.cpp:273-294, 301-334); any may be NULL.
 * color [3][H][W] (+ bg_color T), motion accumulators [3][H][W], flow [2][H][W] (pixel
 * displacement of the depth-backprojected point moved by the accumulated motion),
 * flow_valid [2][H][W] (fwd, bwd). */
void orc_pass_forward_ext(const orc_pass* p, double* color, double* motion_fwd_acc, double* motion_bwd_acc,
                          double* flow_fwd, double* flow_bwd, double* flow_valid);
/* RenderPass::backward with every upstream of BufferGrads, including d_color [3][H][W] and the
 * motion accumulators; adds d_color_sh (48n), d_motion_fwd / d_motion_bwd (3n), d_bg_color (3). */
void orc_pass_backward_ext(const orc_pass* p, const double* d_quad, const double* d_phasor,
                           const double* d_depth_raw, const double* d_weight, const double* d_distortion,
                           const double* d_transmittance, const double* d_color, const double* d_motion_fwd_acc,
                           const double* d_motion_bwd_acc, double* d_position, double* d_log_scale,
                           double* d_rotation, double* d_opacity_logit, double* d_refl_sh, double* d_bg_quad,
                           double* d_bg_phasor, double* d_color_sh, double* d_motion_fwd, double* d_motion_bwd,
                           double* d_bg_color, double* screen);

/* mse (losses.cpp:9-25): returns mean sq. error; d_pred (may be NULL) += 2/n (pred-target). */
double orc_mse(const double* pred, const double* target, size_t n, double* d_pred);

/* AdamState::step (trainer.cpp:18-31); t is the step count AFTER increment. */
void orc_adam_step(double* params, const double* grads, double* m, double* v, size_t n,
                   int64_t t, double lr, double beta1, double beta2, double eps);

/* Trajectory (trainer.cpp:259-279): Xi = x + d_i; Xip1 = x + d_ip1;
 * P = (w == 0) ? Xi : (1-w) Xi + w Xip1.  All 3n. */
void orc_interp_positions(const double* x, const double* d_i, const double* d_ip1, double w,
                          size_t n, double* out);

/* quat_to_rotation (scene.cpp:10-18), row-major 3x3. */
void orc_quat_to_rotation(const double* q, double* R);
/* sh_basis (sh.hpp:26-50). */
void orc_sh_basis(const double* dir, int degree, double* b16);
void orc_sh_basis_jacobian(const double* dir, int degree, double* J48 /* 16x3 row-major */);

#ifdef __cplusplus
}
#endif
#endif
