/*
 * tsb.h -- C ABI of the B200-native C-ToF Gaussian-splat render/optimise path.
 *
 * This is the drop-in boundary that replaces the reference "tofsplat" hot path
 * (/root/reference/proj, a CPU C++20/Eigen library).  Every entry point names
 * the reference interface it replaces.  Plain pointers and sizes only; no
 * torch / Eigen / STL types cross it.  All device work is issued on the
 * context's CUDA stream; functions return TSB_OK or an error code and set a
 * thread-local message (tsb_last_error) -- the C++ shell in
 * include/tofsplat_b200/splat.hpp rethrows it as std::runtime_error with the
 * reference's messages (splat.cpp:91-100).
 *
 * There is no CPU fallback: if no sm_100 device is present, tsb_ctx_create
 * fails with TSB_ERR_CUDA.
 *
 * Data layouts (reference -> here):
 *   Gaussian parameters (scene.hpp:23-38, 75 doubles AoS) -> fp32 SoA arrays
 *     position 3n, log_scale 3n, rotation 4n (w,x,y,z), opacity_logit n,
 *     reflectivity_dc n (= reflectivity_sh[0]; sh_degree 0),
 *     motion 3n per keyframe (the per-Gaussian keyframe offsets that stand in for
 *     the DeformNet tick offsets, trainer.cpp:259-279 / SURVEY.md App. B).
 *     "3n" means 3 x n column-major == Eigen::Matrix3Xd storage.
 *   Image (image.hpp:12-38, planar channel-major double) -> planar fp32 [C][H][W].
 *   SceneGrads (splat.hpp:79-92) -> fp32 arrays with the same shapes as the params.
 */
#ifndef TSB_H
#define TSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSB_ABI_VERSION 3

enum {
    TSB_OK = 0,
    TSB_ERR_INVALID = 1,     /* bad argument (reference: std::runtime_error) */
    TSB_ERR_CUDA = 2,        /* CUDA runtime failure / no device */
    TSB_ERR_NOMEM = 3,       /* device allocation failed */
    TSB_ERR_UNSUPPORTED = 4, /* valid reference input this build does not handle */
    TSB_ERR_NCCL = 5
};

/* Where a pointer argument lives. */
enum { TSB_HOST = 0, TSB_DEVICE = 1 };

/* Output channel bits (RenderChannels, splat.hpp:13-20). */
enum {
    TSB_CH_QUAD = 1u << 0,      /* 4 raw samples per modulation frequency */
    TSB_CH_DEPTH = 1u << 1,     /* depth_raw and depth */
    TSB_CH_WEIGHT = 1u << 2,    /* weight (= alpha, sum_k w_k); always computed */
    TSB_CH_TRANSM = 1u << 3,    /* transmittance T_N; always computed */
    TSB_CH_COUNTS = 1u << 4,    /* per-pixel n_contrib / n_processed (parity) */
    TSB_CH_FULL_LISTS = 1u << 5, /* bin every tile's complete list (parity); default stops at termination */
    TSB_CH_PHASOR = 1u << 6,     /* (re, im) per frequency; always computed (free: 2x the quad sums) */
    TSB_CH_DISTORTION = 1u << 7, /* sum_kl w_k w_l (d_k - d_l)^2; required for a distortion upstream */
    TSB_CH_COLOR = 1u << 8,      /* RGB from the colour SH (scene created with color = 1), + bg_color T */
    TSB_CH_FLOW = 1u << 9,       /* motion accumulators + projected flow (tsb_pass_set_motion) */
    TSB_CH_EXACT = 1u << 10,     /* reference-exact mode: every pixel composited in fp64 (the fix-up path,
                                    forward and backward) and the outputs also kept as fp64 planes
                                    (TSB_OUT_F64 / TSB_OUT_EXT_F64) -- for finite-difference checks
                                    (gradcheck.cpp); costs an fp64 walk per pixel */
    TSB_CH_DETERMINISTIC = 1u << 11 /* bit-reproducible ToF gradients and loss (the reference's fixed-order
                                    reduction, splat.cpp:521-543): every raster block writes its per-entry
                                    sums to a private (rank, tile, sub-block) slot, reduced per Gaussian in
                                    a fixed order; no float atomics on the path (colour / flow upstreams
                                    excepted).  Costs a slot buffer and a host sync per backward */
};

/* CameraModel (camera.hpp:9-17).  R row-major; p_cam = R p_world + t. */
typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double near_plane, far_plane;
    double R[9];
    double t[3];
} tsb_camera;

/* RenderOptions + Backgrounds (splat.hpp:22-37).  bg_quad holds 4 values and
 * bg_phasor 2 values per modulation frequency. */
typedef struct {
    double alpha_threshold;     /* 1/255 */
    double transmittance_floor; /* 1e-4 */
    double dilation;            /* 0.3 px^2 */
    double sigma_cutoff;        /* 3 */
    double coverage_eps;        /* 1e-12 */
    int32_t tile_size;          /* 16 */
    uint32_t channels;          /* TSB_CH_* */
    double bg_quad[8];
    double bg_phasor[4];
    double bg_color[3];         /* Backgrounds::color */
} tsb_render_options;

/* CanonicalScene header (scene.hpp:44-52) + ToFConfig (tof.hpp:13-21).
 * n_freq = 2 renders two quads that share geometry (the
 * oracle for that is two reference renders with different frequencies). */
typedef struct {
    int32_t n;            /* Gaussians */
    int32_t n_keyframes;  /* 0 = static; else >= 2 keyframe offsets per Gaussian */
    int32_t sh_degree;    /* 0 (view-independent reflectivity) */
    int32_t n_freq;       /* 1 or 2 */
    double frequency[2];  /* Hz */
    double source_intensity;
    double speed_of_light;
    int32_t color;        /* 1: the scene carries colour SH (Gaussian::color_sh, 16 x 3) */
    int32_t _pad;
} tsb_scene_desc;

/* Frame selector for dynamic scenes: rendered mean = (1-w)(x + d_k) + w (x + d_{k+1})
 * (trainer.cpp:279); w == 0 renders x + d_k exactly (trainer.cpp:278). */
typedef struct {
    int32_t key;  /* k in [0, n_keyframes-2] */
    int32_t _pad;
    double w;     /* in [0, 1] */
} tsb_frame;

typedef struct tsb_ctx tsb_ctx;
typedef struct tsb_scene tsb_scene;
typedef struct tsb_pass tsb_pass;
typedef struct tsb_comm tsb_comm;

/* ---- context ------------------------------------------------------------ */
const char* tsb_last_error(void);
int tsb_abi_version(void);
/* One context per (host thread, GPU): owns a CUDA stream. */
int tsb_ctx_create(int device, tsb_ctx** out);
void tsb_ctx_destroy(tsb_ctx* ctx);
int tsb_ctx_synchronize(tsb_ctx* ctx);
/* The context's cudaStream_t (as void*), for callers that time on it. */
void* tsb_ctx_stream(tsb_ctx* ctx);
/* Each render pass runs on its own stream (forked from the context stream by
 * events), so passes used for consecutive frames overlap.  tsb_ctx_join makes the
 * context stream wait for all work enqueued so far on every pass of the context. */
int tsb_ctx_join(tsb_ctx* ctx);
/* Number of kernels this context has launched (bench.py gpu_launches). */
int64_t tsb_ctx_launch_count(tsb_ctx* ctx);
/* Frames redone after a device-side abort (tile-list storage overflow or an
 * over-long fp32 depth tie run).  Passes never wait for the device inside
 * prepare/forward/backward; a pass is settled (synchronised, and redone if its
 * frame aborted) before its results are read or the scene it read is changed. */
int64_t tsb_ctx_redo_count(tsb_ctx* ctx);

/* Per-stage device timing (CUDA events recorded on the context stream around each
 * stage's kernels).  Stages: see TSB_STAGE_*.  tsb_ctx_stage_times synchronises,
 * returns summed milliseconds and launch counts per stage, and resets. */
enum {
    TSB_STAGE_PREPROCESS = 0, TSB_STAGE_DEPTH_SORT = 1, TSB_STAGE_SCAN = 2, TSB_STAGE_BINNING = 3,
    TSB_STAGE_TILE_SORT = 4, TSB_STAGE_RANGES = 5, TSB_STAGE_RASTER_FWD = 6, TSB_STAGE_FIXUP = 7,
    TSB_STAGE_LOSS = 8, TSB_STAGE_RASTER_BWD = 9, TSB_STAGE_CHAIN = 10, TSB_STAGE_ADAM = 11,
    TSB_STAGE_ALLREDUCE = 12, TSB_STAGE_BIN_COUNT = 13, TSB_STAGE_BIN_EMIT = 14, TSB_NUM_STAGES = 15
};
/* Profiling mode also runs the forward eagerly (no CUDA graph) so each stage's
 * kernels are bracketed by events, and counts the raster's per-pixel work. */
int tsb_ctx_set_profiling(tsb_ctx* ctx, int enabled);
int tsb_ctx_stage_times(tsb_ctx* ctx, double* ms /* TSB_NUM_STAGES */, int64_t* calls /* TSB_NUM_STAGES */);
/* Forward-raster work since the last call (profiling mode only; resets):
 * (pixel, list entry) evaluations and contributing evaluations (alpha >= threshold). */
int tsb_ctx_raster_counts(tsb_ctx* ctx, int64_t* evaluations, int64_t* contributions);
/* Order work since the last call (profiling mode only; resets): ranks of the frames'
 * depth orders and (rank, super-tile) entries of their super-tile lists. */
int tsb_ctx_scan_counts(tsb_ctx* ctx, int64_t* ranks, int64_t* list_entries);

/* ---- scene: parameters, gradients, Adam state (trainer.cpp:63-132) ------- */
int tsb_scene_create(tsb_ctx* ctx, const tsb_scene_desc* desc, tsb_scene** out);
void tsb_scene_destroy(tsb_scene* s);
/* Upload parameters (replaces Params::from_scene / to_scene, trainer.cpp:70-104).
 * motion: n_keyframes * 3n floats (keyframe-major), may be NULL when static. */
int tsb_scene_set_params(tsb_scene* s, int where, const float* position, const float* log_scale,
                         const float* rotation, const float* opacity_logit,
                         const float* reflectivity_dc, const float* motion);
int tsb_scene_get_params(tsb_scene* s, float* position, float* log_scale, float* rotation,
                         float* opacity_logit, float* reflectivity_dc, float* motion);
/* Accumulated gradients (GroupGrads, trainer.cpp:107-132).  d_position is the
 * gradient w.r.t. the canonical mean (trainer.cpp:329-331); d_motion per keyframe.
 * d_bg_quad: 4 per frequency (SceneGrads::d_bg_quad); loss: summed loss. */
int tsb_scene_get_grads(tsb_scene* s, float* d_position, float* d_log_scale, float* d_rotation,
                        float* d_opacity_logit, float* d_reflectivity_dc, float* d_motion,
                        double* d_bg_quad, double* loss);
int tsb_scene_zero_grads(tsb_scene* s);
/* SceneGrads::d_bg_quad / d_bg_phasor (splat.hpp:87-89): 4 resp. 2 per frequency. */
int tsb_scene_get_bg_grads(tsb_scene* s, double* d_bg_quad, double* d_bg_phasor);
/* View-dependent reflectivity (sh_degree 1..3; sh.hpp:26-50, splat.cpp:163-165): all 16
 * reflectivity SH coefficients per Gaussian, [n][16] (coefficient 0 == reflectivity_dc).
 * tsb_scene_get_sh returns the parameters (grads = 0) or their accumulated gradients (grads = 1). */
int tsb_scene_set_sh(tsb_scene* s, int where, const float* refl_sh);
int tsb_scene_get_sh(tsb_scene* s, float* refl_sh, int grads);
/* Colour SH (Gaussian::color_sh, scene.hpp:23-38; tsb_scene_desc.color = 1): [n][48], row i =
 * Gaussian i's Eigen 16x3 block in storage order (coefficient k of channel c at 16 c + k).
 * tsb_scene_get_color returns the parameters (grads = 0) or SceneGrads::d_color_sh (grads = 1). */
int tsb_scene_set_color(tsb_scene* s, int where, const float* color_sh);
int tsb_scene_get_color(tsb_scene* s, float* color_sh, int grads);
/* SceneGrads::d_bg_color (splat.hpp:87-89), accumulated like the other background grads. */
int tsb_scene_get_bg_color_grad(tsb_scene* s, double* d_bg_color);
/* Adam moments (AdamState m_/v_, trainer.cpp:18-31), same layout as the params. */
int tsb_scene_get_adam_state(tsb_scene* s, float* m_position, float* v_position);
/* Densification statistic sum_i ||dL/dx_canon,i|| (trainer.cpp:381-384), n floats. */
int tsb_scene_get_densify_stat(tsb_scene* s, float* grad_norm_sum, int64_t* count);

/* Learning rates per parameter group (LrTable, trainer.hpp:36-44 resolved the
 * way fit() does, trainer.cpp:339-366). */
typedef struct {
    double position, log_scale, rotation, opacity, reflectivity, motion;
    double beta1, beta2, eps; /* AdamParams, trainer.hpp:14-18 */
    double color;             /* colour SH (LrTable::color) */
} tsb_adam_config;
/* One fused AdamState::step over every group (trainer.cpp:18-31, 339-366) +
 * densify statistic (trainer.cpp:381-384); clears the gradients afterwards. */
int tsb_scene_adam_step(tsb_scene* s, const tsb_adam_config* cfg);

/* AdamState::step on one flat parameter vector (trainer.cpp:18-31): m, v, params
 * updated in place; t is the step count after increment.  `where`: pointers are
 * host (copied through the device) or device memory. */
/* Densification surgery (trainer.cpp:385-470) with the Adam reindex (AdamState::reindex,
 * trainer.cpp:33-47), on the device: prune splats with sigmoid(opacity_logit) < opacity_floor
 * (in index order, never below min_count), then every survivor whose mean densify
 * statistic exceeds grad_threshold splits in two along its largest axis (largest scale >
 * split_scale_fraction x scene_extent) or is cloned.  New order: kept Gaussians, then the
 * extras in their parents' order; Adam moments follow kept Gaussians and start at zero for
 * new ones; gradients and the densify statistic are cleared.  *n_new = the new count. */
typedef struct {
    double grad_threshold, opacity_floor, split_scale_fraction, split_shrink;
    int32_t min_count;
} tsb_densify_config;
int tsb_scene_densify(tsb_scene* s, const tsb_densify_config* cfg, double scene_extent, int32_t* n_new);

int tsb_adam_step_flat(tsb_ctx* ctx, int where, float* params, const float* grads, float* m, float* v, size_t n,
                       int64_t t, double lr, double beta1, double beta2, double eps);
/* AdamState::reindex(src, stride) (trainer.hpp:25-29, trainer.cpp:33-47) on flat moment
 * vectors: new slot i (stride values) takes old slot src[i]'s m and v, or zeros when
 * src[i] < 0.  m / v hold n_old slots, src and the outputs n_new.  A device gather;
 * `where` = where all five pointers live. */
int tsb_adam_reindex_flat(tsb_ctx* ctx, int where, const float* m, const float* v, size_t n_old, const int32_t* src,
                          size_t n_new, int32_t stride, float* m_out, float* v_out);

/* ---- render pass (RenderPass, splat.hpp:97-117) ------------------------- */
/* A pass is a reusable per-frame workspace: prepare() == the RenderPass ctor
 * (prepare + depth sort + build_tiles, splat.cpp:90-200). */
int tsb_pass_create(tsb_ctx* ctx, tsb_pass** out);
void* tsb_pass_stream(tsb_pass* p);
void tsb_pass_destroy(tsb_pass* p);
int tsb_pass_prepare(tsb_pass* p, tsb_scene* s, const tsb_camera* cam,
                     const tsb_render_options* opt, const tsb_frame* frame);
/* RenderPass::visible_count (splat.hpp:108). */
int tsb_pass_visible_count(tsb_pass* p, int32_t* out);
/* Total length of the reference's tile lists (splat.cpp:187-200) for the frame: sum over
 * tiles of the visible Gaussians whose tile rect covers the tile.  The raster never
 * materialises these lists (each block scans the depth order for its own tile and stops
 * at termination); this count is computed on demand (parity / diagnostics). */
int tsb_pass_num_keys(tsb_pass* p, int64_t* out);

/* RenderPass::forward (splat.cpp:209-339).  Results stay in pass-owned device
 * buffers (tsb_pass_output).  With a target bound (planar [4*n_freq][H][W]
 * fp32, `where` = TSB_HOST/TSB_DEVICE), the forward epilogue also evaluates
 * sum_c channel_weight[c] * mse(quad_c, target_c) (losses.cpp:9-25,
 * trainer.cpp:210-219) and writes d_quad for the backward pass. */
int tsb_pass_forward(tsb_pass* p);
int tsb_pass_forward_loss(tsb_pass* p, int where, const float* target,
                          const double* channel_weight /* 4*n_freq */, double* loss_out /* may be NULL: no sync */);
/* The trainer's full image loss per quad channel c (losses.cpp:148-166, trainer.cpp:210-219):
 * sum_c channel_weight[c] * [(1 - ssim_mix) mse_c + ssim_mix (1 - SSIM_c)], SSIM with the
 * reference's 11-tap Gaussian window; d_quad for the backward.  ssim_mix 0 = forward_loss. */
int tsb_pass_forward_image_loss(tsb_pass* p, int where, const float* target, const double* channel_weight,
                                double ssim_mix, double* loss_out);

enum {
    TSB_OUT_QUAD = 0,      /* [4*n_freq][H][W] f32 */
    TSB_OUT_DEPTH_RAW = 1, /* [H][W] f32 */
    TSB_OUT_DEPTH = 2,     /* [H][W] f32 (NaN where weight <= coverage_eps) */
    TSB_OUT_WEIGHT = 3,    /* [H][W] f32 */
    TSB_OUT_TRANSM = 4,    /* [H][W] f32 */
    TSB_OUT_N_CONTRIB = 5, /* [H][W] i32 */
    TSB_OUT_N_PROCESSED = 6, /* [H][W] i32 */
    TSB_OUT_D_QUAD = 7,    /* [4*n_freq][H][W] f32 upstream gradient */
    TSB_OUT_PHASOR = 8,    /* [2*n_freq][H][W] f32 (re, im) */
    TSB_OUT_DISTORTION = 9, /* [H][W] f32 (TSB_CH_DISTORTION) */
    TSB_OUT_COLOR = 10,          /* [3][H][W] f32 (TSB_CH_COLOR) */
    TSB_OUT_MOTION_FWD_ACC = 11, /* [3][H][W] f32 sum_k w_k motion_fwd_k (TSB_CH_FLOW) */
    TSB_OUT_MOTION_BWD_ACC = 12, /* [3][H][W] */
    TSB_OUT_FLOW_FWD = 13,       /* [2][H][W] pixel displacement */
    TSB_OUT_FLOW_BWD = 14,       /* [2][H][W] */
    TSB_OUT_FLOW_VALID = 15,     /* [2][H][W] 1 where covered and projected in front (fwd, bwd) */
    TSB_OUT_D_MOTION_FWD_ACC = 16, /* [3][H][W] FlowLossResult::d_motion_fwd_acc (tsb_pass_flow_loss) */
    TSB_OUT_D_MOTION_BWD_ACC = 17, /* [3][H][W] */
    TSB_OUT_F64 = 18,            /* TSB_CH_EXACT: every plane of outputs 0-9 in fp64, [6*n_freq+5][H][W] double:
                                    quad (4*n_freq), depth_raw, depth, weight, T, phasor (2*n_freq), distortion */
    TSB_OUT_EXT_F64 = 19         /* TSB_CH_EXACT with colour / flow: [9][H][W] double (colour 3,
                                    motion_fwd_acc 3, motion_bwd_acc 3) */
};
/* Device pointer and byte size of a pass-owned buffer. */
int tsb_pass_output(tsb_pass* p, int which, void** dptr, size_t* bytes);
/* Per-Gaussian motions of the frame (RenderInput::motion_fwd / motion_bwd, splat.hpp:46-47;
 * n x 3 row-major = Matrix3Xd columns; NULL = zero) for TSB_CH_FLOW.  Call after prepare. */
int tsb_pass_set_motion(tsb_pass* p, int where, const float* motion_fwd, const float* motion_bwd);
/* flow_loss (losses.cpp:168-251) of the pass's last forward (needs TSB_CH_FLOW; settles it):
 * targets [3][H][W] = (u, v, valid) per direction or NULL.  value = mean squared flow error
 * over the directions with valid pixels; the motion-accumulator gradients, multiplied by
 * `weight` (the trainer's loss.flow factor, trainer.cpp:297-305), stay on the device as
 * outputs TSB_OUT_D_MOTION_FWD_ACC / _BWD_ACC (has_grads bit 0 / 1) for a
 * tsb_pass_backward_ext(TSB_DEVICE, ...). */
int tsb_pass_flow_loss(tsb_pass* p, int where, const float* target_fwd, const float* target_bwd, double weight,
                       double* value, int64_t* valid_pixels, int32_t* has_grads);
/* One render stack of write_render_stacks (eval.cpp:96-121, 165-185) from the pass's last
 * forward (needs TSB_CH_DISTORTION; colour written when TSB_CH_COLOR): into `dir` (created),
 * quad_QQQQQ_p0/_p90/_p180/_p270.pfm (first frequency), depth_QQQQQ.pfm (mean depth where
 * weight > 0.5, NaN elsewhere), dtof_QQQQQ.pfm (depth decoded from the rendered quad),
 * dd_QQQQQ.pfm (distortion) and color_QQQQQ.pfm, QQQQQ = quartet zero-padded to 5 digits.
 * The derived planes are computed on the device; the files are written on the host. */
int tsb_pass_render_stack(tsb_pass* p, const char* dir, int quartet);
/* SceneGrads::d_motion_fwd / d_motion_bwd (splat.hpp:86) of the last backward, n x 3 each. */
int tsb_pass_get_motion_grads(tsb_pass* p, float* d_motion_fwd, float* d_motion_bwd);
/* Copy a pass-owned buffer to host memory (synchronous). */
int tsb_pass_download(tsb_pass* p, int which, void* host, size_t bytes);
/* Enqueue the copy of a pass-owned buffer into host memory (pinned memory for
 * overlap) without waiting.  The bytes are valid after tsb_pass_wait or
 * tsb_ctx_synchronize (a frame redone after a device-side abort re-issues its
 * downloads).  The pass's next tsb_pass_prepare waits only for the forward, so
 * copies of consecutive frames stay in flight behind it (stream-ordered). */
int tsb_pass_download_async(tsb_pass* p, int which, void* host, size_t bytes);
/* Settle the pass (redo an aborted frame) and wait for everything enqueued on it. */
int tsb_pass_wait(tsb_pass* p);

/* RenderPass::backward (splat.cpp:347-650) for the quad channel.  d_quad: NULL
 * uses the loss residual written by tsb_pass_forward_loss, else an upstream
 * image [4*n_freq][H][W] (`where`).  Gradients are ACCUMULATED into the scene
 * (GroupGrads::add + trajectory chain, trainer.cpp:256, 312-331). */
int tsb_pass_backward(tsb_pass* p, int where, const float* d_quad);
/* RenderPass::backward(BufferGrads) (splat.cpp:347-650) with every ToF upstream
 * image of BufferGrads (splat.hpp:73-77): NULL skips a channel, as an empty Image
 * does in the reference.  Shapes: d_quad [4*n_freq][H][W], d_phasor [2*n_freq][H][W],
 * the rest [H][W].  A distortion upstream requires TSB_CH_DISTORTION in the forward. */
int tsb_pass_backward_buffers(tsb_pass* p, int where, const float* d_quad, const float* d_phasor,
                              const float* d_depth_raw, const float* d_weight,
                              const float* d_distortion, const float* d_transmittance);
/* The same with the colour / flow upstreams of BufferGrads (splat.hpp:73-77): d_color [3][H][W]
 * (needs TSB_CH_COLOR in the forward), d_motion_fwd_acc / d_motion_bwd_acc [3][H][W] (TSB_CH_FLOW). */
int tsb_pass_backward_ext(tsb_pass* p, int where, const float* d_quad, const float* d_phasor,
                          const float* d_depth_raw, const float* d_weight, const float* d_distortion,
                          const float* d_transmittance, const float* d_color, const float* d_motion_fwd_acc,
                          const float* d_motion_bwd_acc);

/* Parity / diagnostics: integer intermediates the reference keeps private
 * (splat.cpp:86-87).  Sizes: gidx V, rect 4V (x0,x1,y0,y1 per rank), tiles+1
 * offsets, K ids (indices into the prepared order; the complete lists, built on
 * demand from the depth order). */
int tsb_pass_debug_prepared(tsb_pass* p, int32_t* gidx, int32_t* rect);
int tsb_pass_debug_tiles(tsb_pass* p, int32_t* tiles_x, int32_t* tiles_y, int64_t* offsets,
                         int32_t* ids);
/* fp32 per-rank raster records (mean x/y, conic a/b/c, opacity, coef, depth,
 * sin/cos per frequency) and per-rank screen-space gradients after backward
 * (8 floats: d_mean2d x,y, d_conic a,b,c, d_opacity, d_coef, d_depth). */
int tsb_pass_debug_records(tsb_pass* p, float* rec12 /* 12 per rank */);
int tsb_pass_debug_screen_grads(tsb_pass* p, float* g8 /* 8 per rank */);
/* Keep a copy of the screen-space gradients of every following backward (the chain kernel
 * consumes them); required before tsb_pass_debug_screen_grads. */
int tsb_pass_debug_keep_screen(tsb_pass* p, int enabled);
/* Test hook: the pass builds super-tile lists for every frame (not only long orders) and
 * their storage (entries = (rank, super-tile) pairs) is set to `entries`; a frame that
 * needs more aborts on the device and is redone with grown lists when the pass settles
 * (the abort + settle/redo path). */
int tsb_pass_debug_set_list_capacity(tsb_pass* p, uint32_t entries);
/* Pixels the fp32 raster flagged as decision-ambiguous and recomposited in fp64. */
int tsb_pass_debug_fixups(tsb_pass* p, int32_t* count);
/* The fixed pixels themselves: pixel index | reason << 24 (1 maha, 2 alpha, 4 T band, 8 T relative
 * error bound above 1e-4 -- an almost opaque splat). */
int tsb_pass_debug_fixup_list(tsb_pass* p, int32_t* entries, int32_t capacity, int32_t* count);

/* ---- data-parallel gradient reduction (trainer.cpp:123-131 -> NCCL) ----- */
int tsb_comm_unique_id(void* out /* 128 bytes */);
int tsb_comm_create(tsb_ctx* ctx, const void* unique_id, int nranks, int rank, tsb_comm** out);
void tsb_comm_destroy(tsb_comm* c);
/* In-place sum of the scene's gradient buffer (+ bg grads + loss) across ranks. */
int tsb_scene_allreduce_grads(tsb_scene* s, tsb_comm* c);

/* ---- DeformNet on the tensor cores (deform.hpp:19-66, deform.cpp) -----
 * MLP (canonical position, time) -> position offset: positional encodings
 * (deform.cpp:10-26), `hidden_layers` ReLU layers of `width` units, a linear
 * 3-output layer.  Every layer is a tcgen05 GEMM (kind::tf32 with a 3xTF32 split,
 * fp32 accumulation in tensor memory).  Parameters are flat in the reference's
 * get_parameters order (per layer: W row-major, then b).  Limits: width <= 128,
 * input_dim = 3(1 + 2 l_x) + 1 + 2 l_t <= 128 (the reference's default 4 x 128, l = 10).
 * Each of TSB_DEFORM_SLOTS caches one forward (DeformNet::Cache) for its backward. */
#define TSB_DEFORM_SLOTS 4
typedef struct {
    int32_t hidden_layers, width, l_x, l_t;
    double coord_scale;
} tsb_deform_config;
typedef struct tsb_deform tsb_deform;
int tsb_deform_create(tsb_ctx* ctx, const tsb_deform_config* cfg, tsb_deform** out);
void tsb_deform_destroy(tsb_deform* net);
int64_t tsb_deform_param_count(const tsb_deform* net);
int tsb_deform_set_params(tsb_deform* net, int where, const float* flat);   /* DeformNet::set_parameters */
int tsb_deform_get_params(tsb_deform* net, float* host_flat);               /* DeformNet::get_parameters */
int tsb_deform_get_grads(tsb_deform* net, float* host_flat);                /* Grads::add_flat_to order */
int tsb_deform_zero_grads(tsb_deform* net);
/* DeformNet::offsets (deform.cpp:80-102): positions / offsets are n x 3 row-major
 * (the columns of a Matrix3Xd), host or device memory. */
int tsb_deform_offsets(tsb_deform* net, int slot, int where, const float* positions, int64_t n, double t,
                       float* offsets);
/* DeformNet::backward (deform.cpp:124-159) for the slot's cached forward: accumulates
 * dW / db; d_positions (n x 3, nullable) receives the input-position gradient. */
int tsb_deform_backward(tsb_deform* net, int slot, int where, const float* d_offsets, float* d_positions);
/* Scene coupling (trainer.cpp:262-271, 325-335): offsets of the scene's canonical
 * positions at time t become keyframe `keyframe`'s offsets; the backward consumes that
 * keyframe's accumulated gradient and adds d(offsets)/d(position) to the position grads. */
int tsb_deform_scene_offsets(tsb_deform* net, int slot, tsb_scene* scene, int keyframe, double t);
int tsb_deform_scene_backward(tsb_deform* net, int slot, tsb_scene* scene, int keyframe);
/* Test hook: the slot's cached post-ReLU activations of hidden layer `layer` (n x width). */
int tsb_deform_debug_activation(tsb_deform* net, int slot, int layer, float* host_out);
/* AdamState::step on the network parameters (trainer.cpp:18-31, 367-378). */
int tsb_deform_adam_step(tsb_deform* net, double lr, double beta1, double beta2, double eps);

/* Test hook for the DeformNet GEMM (tsb_mlp.cu): C[m][n] = act(sum_k A(m,k) B(n,k) + bias[n])
 * on the tcgen05 tensor cores (3xTF32), host buffers, A(m,k) = A[m*a_m + k*a_k],
 * B(n,k) = B[n*b_n + k*b_k], N <= 128, split over `slices` K ranges then reduced.
 * mask (nullable, M x N row-major): C *= (mask > 0). */
int tsb_debug_gemm(tsb_ctx* ctx, int M, int N, int K, int slices, const float* A, int64_t a_m, int64_t a_k,
                   const float* B, int64_t b_n, int64_t b_k, const float* bias, int relu, const float* mask,
                   float* C);

/* Portable FloatMap I/O (pfm.hpp, pfm.cpp:51-114) on planar [C][H][W] fp32 images: "Pf" = 1
 * channel, "PF" = 3 channels; rows bottom to top; written little-endian (scale -1.0), read in
 * either byte order.  tsb_read_pfm with planar = NULL only reports the dimensions.  Host only. */
int tsb_write_pfm(const char* path, const float* planar, int width, int height, int channels);
int tsb_read_pfm(const char* path, float* planar, size_t capacity_floats, int* width, int* height, int* channels);

/* ---- small host helpers mirroring the Python _core surface --------------- */
/* unambiguous_range (tof.hpp:36-38), quad_to_depth (tof.hpp:59-65),
 * quad_basis (tof.hpp:75-79); frequency <= 0 uses the default sensor. */
double tsb_unambiguous_range(double frequency);
double tsb_quad_to_depth(double q0, double q90, double q180, double q270, double frequency);
void tsb_quad_basis(double depth, double frequency, double* out4);

#ifdef __cplusplus
}
#endif
#endif /* TSB_H */
