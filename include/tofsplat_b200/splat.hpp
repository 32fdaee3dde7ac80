// tofsplat_b200/splat.hpp -- C++ drop-in shell for the reference renderer /
// optimiser API (proj/include/tofsplat/splat.hpp, trainer.hpp), implemented over
// the C ABI in tsb.h (link with paper_2505_05356_b200/lib/libtsb.so).
//
// Names, semantics and host layouts follow the reference:
//   Image            planar channel-major doubles, rows top to bottom (image.hpp:12-38)
//   Matrix3Xd/4Xd    3 x N / 4 x N column-major doubles (the Eigen storage order)
//   CameraModel      camera.hpp:9-49 (rotation row-major here)
//   Gaussian, CanonicalScene  scene.hpp:23-52 (reflectivity SH; colour is not on the ToF path)
//   RenderOptions, RenderInput, RenderedBuffers, BufferGrads, SceneGrads  splat.hpp:13-92
//   RenderPass{forward, backward, visible_count}, render, render_backward  splat.hpp:97-117
//   AdamParams, AdamState::step  trainer.hpp:14-34
// The Eigen headers the reference uses are absent from this image, so the matrix
// types are minimal layout-compatible stand-ins.  Errors are thrown as
// std::runtime_error carrying the reference's messages (splat.cpp:91-100).
// Parameters are converted to fp32 at the boundary; compute runs on the GPU only.
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "tsb.h"

namespace tofsplat {

inline void tsb_check(int rc) {
    if (rc != TSB_OK) throw std::runtime_error(tsb_last_error());
}

// ---- containers -------------------------------------------------------------
struct Image {
    int width = 0, height = 0, channels = 0;
    std::vector<double> data;
    Image() = default;
    Image(int w, int h, int c, double fill = 0.0)
        : width(w), height(h), channels(c), data(static_cast<size_t>(w) * h * c, fill) {}
    size_t plane_size() const { return static_cast<size_t>(width) * height; }
    double& at(int x, int y, int c = 0) { return data[c * plane_size() + static_cast<size_t>(y) * width + x]; }
    double at(int x, int y, int c = 0) const { return data[c * plane_size() + static_cast<size_t>(y) * width + x]; }
    const double* plane(int c) const { return data.data() + c * plane_size(); }
    double* plane(int c) { return data.data() + c * plane_size(); }
};
inline double invalid_value() { return std::numeric_limits<double>::quiet_NaN(); }
inline bool is_valid(double v) { return std::isfinite(v); }

template <int R>
struct MatrixRXd {  // R x N, column-major
    std::vector<double> storage;
    int n = 0;
    MatrixRXd() = default;
    explicit MatrixRXd(int cols) : storage(static_cast<size_t>(R) * cols, 0.0), n(cols) {}
    int cols() const { return n; }
    int rows() const { return R; }
    double& operator()(int r, int c) { return storage[static_cast<size_t>(c) * R + r]; }
    double operator()(int r, int c) const { return storage[static_cast<size_t>(c) * R + r]; }
    double* data() { return storage.data(); }
    const double* data() const { return storage.data(); }
};
using Matrix3Xd = MatrixRXd<3>;
using Matrix4Xd = MatrixRXd<4>;
using Matrix16Xd = MatrixRXd<16>;

constexpr double SH_C0 = 0.28209479177387814;
constexpr int kShCoeffCount = 16;

struct ToFConfig {
    double modulation_frequency = 29.9792458e6;
    double source_intensity = 1.0;
    double speed_of_light = 299792458.0;
};

struct CameraModel {
    double fx = 1.0, fy = 1.0, cx = 0.0, cy = 0.0;
    int width = 0, height = 0;
    double near_plane = 0.2, far_plane = 100.0;
    std::array<double, 9> rotation{1, 0, 0, 0, 1, 0, 0, 0, 1};  // row-major, p_cam = R p + t
    std::array<double, 3> translation{0, 0, 0};
    bool valid() const {
        return fx > 0 && fy > 0 && width > 0 && height > 0 && near_plane > 0 && far_plane > near_plane;
    }
};

struct Gaussian {
    std::array<double, 3> position{0, 0, 0};
    std::array<double, 3> log_scale{0, 0, 0};
    std::array<double, 4> rotation{1, 0, 0, 0};  // (w, x, y, z)
    double opacity_logit = 0.0;
    std::array<double, kShCoeffCount> reflectivity_sh{};
    std::array<std::array<double, 3>, kShCoeffCount> color_sh{};  // color_sh(k, c) = color_sh[k][c]
};

struct CanonicalScene {
    std::vector<Gaussian> gaussians;
    std::array<double, 4> bg_quad{0, 0, 0, 0};
    std::array<double, 3> bg_color{0, 0, 0};
    int sh_degree = 0;  // 0..3: reflectivity SH degree evaluated on the GPU
    ToFConfig tof;
    int size() const { return static_cast<int>(gaussians.size()); }
};

inline double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }
inline double logit(double p) { return std::log(p / (1.0 - p)); }

// ---- render API (splat.hpp:13-117) -----------------------------------------
struct RenderChannels {
    bool color = false;
    bool quad = true;
    bool phasor = false;
    bool depth = true;
    bool distortion = false;
    bool flow = false;  // implies depth (backprojection needs it)
};
struct Backgrounds {
    std::array<double, 3> color{0, 0, 0};
    std::array<double, 4> quad{0, 0, 0, 0};
    std::array<double, 2> phasor{0, 0};
};
struct RenderOptions {
    RenderChannels channels;
    Backgrounds bg;
    double alpha_threshold = 1.0 / 255.0;
    double transmittance_floor = 1e-4;
    double dilation = 0.3;
    double sigma_cutoff = 3.0;
    double coverage_eps = 1e-12;
    int tile_size = 16;
};
struct RenderInput {
    const CanonicalScene* scene = nullptr;
    const CameraModel* camera = nullptr;
    const Matrix3Xd* positions = nullptr;  // optional override of the means (one column per Gaussian)
    const Matrix3Xd* motion_fwd = nullptr;  // per-Gaussian motions for the flow channel
    const Matrix3Xd* motion_bwd = nullptr;
    RenderOptions opts;
};
struct RenderedBuffers {
    int width = 0, height = 0;
    Image color, quad, phasor, depth_raw, weight, depth, distortion, transmittance;
    Image motion_fwd_acc, motion_bwd_acc, flow_fwd, flow_bwd, flow_valid;
};
struct BufferGrads {  // leave an image empty to skip that channel (splat.hpp:68-77)
    Image d_color, d_quad, d_phasor;
    Image d_depth_raw, d_weight, d_distortion, d_transmittance;
    Image d_motion_fwd_acc, d_motion_bwd_acc;
};
struct SceneGrads {
    Matrix3Xd d_position, d_log_scale;
    Matrix4Xd d_rotation;
    std::vector<double> d_opacity_logit;
    Matrix16Xd d_reflectivity_sh;
    std::vector<std::array<std::array<double, 3>, kShCoeffCount>> d_color_sh;
    Matrix3Xd d_motion_fwd, d_motion_bwd;
    std::array<double, 4> d_bg_quad{0, 0, 0, 0};
    std::array<double, 3> d_bg_color{0, 0, 0};
    std::array<double, 2> d_bg_phasor{0, 0};
};

namespace detail {
struct Ctx {
    tsb_ctx* ctx = nullptr;
    Ctx() { tsb_check(tsb_ctx_create(0, &ctx)); }
    ~Ctx() { tsb_ctx_destroy(ctx); }
};
inline tsb_ctx* context() {
    static Ctx c;  // one context (stream) per process, device 0
    return c.ctx;
}
}  // namespace detail

class RenderPass {
public:
    explicit RenderPass(const RenderInput& in) : in_(in) {
        if (!in.scene || !in.camera) throw std::runtime_error("render: scene and camera required");
        if (!in.camera->valid()) throw std::runtime_error("render: invalid camera");
        const int n = in.scene->size();
        if (in.positions && in.positions->cols() != n) throw std::runtime_error("render: positions count mismatch");
        tsb_ctx* ctx = detail::context();
        tsb_scene_desc d{};
        d.n = n;
        d.n_keyframes = 0;
        d.sh_degree = in.scene->sh_degree;
        d.n_freq = 1;
        d.frequency[0] = in.scene->tof.modulation_frequency;
        d.source_intensity = in.scene->tof.source_intensity;
        d.speed_of_light = in.scene->tof.speed_of_light;
        const bool color = in.opts.channels.color;
        d.color = color ? 1 : 0;
        if (in.motion_fwd && in.motion_fwd->cols() != n) throw std::runtime_error("render: motion_fwd count mismatch");
        if (in.motion_bwd && in.motion_bwd->cols() != n) throw std::runtime_error("render: motion_bwd count mismatch");
        tsb_scene* s = nullptr;
        tsb_check(tsb_scene_create(ctx, &d, &s));
        scene_.reset(s);
        std::vector<float> pos(3 * (size_t)n), ls(3 * (size_t)n), rot(4 * (size_t)n), op(n), refl(n);
        for (int i = 0; i < n; ++i) {
            const Gaussian& g = in.scene->gaussians[i];
            for (int k = 0; k < 3; ++k) {
                pos[3 * i + k] = (float)(in.positions ? (*in.positions)(k, i) : g.position[k]);
                ls[3 * i + k] = (float)g.log_scale[k];
            }
            for (int k = 0; k < 4; ++k) rot[4 * i + k] = (float)g.rotation[k];
            op[i] = (float)g.opacity_logit;
            refl[i] = (float)g.reflectivity_sh[0];
        }
        tsb_check(tsb_scene_set_params(s, TSB_HOST, pos.data(), ls.data(), rot.data(), op.data(), refl.data(),
                                       nullptr));
        if (d.sh_degree > 0) {
            std::vector<float> sh(16 * (size_t)n);
            for (int i = 0; i < n; ++i)
                for (int k = 0; k < 16; ++k) sh[16 * (size_t)i + k] = (float)in.scene->gaussians[i].reflectivity_sh[k];
            tsb_check(tsb_scene_set_sh(s, TSB_HOST, sh.data()));
        }
        if (color) {
            std::vector<float> cs(48 * (size_t)n);
            for (int i = 0; i < n; ++i)
                for (int c = 0; c < 3; ++c)
                    for (int k = 0; k < 16; ++k)
                        cs[48 * (size_t)i + 16 * c + k] = (float)in.scene->gaussians[i].color_sh[k][c];
            tsb_check(tsb_scene_set_color(s, TSB_HOST, cs.data()));
        }
        tsb_pass* p = nullptr;
        tsb_check(tsb_pass_create(ctx, &p));
        pass_.reset(p);
        cam_ = tsb_camera{in.camera->fx, in.camera->fy, in.camera->cx, in.camera->cy, in.camera->width,
                          in.camera->height, in.camera->near_plane, in.camera->far_plane, {}, {}};
        for (int k = 0; k < 9; ++k) cam_.R[k] = in.camera->rotation[k];
        for (int k = 0; k < 3; ++k) cam_.t[k] = in.camera->translation[k];
        const RenderOptions& o = in.opts;
        opt_ = tsb_render_options{o.alpha_threshold, o.transmittance_floor, o.dilation, o.sigma_cutoff,
                                  o.coverage_eps, o.tile_size, TSB_CH_QUAD | TSB_CH_DEPTH | TSB_CH_PHASOR, {}, {}};
        if (o.channels.distortion) opt_.channels |= TSB_CH_DISTORTION;
        if (o.channels.color) opt_.channels |= TSB_CH_COLOR;
        if (o.channels.flow) opt_.channels |= TSB_CH_FLOW;
        for (int k = 0; k < 4; ++k) opt_.bg_quad[k] = o.bg.quad[k];
        for (int k = 0; k < 2; ++k) opt_.bg_phasor[k] = o.bg.phasor[k];
        for (int k = 0; k < 3; ++k) opt_.bg_color[k] = o.bg.color[k];
        tsb_check(tsb_pass_prepare(p, s, &cam_, &opt_, nullptr));
        if (o.channels.flow && (in.motion_fwd || in.motion_bwd)) {
            std::vector<float> m[2];
            const Matrix3Xd* src[2] = {in.motion_fwd, in.motion_bwd};
            for (int k = 0; k < 2; ++k) {
                if (!src[k]) continue;
                m[k].resize(3 * (size_t)n);
                for (int i = 0; i < n; ++i)
                    for (int a = 0; a < 3; ++a) m[k][3 * (size_t)i + a] = (float)(*src[k])(a, i);
            }
            tsb_check(tsb_pass_set_motion(p, TSB_HOST, src[0] ? m[0].data() : nullptr, src[1] ? m[1].data() : nullptr));
        }
    }

    int visible_count() const {
        int32_t v = 0;
        tsb_check(tsb_pass_visible_count(pass_.get(), &v));
        return v;
    }

    RenderedBuffers forward() const {
        tsb_check(tsb_pass_forward(pass_.get()));
        const int W = in_.camera->width, H = in_.camera->height;
        RenderedBuffers out;
        out.width = W;
        out.height = H;
        out.quad = download(TSB_OUT_QUAD, 4);
        out.depth_raw = download(TSB_OUT_DEPTH_RAW, 1);
        out.depth = download(TSB_OUT_DEPTH, 1);
        out.weight = download(TSB_OUT_WEIGHT, 1);
        out.transmittance = download(TSB_OUT_TRANSM, 1);
        if (in_.opts.channels.phasor) out.phasor = download(TSB_OUT_PHASOR, 2);
        if (in_.opts.channels.distortion) out.distortion = download(TSB_OUT_DISTORTION, 1);
        if (in_.opts.channels.color) out.color = download(TSB_OUT_COLOR, 3);
        if (in_.opts.channels.flow) {
            out.motion_fwd_acc = download(TSB_OUT_MOTION_FWD_ACC, 3);
            out.motion_bwd_acc = download(TSB_OUT_MOTION_BWD_ACC, 3);
            out.flow_fwd = download(TSB_OUT_FLOW_FWD, 2);
            out.flow_bwd = download(TSB_OUT_FLOW_BWD, 2);
            out.flow_valid = download(TSB_OUT_FLOW_VALID, 2);
        }
        forwarded_ = true;
        return out;
    }

    SceneGrads backward(const BufferGrads& up) const {
        if (!forwarded_) forward();
        const int n = in_.scene->size();
        tsb_check(tsb_scene_zero_grads(scene_.get()));
        const size_t HW = (size_t)in_.camera->width * in_.camera->height;
        std::vector<float> f[9];
        const Image* imgs[9] = {&up.d_quad, &up.d_phasor, &up.d_depth_raw, &up.d_weight, &up.d_distortion,
                                &up.d_transmittance, &up.d_color, &up.d_motion_fwd_acc, &up.d_motion_bwd_acc};
        const int nch[9] = {4, 2, 1, 1, 1, 1, 3, 3, 3};
        const float* ptr[9] = {};
        for (int i = 0; i < 9; ++i) {
            if (imgs[i]->data.empty()) continue;
            if (imgs[i]->data.size() != nch[i] * HW) throw std::runtime_error("render_backward: upstream size mismatch");
            f[i].assign(imgs[i]->data.begin(), imgs[i]->data.end());
            ptr[i] = f[i].data();
        }
        tsb_check(tsb_pass_backward_ext(pass_.get(), TSB_HOST, ptr[0], ptr[1], ptr[2], ptr[3], ptr[4], ptr[5], ptr[6],
                                        ptr[7], ptr[8]));
        std::vector<float> dp(3 * (size_t)n), dl(3 * (size_t)n), dr(4 * (size_t)n), dop(n), drf(n);
        double dbg[8] = {0};
        tsb_check(tsb_scene_get_grads(scene_.get(), dp.data(), dl.data(), dr.data(), dop.data(), drf.data(), nullptr,
                                      dbg, nullptr));
        SceneGrads g;
        g.d_position = Matrix3Xd(n);
        g.d_log_scale = Matrix3Xd(n);
        g.d_rotation = Matrix4Xd(n);
        g.d_opacity_logit.assign(n, 0.0);
        g.d_reflectivity_sh = Matrix16Xd(n);
        for (int i = 0; i < n; ++i) {
            for (int k = 0; k < 3; ++k) {
                g.d_position(k, i) = dp[3 * i + k];
                g.d_log_scale(k, i) = dl[3 * i + k];
            }
            for (int k = 0; k < 4; ++k) g.d_rotation(k, i) = dr[4 * i + k];
            g.d_opacity_logit[i] = dop[i];
            g.d_reflectivity_sh(0, i) = drf[i];
        }
        for (int k = 0; k < 4; ++k) g.d_bg_quad[k] = dbg[k];
        double dbp[4] = {0};
        tsb_check(tsb_scene_get_bg_grads(scene_.get(), nullptr, dbp));
        for (int k = 0; k < 2; ++k) g.d_bg_phasor[k] = dbp[k];
        if (in_.scene->sh_degree > 0) {
            std::vector<float> dsh(16 * (size_t)n);
            tsb_check(tsb_scene_get_sh(scene_.get(), dsh.data(), 1));
            for (int i = 0; i < n; ++i)
                for (int k = 0; k < 16; ++k) g.d_reflectivity_sh(k, i) = dsh[16 * (size_t)i + k];
        }
        g.d_color_sh.assign(n, {});
        g.d_motion_fwd = Matrix3Xd(n);
        g.d_motion_bwd = Matrix3Xd(n);
        if (in_.opts.channels.color) {
            std::vector<float> dcs(48 * (size_t)n);
            tsb_check(tsb_scene_get_color(scene_.get(), dcs.data(), 1));
            for (int i = 0; i < n; ++i)
                for (int c = 0; c < 3; ++c)
                    for (int k = 0; k < 16; ++k) g.d_color_sh[i][k][c] = dcs[48 * (size_t)i + 16 * c + k];
            double dbc[3] = {0, 0, 0};
            tsb_check(tsb_scene_get_bg_color_grad(scene_.get(), dbc));
            for (int k = 0; k < 3; ++k) g.d_bg_color[k] = dbc[k];
        }
        if (!up.d_color.data.empty() || !up.d_motion_fwd_acc.data.empty() || !up.d_motion_bwd_acc.data.empty()) {
            std::vector<float> mf(3 * (size_t)n), mb(3 * (size_t)n);
            tsb_check(tsb_pass_get_motion_grads(pass_.get(), mf.data(), mb.data()));
            for (int i = 0; i < n; ++i)
                for (int a = 0; a < 3; ++a) {
                    g.d_motion_fwd(a, i) = mf[3 * (size_t)i + a];
                    g.d_motion_bwd(a, i) = mb[3 * (size_t)i + a];
                }
        }
        return g;
    }

private:
    struct SceneDel {
        void operator()(tsb_scene* s) const { tsb_scene_destroy(s); }
    };
    struct PassDel {
        void operator()(tsb_pass* p) const { tsb_pass_destroy(p); }
    };
    Image download(int which, int channels) const {
        Image img(in_.camera->width, in_.camera->height, channels);
        std::vector<float> f(img.data.size());
        tsb_check(tsb_pass_download(pass_.get(), which, f.data(), f.size() * sizeof(float)));
        for (size_t i = 0; i < f.size(); ++i) img.data[i] = f[i];
        return img;
    }
    RenderInput in_;
    std::unique_ptr<tsb_scene, SceneDel> scene_;
    std::unique_ptr<tsb_pass, PassDel> pass_;
    tsb_camera cam_{};
    tsb_render_options opt_{};
    mutable bool forwarded_ = false;
};

inline RenderedBuffers render(const RenderInput& in) { return RenderPass(in).forward(); }
inline SceneGrads render_backward(const RenderInput& in, const BufferGrads& up) { return RenderPass(in).backward(up); }

// ---- optimiser (trainer.hpp:14-34) ------------------------------------------
struct AdamParams {
    double beta1 = 0.9;
    double beta2 = 0.999;
    double eps = 1e-15;
};

class AdamState {
public:
    void step(std::vector<double>& params, const std::vector<double>& grads, double lr, const AdamParams& ap) {
        if (params.size() != grads.size()) throw std::runtime_error("adam_step: size mismatch");
        if (m_.size() != params.size()) {
            m_.assign(params.size(), 0.f);
            v_.assign(params.size(), 0.f);
        }
        ++t_;
        std::vector<float> p(params.begin(), params.end()), g(grads.begin(), grads.end());
        tsb_check(tsb_adam_step_flat(detail::context(), TSB_HOST, p.data(), g.data(), m_.data(), v_.data(), p.size(),
                                     t_, lr, ap.beta1, ap.beta2, ap.eps));
        for (size_t i = 0; i < p.size(); ++i) params[i] = p[i];
    }
    long steps() const { return t_; }
    // trainer.cpp:33-47: slot i of the new parameter layout takes the moments of old slot
    // src[i] (stride values per slot), fresh zeros where src[i] < 0; never-stepped: no-op.
    void reindex(const std::vector<int>& src, int stride) {
        if (m_.empty()) return;
        if (stride < 1) throw std::runtime_error("adam_reindex: stride must be >= 1");
        const size_t n_old = m_.size() / (size_t)stride;
        std::vector<int32_t> s(src.begin(), src.end());
        std::vector<float> m2(s.size() * (size_t)stride), v2(s.size() * (size_t)stride);
        tsb_check(tsb_adam_reindex_flat(detail::context(), TSB_HOST, m_.data(), v_.data(), n_old, s.data(), s.size(),
                                        stride, m2.data(), v2.data()));
        m_ = std::move(m2);
        v_ = std::move(v2);
    }

private:
    std::vector<float> m_, v_;
    long t_ = 0;
};

// ---- tof.hpp helpers ----------------------------------------------------------
inline double unambiguous_range(const ToFConfig& tof) { return tsb_unambiguous_range(tof.modulation_frequency); }
inline std::array<double, 4> quad_basis(double depth, const ToFConfig& tof) {
    std::array<double, 4> b{};
    tsb_quad_basis(depth, tof.modulation_frequency, b.data());
    return b;
}

}  // namespace tofsplat
