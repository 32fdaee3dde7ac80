// C++ drop-in test: the reference's test_splat.cpp / test_trainer.cpp cases
// (proj/tests/unit/test_splat.cpp:62-292, test_trainer.cpp:14-35) written against
// include/tofsplat_b200/splat.hpp, i.e. the reference API names running on the B200
// library.  Tolerances are the fp32 ones stated in DESIGN.md.
#include <cmath>
#include <cstdio>
#include <random>

#include "tofsplat_b200/splat.hpp"

using namespace tofsplat;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        ++g_checks;                                                          \
        if (!(cond)) {                                                       \
            ++g_fail;                                                        \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);      \
        }                                                                    \
    } while (0)
static bool close_rel(double a, double b, double rel, double abs_ = 0.0) {
    return std::abs(a - b) <= std::max(abs_, rel * std::max(std::abs(a), std::abs(b)));
}

static CameraModel test_camera(int w = 64, int h = 48, double f = 40.0) {
    CameraModel cam;
    cam.fx = cam.fy = f;
    cam.cx = w / 2 + 0.5;
    cam.cy = h / 2 + 0.5;
    cam.width = w;
    cam.height = h;
    return cam;
}

static Gaussian dc_gaussian(std::array<double, 3> pos, double scale, double reflectivity, double opacity_logit) {
    Gaussian g;
    g.position = pos;
    g.log_scale = {std::log(scale), std::log(scale), std::log(scale)};
    g.opacity_logit = opacity_logit;
    g.reflectivity_sh[0] = reflectivity / SH_C0;
    return g;
}

static CanonicalScene random_scene(int n, unsigned seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    CanonicalScene s;
    s.gaussians.resize(n);
    for (Gaussian& g : s.gaussians) {
        g.position = {2 * u(rng) - 1, 2 * u(rng) - 1, 0.8 + 4 * u(rng)};
        const double ls = std::log(0.05 + 0.4 * u(rng));
        g.log_scale = {ls + 0.3 * u(rng), ls + 0.3 * u(rng), ls + 0.3 * u(rng)};
        g.rotation = {1 + u(rng), u(rng) - 0.5, u(rng) - 0.5, u(rng) - 0.5};
        g.opacity_logit = 4 * u(rng) - 2;
        g.reflectivity_sh[0] = (0.2 + 0.6 * u(rng)) / SH_C0;
    }
    return s;
}

static void empty_scene_passes_background() {
    CanonicalScene scene;
    const CameraModel cam = test_camera();
    RenderInput in;
    in.scene = &scene;
    in.camera = &cam;
    in.opts.bg.quad = {1.0, 2.0, 3.0, 4.0};
    RenderPass pass(in);
    CHECK(pass.visible_count() == 0);
    const RenderedBuffers out = pass.forward();
    bool ok = true;
    for (int y = 0; y < out.height; ++y)
        for (int x = 0; x < out.width; ++x) {
            ok &= out.transmittance.at(x, y) == 1.0 && out.weight.at(x, y) == 0.0 && !is_valid(out.depth.at(x, y));
            for (int c = 0; c < 4; ++c) ok &= out.quad.at(x, y, c) == in.opts.bg.quad[c];
        }
    CHECK(ok);
    BufferGrads up;
    up.d_quad = Image(out.width, out.height, 4, 1.0);
    const SceneGrads g = pass.backward(up);
    for (int c = 0; c < 4; ++c) CHECK(close_rel(g.d_bg_quad[c], out.width * out.height, 1e-12));
}

static void single_on_axis_splat() {
    const CameraModel cam = test_camera(64, 48, 50.0);
    CanonicalScene scene;
    const double z = 2.0, s = 0.2, o = 0.7, r = 0.5;
    scene.gaussians.push_back(dc_gaussian({0.0, 0.0, z}, s, r, logit(o)));
    RenderInput in;
    in.scene = &scene;
    in.camera = &cam;
    in.opts.bg.quad = {0.3, 0.1, -0.2, 0.4};
    const RenderedBuffers out = render(in);
    const double var = (cam.fx * s / z) * (cam.fx * s / z) + in.opts.dilation;
    const auto basis = quad_basis(z, scene.tof);
    const double coef = r / (z * z);
    const int offs[5][2] = {{0, 0}, {1, 0}, {0, 2}, {-3, 4}, {5, -2}};
    for (const auto& off : offs) {
        const int x = 32 + off[0], y = 24 + off[1];
        const double alpha = o * std::exp(-0.5 * (off[0] * off[0] + off[1] * off[1]) / var);
        CHECK(close_rel(out.weight.at(x, y), alpha, 2e-6));
        CHECK(close_rel(out.transmittance.at(x, y), 1.0 - alpha, 2e-6));
        CHECK(close_rel(out.depth.at(x, y), z, 1e-6));
        const double t = 1.0 - alpha;
        for (int c = 0; c < 4; ++c)
            CHECK(close_rel(out.quad.at(x, y, c), coef * alpha * basis[c] + in.opts.bg.quad[c] * t * t, 1e-5, 1e-6));
    }
    CHECK(out.weight.at(0, 0) == 0.0 && !is_valid(out.depth.at(0, 0)));
}

static void two_layered_splats() {
    CanonicalScene scene;
    scene.tof.source_intensity = 32.0;
    scene.gaussians.push_back(dc_gaussian({0.0, 0.0, 1.0}, 0.1, 1.0 / 32.0, 0.0));
    scene.gaussians.push_back(dc_gaussian({0.0, 0.0, 4.0}, 0.4, 1.0, 40.0));
    const CameraModel cam = test_camera();
    RenderInput in;
    in.scene = &scene;
    in.camera = &cam;
    const RenderedBuffers out = render(in);
    const double c5 = std::cos(2.0 * M_PI / 5.0);
    CHECK(std::abs(out.quad.at(32, 24, 0)) < 1e-6 && std::abs(out.quad.at(32, 24, 2)) < 1e-6);
    CHECK(close_rel(out.quad.at(32, 24, 1), c5, 1e-5) && close_rel(out.quad.at(32, 24, 3), -c5, 1e-5));
    CHECK(close_rel(out.weight.at(32, 24), 1.0, 1e-6));
    CHECK(close_rel(out.depth.at(32, 24), 2.5, 1e-6));
}

// RenderChannels::phasor / ::distortion (splat.cpp:305-314) and the phasor background gradient.
static void phasor_and_distortion() {
    CanonicalScene scene;
    scene.tof.source_intensity = 32.0;
    scene.gaussians.push_back(dc_gaussian({0.0, 0.0, 1.0}, 0.1, 1.0 / 32.0, 0.0));
    scene.gaussians.push_back(dc_gaussian({0.0, 0.0, 4.0}, 0.4, 1.0, 40.0));
    const CameraModel cam = test_camera();
    RenderInput in;
    in.scene = &scene;
    in.camera = &cam;
    in.opts.channels.phasor = true;
    in.opts.channels.distortion = true;
    const RenderedBuffers out = render(in);
    // phasor = (q90 - q270, q0 - q180) without background; weights 0.5 / 0.5 at depths 1 and 4
    CHECK(close_rel(out.phasor.at(32, 24, 0), out.quad.at(32, 24, 1) - out.quad.at(32, 24, 3), 1e-5, 1e-7));
    CHECK(close_rel(out.phasor.at(32, 24, 1), out.quad.at(32, 24, 0) - out.quad.at(32, 24, 2), 1e-5, 1e-6));
    CHECK(close_rel(out.distortion.at(32, 24), 2.0 * 0.5 * 0.5 * 9.0, 1e-5));
    CHECK(out.distortion.at(0, 0) == 0.0);

    CanonicalScene empty;
    RenderInput ein = in;
    ein.scene = &empty;
    ein.opts.bg.phasor = {0.5, -0.25};
    RenderPass pass(ein);
    const RenderedBuffers eo = pass.forward();
    CHECK(eo.phasor.at(3, 4, 0) == 0.5 && eo.phasor.at(3, 4, 1) == -0.25);
    BufferGrads up;
    up.d_phasor = Image(cam.width, cam.height, 2, 1.0);
    up.d_transmittance = Image(cam.width, cam.height, 1, 1.0);
    const SceneGrads g = pass.backward(up);
    for (int c = 0; c < 2; ++c) CHECK(close_rel(g.d_bg_phasor[c], cam.width * cam.height, 1e-12));
    CHECK(g.d_bg_quad[0] == 0.0);
}

static void culling() {
    const CameraModel cam = test_camera();
    CanonicalScene scene;
    scene.gaussians.push_back(dc_gaussian({0.0, 0.0, 0.05}, 0.01, 0.5, 2.0));
    scene.gaussians.push_back(dc_gaussian({0.0, 0.0, -2.0}, 0.1, 0.5, 2.0));
    scene.gaussians.push_back(dc_gaussian({100.0, 0.0, 2.0}, 0.1, 0.5, 2.0));
    RenderInput in;
    in.scene = &scene;
    in.camera = &cam;
    RenderPass pass(in);
    CHECK(pass.visible_count() == 0);
    CHECK(pass.forward().weight.at(32, 24) == 0.0);
}

static void tile_size_and_override() {
    const CanonicalScene scene = random_scene(50, 303);
    const CameraModel cam = test_camera(48, 36, 30.0);
    RenderInput in;
    in.scene = &scene;
    in.camera = &cam;
    in.opts.tile_size = 16;
    const RenderedBuffers a = render(in);
    for (int ts : {5, 64}) {
        in.opts.tile_size = ts;
        const RenderedBuffers b = render(in);
        bool ok = true;
        for (size_t i = 0; i < a.quad.data.size(); ++i) ok &= close_rel(a.quad.data[i], b.quad.data[i], 1e-5, 1e-7);
        for (size_t i = 0; i < a.weight.data.size(); ++i) ok &= close_rel(a.weight.data[i], b.weight.data[i], 1e-5);
        CHECK(ok);
    }
    in.opts.tile_size = 16;
    const RenderedBuffers again = render(in);
    CHECK(again.quad.data == a.quad.data);  // repeated renders are bit-identical
    // position override == scene with moved means (bitwise)
    Matrix3Xd moved(scene.size());
    CanonicalScene baked = scene;
    for (int i = 0; i < scene.size(); ++i)
        for (int k = 0; k < 3; ++k) {
            moved(k, i) = scene.gaussians[i].position[k] + (k == 0 ? 0.1 : k == 1 ? -0.05 : 0.2 * (i % 3));
            baked.gaussians[i].position[k] = moved(k, i);
        }
    in.positions = &moved;
    const RenderedBuffers o = render(in);
    RenderInput in2;
    in2.scene = &baked;
    in2.camera = &cam;
    const RenderedBuffers d = render(in2);
    CHECK(o.quad.data == d.quad.data && o.weight.data == d.weight.data);
}

static void errors_match_reference() {
    CanonicalScene scene;
    CameraModel bad;
    RenderInput in;
    in.scene = &scene;
    in.camera = &bad;
    bool threw = false;
    try {
        RenderPass p(in);
    } catch (const std::runtime_error& e) {
        threw = std::string(e.what()) == "render: invalid camera";
    }
    CHECK(threw);
    in.camera = nullptr;
    threw = false;
    try {
        RenderPass p(in);
    } catch (const std::runtime_error& e) {
        threw = std::string(e.what()) == "render: scene and camera required";
    }
    CHECK(threw);
}

static void adam_steps() {
    AdamParams ap;
    AdamState st;
    std::vector<double> p = {1, 2, 3, 4};
    const std::vector<double> before = p;
    st.step(p, {0, 0, 0, 0}, 0.1, ap);
    CHECK(p == before && st.steps() == 1);
    AdamState st2;
    std::vector<double> q = {0, 0, 0};
    st2.step(q, {2.0, -0.5, 1e-3}, 0.01, ap);
    CHECK(close_rel(q[0], -0.01, 1e-6) && close_rel(q[1], 0.01, 1e-6) && close_rel(q[2], -0.01, 1e-6));
    // test_trainer.cpp:50-70: reindex copies and clears moments
    AdamState st3;
    std::vector<double> p3 = {0, 0, 0, 0};  // two gaussians, stride 2
    st3.step(p3, {1.0, 2.0, 3.0, 4.0}, 0.1, ap);
    st3.reindex({1, 1, -1}, 2);  // keep gaussian 1, clone gaussian 1, fresh slot
    std::vector<double> p4(6, 0.0);
    st3.step(p4, std::vector<double>(6, 0.0), 0.1, ap);  // zero grads: moments decay but stay aligned
    CHECK(p4[0] == p4[2] && p4[1] == p4[3] && p4[0] != 0.0);
    CHECK(p4[4] == 0.0 && p4[5] == 0.0);
    CHECK(st3.steps() == 2);
}

// Colour channel + background colour gradient (test_splat.cpp:62-101, colour parts).
static void colour_background() {
    CanonicalScene scene;
    const CameraModel cam = test_camera();
    RenderInput in;
    in.scene = &scene;
    in.camera = &cam;
    in.opts.channels.color = true;
    in.opts.bg.color = {0.2, 0.4, 0.6};
    RenderPass pass(in);
    const RenderedBuffers out = pass.forward();
    bool all_bg = true;
    for (int y = 0; y < out.height; ++y)
        for (int x = 0; x < out.width; ++x)
            for (int c = 0; c < 3; ++c) all_bg &= out.color.at(x, y, c) == (float)in.opts.bg.color[c];
    CHECK(all_bg);
    BufferGrads up;
    up.d_color = Image(out.width, out.height, 3);
    std::fill(up.d_color.data.begin(), up.d_color.data.end(), 1.0);
    const SceneGrads g = pass.backward(up);
    const double npx = out.width * out.height;
    for (int c = 0; c < 3; ++c) CHECK(close_rel(g.d_bg_color[c], npx, 1e-6));
    // an opaque grey splat on axis: colour = c alpha + bg (1 - alpha)
    CanonicalScene one;
    Gaussian gs = dc_gaussian({0.0, 0.0, 2.0}, 0.2, 0.5, logit(0.7));
    for (int c = 0; c < 3; ++c) gs.color_sh[0][c] = (0.25 + 0.25 * c) / SH_C0;
    one.gaussians.push_back(gs);
    in.scene = &one;
    const RenderedBuffers o1 = render(in);
    const double alpha = o1.weight.at(32, 24);
    for (int c = 0; c < 3; ++c)
        CHECK(close_rel(o1.color.at(32, 24, c), (0.25 + 0.25 * c) * alpha + in.opts.bg.color[c] * (1.0 - alpha), 1e-5));
}

// Flow channel (test_splat.cpp:294-333).
static void flow_projection() {
    const CameraModel cam = test_camera(64, 48, 50.0);
    CanonicalScene scene;
    scene.gaussians.push_back(dc_gaussian({0.0, 0.0, 2.0}, 0.2, 0.5, 40.0));
    Matrix3Xd motion_fwd(1), motion_bwd(1);
    const double mf[3] = {0.1, -0.05, 0.3}, mb[3] = {-0.2, 0.0, 0.1};
    for (int a = 0; a < 3; ++a) {
        motion_fwd(a, 0) = mf[a];
        motion_bwd(a, 0) = mb[a];
    }
    RenderInput in;
    in.scene = &scene;
    in.camera = &cam;
    in.motion_fwd = &motion_fwd;
    in.motion_bwd = &motion_bwd;
    in.opts.channels.flow = true;
    const RenderedBuffers out = render(in);
    const int cx = 32, cy = 24;
    CHECK(out.flow_valid.at(cx, cy, 0) == 1.0 && out.flow_valid.at(cx, cy, 1) == 1.0);
    CHECK(close_rel(out.flow_fwd.at(cx, cy, 0), 50.0 * 0.1 / 2.3, 1e-5));
    CHECK(close_rel(out.flow_fwd.at(cx, cy, 1), 50.0 * -0.05 / 2.3, 1e-5));
    CHECK(close_rel(out.flow_bwd.at(cx, cy, 0), 50.0 * -0.2 / 2.1, 1e-5));
    CHECK(std::abs(out.flow_bwd.at(cx, cy, 1)) < 1e-5);
    const int x = 36, y = 24;
    const double w = out.weight.at(x, y);
    CHECK(w > 0.1);
    for (int c = 0; c < 3; ++c) CHECK(close_rel(out.motion_fwd_acc.at(x, y, c), w * mf[c], 1e-5));
    CHECK(out.flow_valid.at(0, 0, 0) == 0.0 && out.flow_fwd.at(0, 0, 0) == 0.0);
}

int main() {
    empty_scene_passes_background();
    single_on_axis_splat();
    two_layered_splats();
    phasor_and_distortion();
    culling();
    tile_size_and_override();
    errors_match_reference();
    adam_steps();
    colour_background();
    flow_projection();
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
