"""Pin the CPU oracle (oracle/tofsplat_oracle.c) to the reference's own known-answer
tests and properties.  The reference cannot be built here (Eigen3 absent), so these
restated KATs are the pin.  Each test cites the reference test it restates."""
import math

import numpy as np
import pytest

from oracle import oracle as orc

SH_C0 = 0.28209479177387814
F_DEFAULT = 29.9792458e6
C_LIGHT = 299792458.0


class Cam:
    def __init__(self, w=64, h=48, f=40.0, cx=None, cy=None, near=0.2, far=100.0):
        self.fx = self.fy = f
        self.cx = w // 2 + 0.5 if cx is None else cx
        self.cy = h // 2 + 0.5 if cy is None else cy
        self.width, self.height = w, h
        self.near_plane, self.far_plane = near, far
        self.rotation = np.eye(3)
        self.translation = np.zeros(3)


class Opts:
    def __init__(self, **kw):
        self.alpha_threshold = 1.0 / 255.0
        self.transmittance_floor = 1e-4
        self.dilation = 0.3
        self.sigma_cutoff = 3.0
        self.coverage_eps = 1e-12
        self.tile_size = 16
        self.bg_quad = np.zeros(4)
        self.bg_phasor = np.zeros(2)
        for k, v in kw.items():
            setattr(self, k, v)


def dc_scene(gs, source_intensity=1.0, sh_degree=0):
    """gs: list of (pos, scale, reflectivity, opacity_logit)  (test_splat.cpp:25-34)."""
    n = len(gs)
    pos = np.array([g[0] for g in gs], float).reshape(n, 3)
    ls = np.log(np.array([[g[1]] * 3 for g in gs], float)).reshape(n, 3)
    rot = np.tile([1.0, 0, 0, 0], (n, 1))
    op = np.array([g[3] for g in gs], float)
    refl = np.zeros((n, 16))
    refl[:, 0] = [g[2] / SH_C0 for g in gs]
    return orc.OScene(pos, ls, rot, op, refl, sh_degree, F_DEFAULT, source_intensity, C_LIGHT)


def random_scene(n, seed, sh_degree=3):
    """Same distributions as test_splat.cpp:36-53 (numpy RNG instead of mt19937_64)."""
    rng = np.random.default_rng(seed)
    u = rng.uniform
    pos = np.stack([2 * u(size=n) - 1, 2 * u(size=n) - 1, 0.8 + 4 * u(size=n)], 1)
    ls = np.log(0.05 + 0.4 * u(size=(n, 1))) + 0.3 * u(size=(n, 3))
    rot = np.stack([1 + u(size=n), u(size=n) - 0.5, u(size=n) - 0.5, u(size=n) - 0.5], 1)
    op = 4 * u(size=n) - 2
    refl = np.zeros((n, 16))
    refl[:, 0] = (0.2 + 0.6 * u(size=n)) / SH_C0
    refl[:, 1:] = 0.05 * (u(size=(n, 15)) - 0.5)
    return orc.OScene(pos, ls, rot, op, refl, sh_degree, F_DEFAULT, 1.0, C_LIGHT)


def phase(d, f=F_DEFAULT):
    return 4.0 * math.pi * d * f / C_LIGHT


# ---- tof.hpp / test_tof.cpp ------------------------------------------------
def test_tof_helpers_through_abi():
    """test_tof.cpp:17-57 via the product's host helpers (no GPU needed)."""
    import paper_2505_05356_b200 as tsb
    assert tsb.unambiguous_range() == pytest.approx(5.0, abs=1e-12)
    assert tsb.unambiguous_range(59.9584916e6) == pytest.approx(2.5, abs=1e-12)
    assert tsb.quad_to_depth(3.0, 4.0, 3.0, 2.0) == pytest.approx(0.0, abs=1e-12)

    def synth(d, a, b):
        return [a * x + b for x in tsb.quad_basis(d)]
    assert tsb.quad_to_depth(*synth(2.0, 1.0, 0.0)) == pytest.approx(2.0, rel=1e-9)
    assert tsb.quad_to_depth(*synth(6.0, 1.0, 0.0)) == pytest.approx(1.0, rel=1e-9)
    assert math.isnan(tsb.quad_to_depth(1.0, 1.0, 1.0, 1.0))
    du = tsb.unambiguous_range()
    for i in range(1, 1000, 37):
        d = du * i / 1000.0
        assert abs(tsb.quad_to_depth(*synth(d, 0.7, 0.3)) - d) < 1e-9 * du


# ---- scene.cpp / test_scene.cpp, sh.hpp / test_camera_sh.cpp ----------------
def test_quat_to_rotation():
    """test_scene.cpp:16-27."""
    assert np.allclose(orc.quat_to_rotation([1, 0, 0, 0]), np.eye(3))
    s = math.sqrt(0.5)
    R = orc.quat_to_rotation([s, 0, 0, s])
    assert np.linalg.norm(R @ [1, 0, 0] - np.array([0, 1, 0])) < 1e-12
    q = np.array([0.3, -0.8, 0.5, 0.1])
    assert np.allclose(orc.quat_to_rotation(q), orc.quat_to_rotation(2.5 * q), atol=1e-12)


def test_covariance_eigenvalues():
    """test_scene.cpp:29-54: eigenvalues of R S S^T R^T are exp(2 log_scale)."""
    rng = np.random.default_rng(11)
    for _ in range(10):
        ls = rng.uniform(-1, 1, 3)
        q = np.array([rng.uniform(-1, 1) + 1.5, *rng.uniform(-1, 1, 3)])
        R = orc.quat_to_rotation(q)
        M = R * np.exp(ls)[None, :]
        ev = np.sort(np.linalg.eigvalsh(M @ M.T))
        want = np.sort(np.exp(2 * ls))
        assert np.abs(ev - want).max() < 1e-9 * want.max()


def test_sh_basis_and_jacobian():
    """test_camera_sh.cpp:67-111."""
    b = orc.sh_basis([0, 0, 1], 0)
    assert b[0] == pytest.approx(SH_C0) and (b[1:] == 0).all()
    d = np.array([0.48, -0.6, 0.64])
    b = orc.sh_basis(d, 3)
    assert b[1] == pytest.approx(-0.4886025119029199 * d[1])
    assert b[2] == pytest.approx(0.4886025119029199 * d[2])
    assert b[3] == pytest.approx(-0.4886025119029199 * d[0])
    rng = np.random.default_rng(7)
    h = 1e-6
    for _ in range(10):
        d = rng.uniform(-1, 1, 3)
        if np.linalg.norm(d) < 0.3:
            d[2] += 1.0
        d /= np.linalg.norm(d)
        J = orc.sh_basis_jacobian(d, 3)
        for ax in range(3):
            dp, dm = d.copy(), d.copy()
            dp[ax] += h
            dm[ax] -= h
            fd = (orc.sh_basis(dp, 3) - orc.sh_basis(dm, 3)) / (2 * h)
            assert (np.abs(J[:, ax] - fd) < 1e-5 * np.maximum(1.0, np.maximum(np.abs(fd), np.abs(J[:, ax])))).all()


# ---- splat.cpp / test_splat.cpp ---------------------------------------------
def test_empty_scene_passes_background():
    """test_splat.cpp:62-103."""
    sc = dc_scene([])
    cam = Cam()
    p = orc.OraclePass(sc, cam, Opts(bg_quad=np.array([1.0, 2, 3, 4]), bg_phasor=np.array([-0.5, 0.7])))
    assert p.visible_count() == 0
    out = p.forward()
    assert (out["transmittance"] == 1).all() and (out["weight"] == 0).all()
    for c in range(4):
        assert (out["quad"][c] == c + 1.0).all()
    assert np.isnan(out["depth"]).all()
    g = p.backward(d_quad=np.ones((4, 48, 64)))
    assert np.allclose(g["d_bg_quad"], 64 * 48)


def test_single_on_axis_splat():
    """test_splat.cpp:105-143 (closed form to 1e-9)."""
    cam = Cam(64, 48, 50.0)
    z, s, o, r = 2.0, 0.2, 0.7, 0.5
    sc = dc_scene([([0, 0, z], s, r, math.log(o / (1 - o)))])
    bg = np.array([0.3, 0.1, -0.2, 0.4])
    out = orc.OraclePass(sc, cam, Opts(bg_quad=bg)).forward()
    var = (cam.fx * s / z) ** 2 + 0.3
    psi = phase(z)
    basis = [math.sin(psi), math.cos(psi), -math.sin(psi), -math.cos(psi)]
    coef = r / (z * z)
    for dx, dy in [(0, 0), (1, 0), (0, 2), (-3, 4), (5, -2)]:
        x, y = 32 + dx, 24 + dy
        alpha = o * math.exp(-0.5 * (dx * dx + dy * dy) / var)
        assert out["weight"][y, x] == pytest.approx(alpha, rel=1e-9)
        assert out["transmittance"][y, x] == pytest.approx(1 - alpha, rel=1e-9)
        assert out["depth"][y, x] == pytest.approx(z, rel=1e-12)
        assert out["distortion"][y, x] == pytest.approx(0.0, abs=1e-12)
        t = 1 - alpha
        for c in range(4):
            assert out["quad"][c, y, x] == pytest.approx(coef * alpha * basis[c] + bg[c] * t * t, rel=1e-9, abs=1e-12)
    assert out["weight"][0, 0] == 0.0 and np.isnan(out["depth"][0, 0])


def test_conservation_and_phasor_agreement():
    """test_splat.cpp:145-175 (weight + T = 1 to 1e-12; phasor = (q90-q270, q0-q180)*... to 1e-13)."""
    for seed in (101, 202):
        p = orc.OraclePass(random_scene(60, seed), Cam(48, 36, 30.0), Opts())
        out = p.forward()
        assert np.abs(out["weight"] + out["transmittance"] - 1.0).max() < 1e-12
        q = out["quad"]
        # phasor = 2 coef w2 (cos, sin) and q90 - q270 = 2 coef w2 cos, q0 - q180 = 2 coef w2 sin
        assert np.abs(out["phasor"][0] - (q[1] - q[3])).max() < 1e-13
        assert np.abs(out["phasor"][1] - (q[0] - q[2])).max() < 1e-13


def test_two_layered_splats():
    """test_splat.cpp:177-217 and acceptance check 3 (acceptance.cpp:154-201)."""
    sc = dc_scene([([0, 0, 1.0], 0.1, 1 / 32, 0.0), ([0, 0, 4.0], 0.4, 1.0, 40.0)], source_intensity=32.0)
    out = orc.OraclePass(sc, Cam(), Opts()).forward()
    x, y = 32, 24
    c5 = math.cos(2 * math.pi / 5)
    q = out["quad"][:, y, x]
    assert q[0] == pytest.approx(0, abs=1e-9) and q[2] == pytest.approx(0, abs=1e-9)
    assert q[1] == pytest.approx(c5, rel=1e-9) and q[3] == pytest.approx(-c5, rel=1e-9)
    assert out["weight"][y, x] == pytest.approx(1.0, rel=1e-9)
    assert out["depth"][y, x] == pytest.approx(2.5, rel=1e-9)
    assert out["distortion"][y, x] == pytest.approx(4.5, rel=1e-9)
    assert out["transmittance"][y, x] == pytest.approx(0.0, abs=1e-9)
    assert out["phasor"][0, y, x] == pytest.approx(2 * c5, rel=1e-9)
    # acceptance 3 on an 8x8 camera with principal point on a pixel centre
    cam = Cam(8, 8, 50.0, cx=4.5, cy=4.5, far=50.0)
    out = orc.OraclePass(sc, cam, Opts()).forward()
    assert out["weight"][4, 4] == pytest.approx(1.0, abs=1e-6)
    assert out["depth"][4, 4] == pytest.approx(2.5, abs=1e-6)
    assert out["distortion"][4, 4] == pytest.approx(4.5, abs=1e-6)


def test_culling():
    """test_splat.cpp:219-233."""
    sc = dc_scene([([0, 0, 0.05], 0.01, 0.5, 2.0), ([0, 0, -2.0], 0.1, 0.5, 2.0), ([100, 0, 2.0], 0.1, 0.5, 2.0)])
    p = orc.OraclePass(sc, Cam(), Opts())
    assert p.visible_count() == 0
    assert p.forward()["weight"][24, 32] == 0.0


def test_tile_size_invariance_bitwise():
    """test_splat.cpp:235-266: results are bit-identical for tile sizes 16, 5, 64."""
    sc = random_scene(50, 303)
    outs = [orc.OraclePass(sc, Cam(48, 36, 30.0), Opts(tile_size=t)).forward() for t in (16, 5, 64)]
    for o in outs[1:]:
        for k in ("quad", "phasor", "depth_raw", "weight", "transmittance", "distortion", "n_contrib"):
            assert np.array_equal(outs[0][k], o[k]), k
        assert np.array_equal(outs[0]["depth"], o["depth"], equal_nan=True)


def test_tile_lists_follow_global_order():
    """build_tiles (splat.cpp:187-200): each tile's list is the increasing prepared order of
    the splats whose rect touches it."""
    p = orc.OraclePass(random_scene(200, 5), Cam(96, 72, 60.0), Opts())
    off, ids = p.tile_lists()
    rect = p.prepared()["rect"]
    tx, ty = p.tiles()
    for t in range(tx * ty):
        lst = ids[off[t]:off[t + 1]]
        assert (np.diff(lst) > 0).all()
        x, y = (t % tx) * 16, (t // tx) * 16
        want = [i for i, r in enumerate(rect) if r[0] // 16 <= t % tx <= (r[1] - 1) // 16
                and r[2] // 16 <= t // tx <= (r[3] - 1) // 16]
        assert list(lst) == want


def test_invalid_camera_raises():
    """splat.cpp:91-92."""
    with pytest.raises(RuntimeError, match="render: invalid camera"):
        orc.OraclePass(random_scene(3, 1), Cam(0, 10, 10.0), Opts())


# ---- losses.cpp / trainer.cpp -----------------------------------------------
def test_mse():
    """test_losses.cpp:23-37."""
    v, g = orc.mse([1.0, 3.0], [0.0, 1.0])
    assert v == pytest.approx(2.5)
    assert g[0] == pytest.approx(1.0) and g[1] == pytest.approx(2.0)
    assert orc.mse([1.0, 3.0], [1.0, 3.0], False) == 0.0
    with pytest.raises(RuntimeError):
        orc.mse([1.0, 3.0], [0.0, 1.0, 2.0])


def test_adam():
    """test_trainer.cpp:14-49."""
    p = np.linspace(1, 4, 4)
    before = p.copy()
    m, v = np.zeros(4), np.zeros(4)
    orc.adam_step(p, np.zeros(4), m, v, 1, 0.1)
    assert (p == before).all()
    p = np.zeros(3)
    g = np.array([2.0, -0.5, 1e-3])
    m, v = np.zeros(3), np.zeros(3)
    orc.adam_step(p, g, m, v, 1, 0.01)
    assert np.allclose(p, -0.01 * np.sign(g), rtol=1e-9)
    pa = np.full(2, 0.3)
    pb = pa.copy()
    ma, va, mb, vb = (np.zeros(2) for _ in range(4))
    g = np.array([0.7, -0.1])
    for t in range(1, 11):
        orc.adam_step(pa, g.copy(), ma, va, t, 0.05)
        orc.adam_step(pb, g.copy(), mb, vb, t, 0.05)
        g = g * -0.9
    assert (pa == pb).all()


def test_interp_positions_exact_endpoints():
    """acceptance.cpp:334-352 / deform.cpp:248-251: exact endpoints, affine inside."""
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (40, 3))
    da, db = rng.normal(0, 0.05, (2, 40, 3))
    assert np.array_equal(orc.interp_positions(x, da, db, 0.0), x + da)
    assert np.array_equal(orc.interp_positions(x, da, db, 1.0), x + db)
    ws = [s / 7 for s in range(8)]
    P = [orc.interp_positions(x, da, db, w) for w in ws]
    assert max(np.abs(P[s + 2] - 2 * P[s + 1] + P[s]).max() for s in range(6)) < 1e-9


# ---- gradcheck.cpp: finite differences vs the analytic backward -------------
def _gradcheck_setup(seed=7, n=4, w=8, h=8):
    """Restates make_setup (gradcheck.cpp:38-99) with numpy's RNG."""
    rng = np.random.default_rng(seed)
    u = rng.uniform
    cam = Cam(w, h, 0.75 * w, cx=0.5 * w, cy=0.5 * h)
    pos, ls, rot, op, refl = [], [], [], [], []
    for i in range(n):
        z = 1.0 + 0.45 * i + u(0.05, 0.25)
        pos.append([u(-0.25, 0.25) * z, u(-0.2, 0.2) * z, z])
        ls.append(np.log(u(0.08, 0.3, 3)))
        q = u(-1, 1, 4)
        if np.linalg.norm(q) < 0.3:
            q[0] += 1
        rot.append(q)
        op.append(u(-1.0, 1.5))
        r = np.zeros(16)
        r[0] = u(0.3, 0.7) / SH_C0
        r[1:] = u(-0.05, 0.05, 15)
        refl.append(r)
    sc = orc.OScene(np.array(pos), np.array(ls), np.array(rot), np.array(op), np.array(refl), 3, F_DEFAULT, 1.0,
                    C_LIGHT)
    opts = Opts(alpha_threshold=0.0, transmittance_floor=0.0, sigma_cutoff=6.0,
                bg_quad=u(-1, 1, 4), bg_phasor=u(-1, 1, 2))
    ups = {"d_quad": u(-1, 1, (4, h, w)), "d_phasor": u(-1, 1, (2, h, w)), "d_depth_raw": u(-1, 1, (1, h, w)),
           "d_weight": u(-1, 1, (1, h, w)), "d_distortion": u(-1, 1, (1, h, w)),
           "d_transmittance": u(-1, 1, (1, h, w))}
    return sc, cam, opts, ups


def _objective(sc, cam, opts, ups):
    out = orc.OraclePass(sc, cam, opts).forward()
    return (np.sum(out["quad"] * ups["d_quad"]) + np.sum(out["phasor"] * ups["d_phasor"]) +
            np.sum(out["depth_raw"] * ups["d_depth_raw"][0]) + np.sum(out["weight"] * ups["d_weight"][0]) +
            np.sum(out["distortion"] * ups["d_distortion"][0]) +
            np.sum(out["transmittance"] * ups["d_transmittance"][0]))


@pytest.mark.parametrize("seed", [7, 11])
def test_gradcheck_oracle_backward(seed):
    """gradcheck.cpp:155-247 on the oracle: central differences (h = 1e-4), rel < 1e-3
    (acceptance.cpp:67-74) for every parameter group the ToF path has."""
    sc, cam, opts, ups = _gradcheck_setup(seed)
    g = orc.OraclePass(sc, cam, opts).backward(**ups)
    hstep = 1e-4
    worst = {}

    def probe(arr, idx):
        orig = arr[idx]
        arr[idx] = orig + hstep
        jp = _objective(sc, cam, opts, ups)
        arr[idx] = orig - hstep
        jm = _objective(sc, cam, opts, ups)
        arr[idx] = orig
        return (jp - jm) / (2 * hstep)

    def rel(a, b):
        return abs(a - b) / max(abs(a), abs(b), 1e-6)

    groups = [("position", sc.position, g["d_position"]), ("log_scale", sc.log_scale, g["d_log_scale"]),
              ("rotation", sc.rotation, g["d_rotation"]), ("opacity", sc.opacity_logit, g["d_opacity_logit"]),
              ("reflectivity_sh", sc.refl_sh, g["d_refl_sh"]), ("bg_quad", opts.bg_quad, g["d_bg_quad"]),
              ("bg_phasor", opts.bg_phasor, g["d_bg_phasor"])]
    for name, arr, an in groups:
        worst[name] = max(rel(an[idx], probe(arr, idx)) for idx in np.ndindex(arr.shape))
    assert max(worst.values()) < 1e-3, worst


def _objective_ext(sc, cam, opts, ups):
    p = orc.OraclePass(sc, cam, opts)
    out, ext = p.forward(), p.forward_ext()
    return (np.sum(out["quad"] * ups["d_quad"]) + np.sum(out["depth_raw"] * ups["d_depth_raw"][0]) +
            np.sum(ext["color"] * ups["d_color"]) + np.sum(ext["motion_fwd_acc"] * ups["d_motion_fwd_acc"]) +
            np.sum(ext["motion_bwd_acc"] * ups["d_motion_bwd_acc"]))


def test_gradcheck_oracle_colour_and_motion_channels():
    """gradcheck.cpp (all channels) for the colour and flow accumulators: colour SH (degree 3,
    clamp gates), motion vectors, colour background, and their effect on positions/opacity."""
    sc, cam, opts, ups = _gradcheck_setup(5)
    rng = np.random.default_rng(9)
    n, h, w = sc.n, cam.height, cam.width
    cs = np.zeros((n, 48))
    for c in range(3):
        cs[:, 16 * c] = rng.uniform(0.2, 0.8, n) / SH_C0
        cs[:, 16 * c + 1:16 * c + 16] = rng.uniform(-0.05, 0.05, (n, 15))
    sc.color_sh = cs
    sc.motion_fwd = rng.uniform(-0.1, 0.1, (n, 3))
    sc.motion_bwd = rng.uniform(-0.1, 0.1, (n, 3))
    opts.bg_color = rng.uniform(0, 1, 3)
    ups = {"d_quad": ups["d_quad"], "d_depth_raw": ups["d_depth_raw"], "d_color": rng.uniform(-1, 1, (3, h, w)),
           "d_motion_fwd_acc": rng.uniform(-1, 1, (3, h, w)), "d_motion_bwd_acc": rng.uniform(-1, 1, (3, h, w))}
    g = orc.OraclePass(sc, cam, opts).backward(**ups)
    hstep = 1e-5

    def probe(arr, idx):
        orig = arr[idx]
        arr[idx] = orig + hstep
        jp = _objective_ext(sc, cam, opts, ups)
        arr[idx] = orig - hstep
        jm = _objective_ext(sc, cam, opts, ups)
        arr[idx] = orig
        return (jp - jm) / (2 * hstep)

    def rel(a, b):
        return abs(a - b) / max(abs(a), abs(b), 1e-6)

    worst = {}
    for name, arr, an in [("color_sh", sc.color_sh, g["d_color_sh"]), ("motion_fwd", sc.motion_fwd, g["d_motion_fwd"]),
                          ("motion_bwd", sc.motion_bwd, g["d_motion_bwd"]), ("bg_color", opts.bg_color, g["d_bg_color"]),
                          ("position", sc.position, g["d_position"]), ("opacity", sc.opacity_logit,
                                                                       g["d_opacity_logit"])]:
        worst[name] = max(rel(an[idx], probe(arr, idx)) for idx in np.ndindex(arr.shape))
    assert max(worst.values()) < 1e-3, worst


def test_flow_projection_closed_form():
    """A single opaque splat moving by m: flow = projection of (backprojected point + m) minus the
    pixel (splat.cpp:315-333); valid where covered and in front."""
    cam = Cam(16, 16, 20.0, cx=8.0, cy=8.0)
    sc = orc.OScene(np.array([[0.0, 0.0, 2.0]]), np.log(np.full((1, 3), 0.5)), np.array([[1.0, 0, 0, 0]]),
                    np.array([8.0]), np.zeros((1, 16)), 0, F_DEFAULT, 1.0, C_LIGHT)
    sc.motion_fwd = np.array([[0.1, -0.05, 0.0]])
    sc.motion_bwd = np.array([[0.0, 0.0, -3.0]])  # moves behind the camera: bwd flow invalid
    ext = orc.OraclePass(sc, cam, Opts()).forward_ext()
    out = orc.OraclePass(sc, cam, Opts()).forward()
    y, x = 8, 8
    SW = out["weight"][y, x]
    depth = out["depth"][y, x]
    d = np.array([(x + 0.5 - 8.0) / 20.0, (y + 0.5 - 8.0) / 20.0, 1.0])
    xd = depth * d / np.linalg.norm(d) + ext["motion_fwd_acc"][:, y, x]
    assert ext["flow_valid"][0, y, x] == 1.0 and SW > 0.9
    assert np.isclose(ext["flow_fwd"][0, y, x], 20.0 * xd[0] / xd[2] + 8.0 - (x + 0.5), atol=1e-12)
    assert np.isclose(ext["flow_fwd"][1, y, x], 20.0 * xd[1] / xd[2] + 8.0 - (y + 0.5), atol=1e-12)
    assert ext["flow_valid"][1, y, x] == 0.0
