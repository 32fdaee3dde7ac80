"""Colour and flow channels of RenderPass on the B200 (tsb_ext.cu) against the CPU oracle.

Forward: splat.cpp:273-294 (colour / motion accumulators), 301-334 (bg colour, flow by
backprojection of the composited depth + reprojection of x + motion, flow_valid).
Backward: the colour / motion upstreams of BufferGrads (splat.cpp:361-505) and their chain
(colour SH gated by 0 < colour_raw < 1, view-direction term, d_motion_*; splat.cpp:560-571).
Tolerances as the ToF channels: images 1e-4 relative, gradients 1e-3 relative."""
import numpy as np
import pytest

from oracle import oracle as orc

from helpers import rel_err, rel_err_quantile

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4
GRAD_TOL = 1e-3


@pytest.fixture(scope="module")
def tsb():
    import paper_2505_05356_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(tsb):
    return tsb.Context(0)


def _colour_sh(rng, n, degree):
    """(n, 16, 3): DC around mid-grey (some channels pushed out of [0, 1] so the clamp gate
    is exercised), small higher-order terms up to `degree`."""
    cs = np.zeros((n, 16, 3), np.float32)
    c0 = 0.28209479177387814
    cs[:, 0, :] = (rng.uniform(0.1, 0.9, (n, 3)) / c0).astype(np.float32)
    out = rng.uniform(size=(n, 3)) < 0.08
    cs[:, 0, :][out] = (rng.choice([-0.5, 1.6], size=out.sum()) / c0).astype(np.float32)
    nk = (degree + 1) ** 2
    if nk > 1:
        cs[:, 1:nk, :] = (0.1 * (rng.uniform(size=(n, nk - 1, 3)) - 0.5)).astype(np.float32)
    return cs


def _setup(tsb, ctx, degree, n=3000, seed=31):
    from paper_2505_05356_b200 import synthetic
    g = synthetic.gaussians(n, seed, n_keyframes=2)
    rng = np.random.default_rng(seed + 1)
    sh = np.zeros((n, 16), np.float32)
    sh[:, 0] = g.reflectivity_dc
    if degree > 0:
        sh[:, 1:(degree + 1) ** 2] = (0.05 * (rng.uniform(size=(n, (degree + 1) ** 2 - 1)) - 0.5)).astype(np.float32)
    cs = _colour_sh(rng, n, degree)
    mf = (0.05 * rng.normal(size=(n, 3))).astype(np.float32)
    mb = (0.05 * rng.normal(size=(n, 3))).astype(np.float32)
    tof = tsb.ToFConfig(30e6)
    scene = tsb.GaussianScene(ctx, n, 2, tof, sh_degree=degree, color=True)
    scene.set_params(g.position, g.log_scale, g.rotation, g.opacity_logit, g.reflectivity_dc, g.motion)
    if degree > 0:
        scene.set_sh(sh)
    scene.set_color(cs)
    return g, sh, cs, mf, mb, scene, tof


def _oscene(g, frame, sh, cs, mf, mb, degree):
    n = g.n
    return orc.OScene(g.rendered_means(frame), g.log_scale.astype(np.float64), g.rotation.astype(np.float64),
                      g.opacity_logit.astype(np.float64), sh.astype(np.float64), degree, 30e6, 1.0, 299792458.0,
                      color_sh=cs.astype(np.float64).transpose(0, 2, 1).reshape(n, 48).copy(),
                      motion_fwd=None if mf is None else mf.astype(np.float64),
                      motion_bwd=None if mb is None else mb.astype(np.float64))


def _check_img(a, b, floor=1e-3):
    assert rel_err(a, b, floor) < IMG_TOL
    assert np.abs(np.asarray(a, np.float64) - b).max() <= 2e-6 * max(np.abs(b).max(), 1e-30)


def _check_signed(a, b):
    """Motion accumulators sum signed terms that cancel (like the raw samples, see
    test_gpu_parity.check_image): 1e-4 relative above 1e-2 max, 99.9th percentile of the
    relative error above 1e-3 max below 1e-4, absolute error below 2e-6 max everywhere."""
    assert rel_err(a, b, 1e-2) < IMG_TOL
    assert rel_err_quantile(a, b, 1e-3, 0.999) < IMG_TOL
    assert np.abs(np.asarray(a, np.float64) - b).max() <= 2e-6 * max(np.abs(b).max(), 1e-30)


def test_color_sh_roundtrip(tsb, ctx):
    _, _, cs, _, _, scene, _ = _setup(tsb, ctx, 2, n=500)
    assert np.array_equal(scene.get_color(), cs)


@pytest.mark.parametrize("degree", [0, 3])
def test_color_flow_forward_and_backward(tsb, ctx, degree):
    from paper_2505_05356_b200 import synthetic
    g, sh, cs, mf, mb, scene, tof = _setup(tsb, ctx, degree)
    cam = synthetic.camera(200, 150, 180.0)
    H, W = cam.height, cam.width
    frame = (0, 0.4)
    opts = tsb.RenderOptions(counts=True, color=True, flow=True, bg_color=(0.2, 0.5, 0.8))
    rp = tsb.RenderPass(ctx).prepare(scene, cam, opts, frame)
    rp.set_motion(mf, mb)
    rp.forward()
    out = rp.outputs()

    op = orc.OraclePass(_oscene(g, frame, sh, cs, mf, mb, degree), cam, opts)
    ref = op.forward()
    ext = op.forward_ext()
    assert np.array_equal(out["n_contrib"], ref["n_contrib"])
    _check_img(out["color"], ext["color"])
    for k in ("motion_fwd_acc", "motion_bwd_acc"):
        _check_signed(out[k], ext[k])
    assert np.array_equal(out["flow_valid"], ext["flow_valid"])
    for k in ("flow_fwd", "flow_bwd"):
        # flow is a pixel displacement: absolute tolerance (1e-4 px + 1e-4 relative)
        d = np.abs(out[k].astype(np.float64) - ext[k])
        assert (d <= 1e-4 + 1e-4 * np.abs(ext[k])).all(), d.max()

    rng = np.random.default_rng(5)
    ups = {"d_color": rng.normal(0, 1e-3, (3, H, W)).astype(np.float32),
           "d_motion_fwd_acc": rng.normal(0, 1e-3, (3, H, W)).astype(np.float32),
           "d_motion_bwd_acc": rng.normal(0, 1e-3, (3, H, W)).astype(np.float32),
           "d_quad": rng.normal(0, 1e-3, (4, H, W)).astype(np.float32)}
    rp.backward_buffers(**ups)
    gr = scene.grads()
    dcs = scene.get_color(grads=True)
    dmf, dmb = rp.motion_grads()
    og = op.backward(**{k: v.astype(np.float64) for k, v in ups.items()})
    k, w = frame
    errs = {"d_position": rel_err(gr["d_position"], og["d_position"], 1e-4),
            "d_log_scale": rel_err(gr["d_log_scale"], og["d_log_scale"], 1e-4),
            "d_rotation": rel_err(gr["d_rotation"], og["d_rotation"], 1e-4),
            "d_opacity_logit": rel_err(gr["d_opacity_logit"], og["d_opacity_logit"], 1e-4),
            "d_motion_k": rel_err(gr["d_motion"][k], (1 - w) * og["d_position"], 1e-4),
            "d_motion_k1": rel_err(gr["d_motion"][k + 1], w * og["d_position"], 1e-4),
            "d_color_sh": rel_err(dcs.transpose(0, 2, 1).reshape(g.n, 48), og["d_color_sh"], 1e-4),
            "d_motion_fwd": rel_err(dmf, og["d_motion_fwd"], 1e-4),
            "d_motion_bwd": rel_err(dmb, og["d_motion_bwd"], 1e-4)}
    assert all(e < GRAD_TOL for e in errs.values()), errs
    assert np.allclose(gr["d_bg_color"], og["d_bg_color"], rtol=1e-4, atol=1e-9)
    # the colour gate: clamped channels get no SH gradient
    assert np.abs(og["d_color_sh"]).max() > 0


def test_color_only_upstream_and_no_motion(tsb, ctx):
    """Colour upstream alone, flow without motions (zero motion -> flow of the static point)."""
    from paper_2505_05356_b200 import synthetic
    g, sh, cs, _, _, scene, tof = _setup(tsb, ctx, 1, n=2000, seed=44)
    cam = synthetic.camera(160, 120, 150.0)
    frame = (0, 0.0)
    opts = tsb.RenderOptions(color=True, flow=True, bg_color=(1.0, 0.0, 0.5))
    rp = tsb.RenderPass(ctx).prepare(scene, cam, opts, frame).forward()
    out = rp.outputs()
    op = orc.OraclePass(_oscene(g, frame, sh, cs, None, None, 1), cam, opts)
    op.forward()
    ext = op.forward_ext()
    _check_img(out["color"], ext["color"])
    assert np.array_equal(out["flow_valid"], ext["flow_valid"])
    assert np.abs(out["flow_fwd"] - ext["flow_fwd"]).max() <= 1e-4
    up = np.random.default_rng(2).normal(0, 1e-3, (3, 120, 160)).astype(np.float32)
    rp.backward_buffers(d_color=up)
    gr = scene.grads()
    og = op.backward(d_color=up.astype(np.float64))
    assert rel_err(gr["d_position"], og["d_position"], 1e-4) < GRAD_TOL
    assert rel_err(scene.get_color(grads=True).transpose(0, 2, 1).reshape(g.n, 48), og["d_color_sh"], 1e-4) < GRAD_TOL
    assert np.allclose(gr["d_bg_color"], og["d_bg_color"], rtol=1e-4, atol=1e-9)


def test_color_upstream_requires_channel(tsb, ctx):
    from paper_2505_05356_b200 import synthetic
    _, _, _, _, _, scene, _ = _setup(tsb, ctx, 0, n=300)
    cam = synthetic.camera(64, 48, 60.0)
    rp = tsb.RenderPass(ctx).prepare(scene, cam, tsb.RenderOptions(), (0, 0.0)).forward()
    with pytest.raises(RuntimeError, match="colour"):
        rp.backward_buffers(d_color=np.zeros((3, 48, 64), np.float32))
    with pytest.raises(RuntimeError, match="motion"):
        rp.backward_buffers(d_motion_fwd_acc=np.zeros((3, 48, 64), np.float32))


def test_flow_loss_and_its_backward(tsb, ctx):
    """flow_loss (losses.cpp:168-251) on the device against oracle/losses.flow_loss on the oracle's
    render, then the backward of image loss + weighted flow loss (trainer.cpp:285-317)."""
    from oracle import losses as ol
    from paper_2505_05356_b200 import synthetic
    g, sh, cs, mf, mb, scene, tof = _setup(tsb, ctx, 0, n=3000, seed=52)
    cam = synthetic.camera(200, 150, 180.0)
    H, W = cam.height, cam.width
    frame = (0, 0.6)
    opts = tsb.RenderOptions(counts=True, flow=True)
    rp = tsb.RenderPass(ctx).prepare(scene, cam, opts, frame)
    rp.set_motion(mf, mb)
    rng = np.random.default_rng(17)
    target = rng.normal(0, 0.05, (4, H, W)).astype(np.float32)
    loss = rp.forward_loss(target)
    out = rp.outputs()
    tf = np.stack([rng.uniform(-2, 2, (H, W)), rng.uniform(-2, 2, (H, W)),
                   (rng.uniform(size=(H, W)) > 0.3).astype(float)]).astype(np.float32)
    tb = np.stack([rng.uniform(-2, 2, (H, W)), rng.uniform(-2, 2, (H, W)), np.ones((H, W))]).astype(np.float32)
    weight = 0.7
    value, valid = rp.flow_loss(tf, tb, weight)
    dmf_up, dmb_up = rp.flow_loss_grads()

    op = orc.OraclePass(_oscene(g, frame, sh, cs, mf, mb, 0), cam, opts)
    ref = dict(op.forward())
    ref.update(op.forward_ext())
    assert np.array_equal(out["flow_valid"], ref["flow_valid"])
    fl = ol.flow_loss(ref, cam, tf.astype(np.float64), tb.astype(np.float64))
    assert valid == fl["valid_pixels"] > 0
    assert value == pytest.approx(fl["value"], rel=1e-4)
    assert rel_err(dmf_up, weight * fl["d_motion_fwd_acc"], 1e-4) < GRAD_TOL
    assert rel_err(dmb_up, weight * fl["d_motion_bwd_acc"], 1e-4) < GRAD_TOL

    rp.backward_flow()
    gr = scene.grads()
    dmf, dmb = rp.motion_grads()
    d_quad = np.zeros((4, H, W))
    for m in range(4):
        _, d = orc.mse(ref["quad"][m], target[m].astype(np.float64))
        d_quad[m] = 0.25 * d
    og = op.backward(d_quad=d_quad, d_motion_fwd_acc=weight * fl["d_motion_fwd_acc"],
                     d_motion_bwd_acc=weight * fl["d_motion_bwd_acc"])
    errs = {"d_position": rel_err(gr["d_position"], og["d_position"], 1e-4),
            "d_opacity_logit": rel_err(gr["d_opacity_logit"], og["d_opacity_logit"], 1e-4),
            "d_log_scale": rel_err(gr["d_log_scale"], og["d_log_scale"], 1e-4),
            "d_motion_fwd": rel_err(dmf, og["d_motion_fwd"], 1e-4),
            "d_motion_bwd": rel_err(dmb, og["d_motion_bwd"], 1e-4)}
    assert all(e < GRAD_TOL for e in errs.values()), errs
    assert loss > 0


def test_flow_loss_masking_and_errors(tsb, ctx):
    """test_losses.cpp:162-217 semantics on the device: target = render -> 0; + (3, 0) -> 9;
    a direction without targets has no gradient; empty validity -> 0 and no gradient."""
    from paper_2505_05356_b200 import synthetic
    _, _, _, mf, mb, scene, _ = _setup(tsb, ctx, 0, n=1500, seed=61)
    cam = synthetic.camera(96, 64, 90.0)
    rp = tsb.RenderPass(ctx).prepare(scene, cam, tsb.RenderOptions(flow=True), (0, 0.3))
    rp.set_motion(mf, mb)
    rp.forward()
    out = rp.outputs()
    tf = np.concatenate([out["flow_fwd"], np.ones((1, 64, 96), np.float32)])
    v, n = rp.flow_loss(tf, None)
    assert abs(v) < 1e-12 and n == int((out["flow_valid"][0] > 0.5).sum()) > 0
    t3 = tf.copy()
    t3[0] += 3.0
    v, _ = rp.flow_loss(t3, None)
    assert v == pytest.approx(9.0, rel=1e-6)
    assert rp.flow_loss_grads()[1] is None and rp.flow_loss_grads()[0] is not None
    none = tf.copy()
    none[2] = 0.0
    v, n = rp.flow_loss(none, None)
    assert v == 0.0 and n == 0 and rp.flow_loss_grads() == (None, None)
    rq = tsb.RenderPass(ctx).prepare(scene, cam, tsb.RenderOptions(), (0, 0.3)).forward()
    with pytest.raises(RuntimeError, match="flow channels"):
        rq.flow_loss(tf, None)


def test_render_stack_files(tsb, ctx, tmp_path):
    """write_render_stacks (eval.cpp:96-121, 165-185) for one quartet: the PFM files and
    their planes against the pass's own outputs and the numpy restatement (oracle/pfm.py)."""
    from oracle import pfm as opfm
    from paper_2505_05356_b200 import synthetic
    g, sh, cs, _, _, scene, tof = _setup(tsb, ctx, 0, n=2500, seed=71)
    cam = synthetic.camera(96, 72, 90.0)
    opts = tsb.RenderOptions(distortion=True, color=True, bg_color=(0.1, 0.2, 0.3))
    rp = tsb.RenderPass(ctx).prepare(scene, cam, opts, (0, 0.5)).forward()
    out = rp.outputs()
    rp.write_render_stack(tmp_path, 7)
    assert sorted(p.name for p in tmp_path.iterdir()) == sorted(opfm.stack_names(7, color=True))
    rd = lambda name: opfm.read_pfm(tmp_path / name)
    for m, s in enumerate(("_p0", "_p90", "_p180", "_p270")):
        assert np.array_equal(rd(f"quad_00007{s}.pfm")[0], out["quad"][m])
    depth = rd("depth_00007.pfm")[0]
    want = opfm.stack_depth(out["depth"], out["weight"])
    assert np.array_equal(np.isnan(depth), np.isnan(want))
    assert np.array_equal(depth[~np.isnan(depth)], want[~np.isnan(want)].astype(np.float32))
    assert 0 < np.isnan(depth).sum() < depth.size
    dtof = rd("dtof_00007.pfm")[0].astype(np.float64)
    wd = opfm.quad_to_depth(out["quad"][:4], 30e6)
    assert np.array_equal(np.isnan(dtof), np.isnan(wd))
    du = tsb.unambiguous_range(30e6)
    diff = np.abs(dtof - wd)[~np.isnan(wd)]
    diff = np.minimum(diff, du - diff)  # phase wrap at 0 / d_u
    assert diff.max() <= 1e-6 * du
    assert np.array_equal(rd("dd_00007.pfm")[0], out["distortion"])
    assert np.array_equal(rd("color_00007.pfm"), out["color"])
    # without the distortion channel the stack is refused (eval.cpp:104 renders it)
    rq = tsb.RenderPass(ctx).prepare(scene, cam, tsb.RenderOptions(), (0, 0.5)).forward()
    with pytest.raises(RuntimeError, match="distortion"):
        rq.write_render_stack(tmp_path / "x", 0)


def test_densify_carries_colour_and_sh(tsb, ctx):
    """Densification surgery (trainer.cpp:385-470) on a scene with reflectivity SH (degree 2)
    and colour SH: every appearance coefficient follows its parent (kept, cloned, split)."""
    from oracle import densify as odn
    from paper_2505_05356_b200 import synthetic
    g, sh, cs, _, _, scene, tof = _setup(tsb, ctx, 2, n=4000, seed=83)
    cam = synthetic.camera(128, 96, 110.0)
    rng = np.random.default_rng(84)
    target = rng.normal(0, 0.05, (4, 96, 128)).astype(np.float32)
    rp = tsb.RenderPass(ctx)
    for it in range(2):
        rp.prepare(scene, cam, tsb.RenderOptions(), (0, 0.4 * it)).forward_loss(target, sync=False)
        rp.backward()
        scene.adam_step(tsb.LrTable.uniform(1e-3))
    prm = scene.get_params()
    prm["refl_sh"] = scene.get_sh()
    prm["color_sh"] = scene.get_color()
    stat, count = scene.densify_stat()
    extent = tsb.render.scene_extent(prm["position"])
    thr = float(np.quantile(stat / count, 0.6))
    n_new = scene.densify(extent, grad_threshold=thr, split_scale_fraction=0.02, min_count=16)
    ref, src = odn.densify(prm, stat, count, extent, grad_threshold=thr, split_scale_fraction=0.02, min_count=16)
    assert n_new == ref["position"].shape[0] and any(s < 0 for s in src)
    assert np.array_equal(scene.get_color(), ref["color_sh"])
    got_sh = scene.get_sh()
    assert np.array_equal(got_sh[:, 1:], ref["refl_sh"][:, 1:])
    assert np.array_equal(got_sh[:, 0], ref["reflectivity_dc"])
    out = tsb.RenderPass(ctx).prepare(scene, cam, tsb.RenderOptions(color=True), (0, 0.5)).forward().outputs()
    assert np.isfinite(out["color"]).all()
