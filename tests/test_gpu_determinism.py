"""Deterministic mode (TSB_CH_DETERMINISTIC): the reference reduces its per-thread gradient
arrays in a fixed order (splat.cpp:521-543), so its fits are bit-identical run to run
(test_trainer.cpp:199-217, acceptance.cpp:453-486).  The default B200 backward adds
per-block sums with float atomics (order-dependent in the last bits); the deterministic
mode writes per-(rank, tile, sub-block) slots and reduces them per Gaussian in a fixed order.
Checked: repeated training steps give bit-identical gradients, loss and parameters, and the
gradients still match the oracle."""
import numpy as np
import pytest

from oracle import oracle as orc

from helpers import gpu_scene, oracle_scene, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tsb():
    import paper_2505_05356_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(tsb):
    return tsb.Context(0)


def _iteration(tsb, ctx, cfg, target, opts, passes=3, frames=None):
    scene = gpu_scene(tsb, ctx, cfg.scene, cfg.tof)
    rps = [tsb.RenderPass(ctx) for _ in range(passes)]
    frames = frames or cfg.frames
    for i, fr in enumerate(frames):
        rp = rps[i % passes]
        rp.prepare(scene, cfg.camera, opts, fr)
        rp.forward_loss(target, sync=False)
        rp.backward()
    g = scene.grads()
    scene.adam_step(tsb.LrTable.uniform(1e-3))
    p = scene.get_params()
    for rp in rps:
        rp.close()
    scene.close()
    return g, p


def test_deterministic_training_step_is_bit_identical(tsb, ctx):
    from paper_2505_05356_b200 import synthetic
    cfg = synthetic.config("c1", n=60_000)
    frames = [(0, 0.2), (0, 0.5), (0, 0.8)]
    rng = np.random.default_rng(4)
    target = rng.normal(0, 0.02, (4, cfg.camera.height, cfg.camera.width)).astype(np.float32)
    det = tsb.RenderOptions(deterministic=True)
    runs = [_iteration(tsb, ctx, cfg, target, det, frames=frames) for _ in range(3)]
    g0, p0 = runs[0]
    assert np.abs(g0["d_position"]).max() > 0
    for g, p in runs[1:]:
        for k in g0:
            assert np.array_equal(np.asarray(g0[k]), np.asarray(g[k])), k
        for k in p0:
            assert np.array_equal(p0[k], p[k]), k
    # the default (atomic) mode agrees to summation order; the oracle to the 1e-3 bar
    ga, _ = _iteration(tsb, ctx, cfg, target, tsb.RenderOptions(), frames=frames)
    assert rel_err(ga["d_position"], g0["d_position"], 1e-4) < 1e-4
    want = np.zeros_like(g0["d_position"], dtype=np.float64)
    for fr in frames:
        op = orc.OraclePass(oracle_scene(cfg.scene, fr, cfg.tof), cfg.camera, tsb.RenderOptions())
        ref = op.forward()
        dq = np.zeros((4,) + target.shape[1:])
        for m in range(4):
            _, d = orc.mse(ref["quad"][m], target[m].astype(np.float64))
            dq[m] = 0.25 * d
        want += op.backward(d_quad=dq)["d_position"]
    assert rel_err(g0["d_position"], want, 1e-4) < 1e-3


def test_deterministic_mode_with_recomposited_pixels(tsb, ctx):
    """Opaque splats force fp64 recomposition (fix-up reasons 4 / 8): their fp64 backward must
    also be reproducible (one warp per raster block, pixel order, private slots)."""
    from paper_2505_05356_b200 import synthetic
    g = synthetic.gaussians(20_000, 44, n_keyframes=2)
    g.opacity_logit[::40] = 8.0
    cfg = synthetic.Config("det", g, synthetic.camera(320, 240, 262.5), tsb.ToFConfig(30e6), [(0, 0.3), (0, 0.6)])
    rng = np.random.default_rng(5)
    target = rng.normal(0, 0.02, (4, 240, 320)).astype(np.float32)
    det = tsb.RenderOptions(deterministic=True)
    (a, pa), (b, pb) = [_iteration(tsb, ctx, cfg, target, det, passes=2) for _ in range(2)]
    for k in a:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
    scene = gpu_scene(tsb, ctx, g, cfg.tof)
    rp = tsb.RenderPass(ctx).prepare(scene, cfg.camera, det, (0, 0.3)).forward()
    assert rp.debug_fixups() > 0


def test_upload_to_one_scene_while_another_renders(tsb, ctx):
    """tsb_scene_set_params waits only for the frames reading its own scene: uploading scene
    B while frames of scene A are still queued leaves A's frames intact, and B's frames see
    B's new parameters (each compared with a synchronous render of the same frame)."""
    from paper_2505_05356_b200 import synthetic
    cfg = synthetic.config("c1", n=30_000)
    ga, gb = synthetic.gaussians(30_000, 3, n_keyframes=2), synthetic.gaussians(30_000, 4, n_keyframes=2)
    sa, sb = gpu_scene(tsb, ctx, ga, cfg.tof), gpu_scene(tsb, ctx, ga, cfg.tof)
    cam, opts = cfg.camera, tsb.RenderOptions()
    H, W = cam.height, cam.width
    frames = [(0, 0.1 * i) for i in range(6)]
    rps = [tsb.RenderPass(ctx) for _ in range(4)]
    bufs = [np.zeros(4 * H * W, np.float32) for _ in range(12)]
    for i, fr in enumerate(frames):  # scene A, queued
        rp = rps[i % 4]
        rp.prepare(sa, cam, opts, fr).forward()
        rp.download_async(tsb._abi.OUT_QUAD, bufs[i])
        if i == 3:  # scene B's upload while A's frames are in flight
            sb.set_params(gb.position, gb.log_scale, gb.rotation, gb.opacity_logit, gb.reflectivity_dc, gb.motion)
    for i, fr in enumerate(frames):  # scene B
        rp = rps[(i + 2) % 4]
        rp.prepare(sb, cam, opts, fr).forward()
        rp.download_async(tsb._abi.OUT_QUAD, bufs[6 + i])
    for rp in rps:
        rp.wait()
    ref = tsb.RenderPass(ctx)
    for k, (sc, base) in enumerate(((sa, 0), (sb, 6))):
        for i, fr in enumerate(frames):
            ref.prepare(sc, cam, opts, fr).forward()
            want = ref.download(tsb._abi.OUT_QUAD)
            assert np.array_equal(bufs[base + i], want), (k, i)
    # and B really holds gb (not A's parameters)
    assert np.array_equal(sb.get_params()["position"], gb.position.astype(np.float32))
