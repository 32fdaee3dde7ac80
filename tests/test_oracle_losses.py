"""The image-loss oracle pinned to the reference's own tests (tests/unit/test_losses.cpp)."""
import math

import numpy as np

from oracle import losses as ol


def rand_img(w, h, c, seed):
    return np.random.default_rng(seed).uniform(0, 1, (c, h, w))


def test_window_is_normalised_gaussian():
    w = ol.window1d()
    assert w.size == 11 and abs(w.sum() - 1) < 1e-15 and np.argmax(w) == 5 and np.allclose(w, w[::-1])


def test_ssim_of_identical_images_is_one():
    """test_losses.cpp:39-44."""
    a = rand_img(16, 12, 3, 5)
    assert abs(ol.ssim(a, a) - 1.0) < 1e-12
    assert ol.ssim(a, rand_img(16, 12, 3, 6)) < 1.0


def test_ssim_gradient_matches_finite_differences():
    """test_losses.cpp:46-62."""
    pred, target = rand_img(8, 8, 1, 7), rand_img(8, 8, 1, 8)
    _, g = ol.ssim(pred, target, True)
    h = 1e-6
    for i in range(pred.size):
        p = pred.copy().ravel()
        p[i] += h
        fp = ol.ssim(p.reshape(pred.shape), target)
        p[i] -= 2 * h
        fm = ol.ssim(p.reshape(pred.shape), target)
        fd = (fp - fm) / (2 * h)
        assert abs(g.ravel()[i] - fd) <= 1e-4 * max(abs(fd), 0.01)


def test_image_loss_blends_mse_and_ssim():
    """test_losses.cpp:64-87."""
    a, b = rand_img(12, 9, 2, 9), rand_img(12, 9, 2, 10)
    assert abs(ol.image_loss(a, a, 0.2)) < 1e-12
    assert np.isclose(ol.image_loss(a, b, 0.0), ol.mse(a, b), rtol=1e-12)
    assert np.isclose(ol.image_loss(a, b, 1.0), 1.0 - ol.ssim(a, b), rtol=1e-12)
    assert np.isclose(ol.image_loss(a, b, 0.2), 0.8 * ol.mse(a, b) + 0.2 * (1.0 - ol.ssim(a, b)), rtol=1e-12)
    pred, target = rand_img(8, 8, 1, 11), rand_img(8, 8, 1, 12)
    _, g = ol.image_loss(pred, target, 0.2, True)
    h = 1e-6
    for i in range(0, pred.size, 7):
        p = pred.copy().ravel()
        p[i] += h
        fp = ol.image_loss(p.reshape(pred.shape), target, 0.2)
        p[i] -= 2 * h
        fm = ol.image_loss(p.reshape(pred.shape), target, 0.2)
        fd = (fp - fm) / (2 * h)
        assert abs(g.ravel()[i] - fd) <= 1e-4 * max(abs(fd), 0.01)


# ---- flow loss (losses.cpp:168-251), pinned to test_losses.cpp:162-296 ----
class _Cam:
    def __init__(self, fx, fy, cx, cy, w, h, R=None, t=None):
        self.fx, self.fy, self.cx, self.cy, self.width, self.height = fx, fy, cx, cy, w, h
        self.near_plane, self.far_plane = 0.2, 100.0
        self.rotation = np.eye(3) if R is None else R
        self.translation = np.zeros(3) if t is None else t


class _Opts:
    alpha_threshold, transmittance_floor, dilation, sigma_cutoff = 1.0 / 255.0, 1e-4, 0.3, 3.0
    coverage_eps, tile_size = 1e-12, 16
    bg_quad, bg_phasor = np.zeros(4), np.zeros(2)


def _flow_render(cam, cam_space=False):
    """test_losses.cpp:134-158 (flow_render) through the C oracle: two splats with motions."""
    from oracle import oracle as orc
    pos = np.array([[0.1, -0.05, 2.0], [-0.2, 0.1, 3.0]])
    if cam_space:  # cam.to_world: R^T (p - t)
        pos = (pos - cam.translation) @ cam.rotation
    refl = np.zeros((2, 16))
    refl[:, 0] = 0.5 / 0.28209479177387814
    sc = orc.OScene(pos, np.full((2, 3), np.log(0.3)), np.tile([1.0, 0, 0, 0], (2, 1)), np.full(2, 1.5), refl, 0,
                    29.9792458e6, 1.0, 299792458.0)
    # Eigen's comma initialiser fills the 3x2 matrices row by row; column i = Gaussian i
    sc.motion_fwd = np.array([[0.05, -0.1], [-0.02, 0.04], [0.2, 0.1]]).T.copy()
    sc.motion_bwd = np.array([[-0.05, 0.02], [0.01, -0.03], [0.1, -0.2]]).T.copy()
    op = orc.OraclePass(sc, cam, _Opts())
    buf = dict(op.forward())
    buf.update(op.forward_ext())
    return buf


def _flow_objective(buf, cam, macc, target, valid_ch):
    """test_losses.cpp:109-131: the flow MSE recomputed from the accumulators."""
    H, W = buf["depth"].shape
    fx, fy, cx, cy = cam.fx, cam.fy, cam.cx, cam.cy
    R, t = cam.rotation, cam.translation
    sse, count = 0.0, 0
    for y in range(H):
        for x in range(W):
            if not (target[2, y, x] > 0.5 and buf["flow_valid"][valid_ch, y, x] > 0.5):
                continue
            xd = ol.backproject(cam, np.array(x + 0.5), np.array(y + 0.5), np.array(buf["depth"][y, x]))
            p = R @ (xd + macc[:, y, x]) + t
            ru = fx * p[0] / p[2] + cx - (x + 0.5) - target[0, y, x]
            rv = fy * p[1] / p[2] + cy - (y + 0.5) - target[1, y, x]
            sse += ru * ru + rv * rv
            count += 1
    return sse / count if count else 0.0


def test_flow_loss_values_and_masking():
    """test_losses.cpp:162-217."""
    cam = _Cam(30.0, 30.0, 16.5, 12.5, 32, 24)
    buf = _flow_render(cam)
    H, W = 24, 32
    tf = np.zeros((3, H, W))
    tb = np.zeros((3, H, W))
    tf[:2], tb[:2] = buf["flow_fwd"], buf["flow_bwd"]
    tf[2] = tb[2] = 1.0
    eq = ol.flow_loss(buf, cam, tf, tb)
    assert abs(eq["value"]) <= 1e-15 and eq["valid_pixels"] > 0
    t3 = tf.copy()
    t3[0] += 3.0
    nine = ol.flow_loss(buf, cam, t3, None)
    assert abs(nine["value"] - 9.0) <= 9.0 * 1e-12 and nine["d_motion_bwd_acc"] is None
    bwd_only = ol.flow_loss(buf, cam, None, tb)
    assert abs(bwd_only["value"]) <= 1e-15
    assert bwd_only["d_motion_fwd_acc"] is None and bwd_only["d_motion_bwd_acc"] is not None
    none = tf.copy()
    none[2] = 0.0
    zero = ol.flow_loss(buf, cam, none, None)
    assert zero["value"] == 0.0 and zero["valid_pixels"] == 0 and zero["d_motion_fwd_acc"] is None
    assert ol.flow_loss(buf, cam, None, None)["value"] == 0.0


def test_flow_loss_gradient_matches_finite_differences():
    """test_losses.cpp:219-296: rotated / translated camera, patchy validity; the gradient on
    the motion accumulators equals the FD of the direction-averaged objective."""
    axis = np.array([0.1, 1.0, -0.3])
    axis /= np.linalg.norm(axis)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    R = np.eye(3) + math.sin(0.2) * K + (1 - math.cos(0.2)) * K @ K  # AngleAxisd(0.2, axis)
    cam = _Cam(28.0, 31.0, 16.1, 12.3, 32, 24, R, np.array([0.05, -0.1, 0.2]))
    buf = _flow_render(cam, cam_space=True)
    H, W = 24, 32
    rng = np.random.default_rng(19)
    tf = np.stack([rng.uniform(-0.5, 0.5, (H, W)), rng.uniform(-0.5, 0.5, (H, W)),
                   (rng.uniform(-0.5, 0.5, (H, W)) > 0).astype(float)])
    tb = np.stack([rng.uniform(-0.5, 0.5, (H, W)), rng.uniform(-0.5, 0.5, (H, W)), np.ones((H, W))])
    res = ol.flow_loss(buf, cam, tf, tb)
    assert res["valid_pixels"] > 0 and res["d_motion_fwd_acc"] is not None
    h = 1e-6
    checked = 0
    for y in range(H):
        for x in range(W):
            if checked >= 40:
                break
            if not buf["flow_valid"][0, y, x] > 0.5:
                continue
            for c in range(3):
                macc = buf["motion_fwd_acc"].copy()
                macc[c, y, x] += h
                fp = _flow_objective(buf, cam, macc, tf, 0)
                macc[c, y, x] -= 2 * h
                fm = _flow_objective(buf, cam, macc, tf, 0)
                fd = 0.5 * (fp - fm) / (2 * h)
                assert abs(res["d_motion_fwd_acc"][c, y, x] - fd) <= 1e-5 * max(abs(fd), 1e-3)
            checked += 1
    assert checked > 5
