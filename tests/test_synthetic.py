"""Seeded synthetic BASELINE configs are deterministic and follow the stated distributions."""
import numpy as np
import pytest

from paper_2505_05356_b200 import synthetic
from paper_2505_05356_b200.render import SH_C0, frame_for_time


def test_deterministic():
    a = synthetic.config("c1", n=5000)
    b = synthetic.config("c1", n=5000)
    for k in ("position", "log_scale", "rotation", "opacity_logit", "reflectivity_dc"):
        assert np.array_equal(getattr(a.scene, k), getattr(b.scene, k))
    assert np.array_equal(a.scene.motion, b.scene.motion)
    assert not np.array_equal(a.scene.position, a.target.position)


def test_c0_distributions():
    g = synthetic.config("c0").scene
    assert g.n == 20_000 and g.position.dtype == np.float32
    assert g.position[:, :2].min() >= -1 and g.position[:, :2].max() <= 1
    assert g.position[:, 2].min() >= 1 and g.position[:, 2].max() <= 5
    assert abs(g.log_scale.mean() + 3) < 0.02 and abs(g.log_scale.std() - 0.3) < 0.01
    assert np.allclose(np.linalg.norm(g.rotation, axis=1), 1, atol=1e-6)
    amp = g.reflectivity_dc * SH_C0
    assert abs(np.log(amp).mean() + 1) < 0.02


def test_c3_depths_and_frames():
    cfg = synthetic.config("c3", n=10_000)
    z = cfg.scene.position[:, 2]
    assert z.min() >= 0.5 and z.max() <= 8
    assert len(cfg.frames) == 300 and cfg.frames[0] == (0, 0.0) and cfg.frames[-1] == (0, 1.0)


@pytest.mark.parametrize("t,nk,want", [(0.0, 2, (0, 0.0)), (0.5, 2, (0, 0.5)), (1.0, 2, (0, 1.0)),
                                       (0.3, 9, (2, 0.3 * 8 - 2)), (1.0, 9, (7, 1.0))])
def test_frame_for_time(t, nk, want):
    k, w = frame_for_time(t, nk)
    assert k == want[0] and w == pytest.approx(want[1])


def test_rendered_means_follow_trainer_lerp():
    g = synthetic.gaussians(100, 3, n_keyframes=2)
    x = g.position.astype(np.float64)
    m = g.rendered_means((0, 0.25))
    want = 0.75 * (x + g.motion[0]) + 0.25 * (x + g.motion[1])
    assert np.allclose(m, want, rtol=0, atol=1e-12)
    assert np.array_equal(g.rendered_means((0, 0.0)), x + g.motion[0].astype(np.float64))
