"""Densification oracle pinned to the reference's trainer tests (test_trainer.cpp:51-70, 232-255)."""
import numpy as np

from oracle import densify as od
from oracle import oracle as orc


def _params(n, seed):
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(n, 4))
    return {"position": rng.uniform(-1, 1, (n, 3)).astype(np.float32),
            "log_scale": rng.normal(-3, 0.3, (n, 3)).astype(np.float32),
            "rotation": (q / np.linalg.norm(q, axis=1, keepdims=True)).astype(np.float32),
            "opacity_logit": rng.normal(0, 1, n).astype(np.float32),
            "reflectivity_dc": rng.uniform(0, 1, n).astype(np.float32),
            "motion": rng.normal(0, 0.05, (2, n, 3)).astype(np.float32)}


def test_threshold_zero_grows_and_high_floor_prunes_to_min_count():
    """test_trainer.cpp:232-255: threshold 0 -> every survivor clones or splits; floor 0.999 ->
    pruning stops at min_count."""
    p = _params(24, 1)
    g = np.ones(24)
    grown, src = od.densify(p, g, 1, 1.0, grad_threshold=0.0, min_count=16)
    assert grown["position"].shape[0] > 24 and len(src) == grown["position"].shape[0]
    pruned, _ = od.densify(p, np.zeros(24), 1, 1.0, grad_threshold=1e9, opacity_floor=0.999, min_count=16)
    assert pruned["position"].shape[0] == 16


def test_split_children_straddle_the_parent_along_its_largest_axis():
    p = _params(1, 2)
    p["log_scale"][0] = [np.log(0.3), np.log(0.1), np.log(0.05)]
    out, src = od.densify(p, [1.0], 1, 1.0, grad_threshold=0.0, split_scale_fraction=0.01, min_count=0)
    assert src == [-1, -1]
    mid = out["position"].astype(np.float64).mean(axis=0)
    assert np.allclose(mid, p["position"][0], atol=1e-6)
    R = od.quat_to_rotation(p["rotation"][0])
    d = out["position"][1].astype(np.float64) - out["position"][0]
    assert np.allclose(d, 2 * 0.25 * 0.3 * R[:, 0], atol=1e-6)
    assert np.allclose(out["log_scale"][0], p["log_scale"][0] - np.log(1.6), atol=1e-6)


def test_adam_reindex_copies_and_clears_moments():
    """test_trainer.cpp:51-70 (keep 1, clone 1, fresh slot), on the oracle Adam."""
    p = np.zeros(4)
    g = np.array([1.0, 2.0, 3.0, 4.0])
    m, v = np.zeros(4), np.zeros(4)
    orc.adam_step(p, g, m, v, 1, 0.1)
    m2, v2 = od.adam_reindex(m.reshape(2, 2), v.reshape(2, 2), [1, 1, -1])
    p2 = np.zeros(6)
    m2, v2 = m2.ravel().copy(), v2.ravel().copy()
    orc.adam_step(p2, np.zeros(6), m2, v2, 2, 0.1)
    assert p2[0] == p2[2] and p2[1] == p2[3] and p2[0] != 0.0
    assert p2[4] == 0.0 and p2[5] == 0.0
