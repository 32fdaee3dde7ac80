"""Shared test helpers: run the same seeded input through the B200 path (C ABI)
and through the CPU oracle, and compare with the tolerances of SURVEY.md App. D."""
from __future__ import annotations

import numpy as np

from oracle import oracle as orc


def rel_err(a, b, floor_frac=1e-6):
    """max |a-b| / max(|a|, |b|, floor), floor = floor_frac * max|b| (gradcheck.cpp:122-125 style)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    mask = np.isfinite(b)
    assert np.array_equal(mask, np.isfinite(a)), "NaN pattern differs"
    if not mask.any():
        return 0.0
    a, b = a[mask], b[mask]
    floor = max(floor_frac * np.abs(b).max(), 1e-300)
    return float((np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)).max())


def rel_err_quantile(a, b, floor_frac=1e-6, q=0.9999):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    mask = np.isfinite(b)
    if not mask.any():
        return 0.0
    a, b = a[mask], b[mask]
    floor = max(floor_frac * np.abs(b).max(), 1e-300)
    return float(np.quantile(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor), q))


def oracle_scene(gset, frame, tof, freq_index=0):
    f = tof.frequencies[freq_index]
    return orc.scene_from_dc(gset.rendered_means(frame), gset.log_scale, gset.rotation, gset.opacity_logit,
                             gset.reflectivity_dc, frequency=f, source_intensity=tof.source_intensity,
                             speed_of_light=tof.speed_of_light)


def gpu_scene(tsb, ctx, gset, tof):
    s = tsb.GaussianScene(ctx, gset.n, gset.n_keyframes, tof)
    s.set_params(gset.position, gset.log_scale, gset.rotation, gset.opacity_logit, gset.reflectivity_dc,
                 gset.motion)
    return s


def oracle_sorted_lists(op):
    off, ids = op.tile_lists()
    return off, ids


# SURVEY App. D figures recorded by the parity tests (written by conftest at session end
# to $TSB_PARITY_REPORT when set): per test and quantity, the max and 99.99th-percentile
# relative error under the App. D floor (1e-6 * max|oracle| for images, 1e-4 * max for
# gradient groups).
REPORT = {}


def app_d(a, b, floor_frac=1e-6):
    return {"max": rel_err(a, b, floor_frac), "p9999": rel_err_quantile(a, b, floor_frac, 0.9999),
            "floor": floor_frac}


def record(test: str, quantity: str, stats) -> None:
    REPORT.setdefault(test, {})[quantity] = stats
