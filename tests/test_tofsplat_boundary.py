"""The reference's Python surface (`tofsplat`, proj/python/bindings.cpp:40-204) over the B200
path: the reference's own smoke cases (proj/tests/python/test_smoke.py:10-78) for the
functions on the render/optimise path, plus checkpoint / dataset parsing and render_timestep
against the oracle.  CPU tests need only the library's host code; the renders are -m gpu."""
import json
import math

import numpy as np
import pytest

import tofsplat
from oracle import pfm as opfm
from paper_2505_05356_b200 import core

HAS_GPU = __import__("os").path.exists("/dev/nvidia0")


# ---- test_smoke.py cases (host helpers) ----------------------------------------------------
def test_unambiguous_range():
    assert tofsplat.unambiguous_range() == pytest.approx(5.0, abs=1e-12)
    assert tofsplat.unambiguous_range(2 * 29.9792458e6) == pytest.approx(2.5, abs=1e-12)


def test_quad_round_trip():
    depth = 1.7
    basis = tofsplat.quad_basis(depth)
    assert len(basis) == 4
    quad = [0.6 * b + 0.2 for b in basis]  # amplitude scaling and a shared offset must not change the decode
    assert tofsplat.quad_to_depth(*quad) == pytest.approx(depth, abs=1e-12)


def test_flat_quartet_is_invalid():
    assert math.isnan(tofsplat.quad_to_depth(0.3, 0.3, 0.3, 0.3))


def test_out_of_path_functions_are_explicit_errors():
    for f in (tofsplat.builtin_scene_names, tofsplat.simulate_dataset, tofsplat.fit_dataset, tofsplat.evaluate):
        with pytest.raises(core.TsbError, match="outside the B200 render/optimise path"):
            f("x", "y")


# ---- generator and file formats --------------------------------------------------------------
def test_mt19937_64_known_answer():
    """C++11 [rand.predef]: the 10000th output of a default-constructed mt19937_64."""
    r = core.MT19937_64(5489)
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042
    u = core.MT19937_64(7).uniform(-1.0, 1.0)
    assert -1.0 <= u < 1.0


def _scene_ckpt(n, seed, sh_degree=1):
    rng = np.random.default_rng(seed)
    refl = np.zeros((n, 16), np.float32)
    refl[:, 0] = rng.uniform(0.3, 0.7, n) / core.SH_C0
    refl[:, 1:4] = rng.uniform(-0.05, 0.05, (n, 3))
    col = np.zeros((n, 16, 3), np.float32)
    col[:, 0] = 0.5 / core.SH_C0
    pos = np.stack([rng.uniform(-0.5, 0.5, n), rng.uniform(-0.4, 0.4, n), rng.uniform(1.5, 4.0, n)], 1)
    q = rng.normal(size=(n, 4))
    return core.SceneCheckpoint(pos.astype(np.float32), np.log(rng.uniform(0.03, 0.12, (n, 3))).astype(np.float32),
                                q.astype(np.float32), rng.normal(0.5, 1.0, n).astype(np.float32), refl, col,
                                sh_degree, core.ToFConfig(29.9792458e6), (0.1, 0.0, -0.1, 0.0), (0.2, 0.3, 0.4))


def test_scene_checkpoint_round_trip(tmp_path):
    sc = _scene_ckpt(37, 3)
    p = tmp_path / "scene.ckpt"
    core.save_scene(p, sc)
    head = p.read_bytes()[:200].decode(errors="replace")
    assert head.startswith("tofsplat_scene 1\ngaussians 37\nsh_degree 1\n")
    back = core.load_scene(p)
    for k in ("position", "log_scale", "rotation", "opacity_logit", "reflectivity_sh", "color_sh"):
        assert np.array_equal(getattr(back, k), getattr(sc, k)), k
    assert back.sh_degree == 1 and back.tof.modulation_frequency == sc.tof.modulation_frequency
    assert back.bg_quad == sc.bg_quad and back.bg_color == sc.bg_color
    assert p.stat().st_size == len(head.split("data\n")[0]) + 5 + 37 * 75 * 4
    p.write_bytes(p.read_bytes()[:-4])
    with pytest.raises(core.TsbError, match="truncated parameter block"):
        core.load_scene(p)
    (tmp_path / "bad.ckpt").write_bytes(b"tofsplat_scene 2\n")
    with pytest.raises(core.TsbError, match="bad header"):
        core.load_scene(tmp_path / "bad.ckpt")


def _deform_ckpt(seed=1):
    from oracle import deform as odf
    cfg = odf.DeformConfig(hidden_layers=1, width=16, l_x=4, l_t=4, coord_scale=1.0, final_std=0.05)
    net = odf.DeformNet.init(cfg, seed)
    flat = net.get_parameters().astype(np.float32)
    net.set_parameters(flat.astype(np.float64))  # the checkpoint stores float32 (deform.cpp:203-207)
    return net, core.DeformCheckpoint(1, 16, 4, 4, 1.0, flat)


def test_deform_checkpoint_round_trip(tmp_path):
    net, ck = _deform_ckpt()
    p = tmp_path / "deform.ckpt"
    core.save_deform(p, ck)
    back = core.load_deform(p)
    assert (back.hidden_layers, back.width, back.l_x, back.l_t) == (1, 16, 4, 4)
    assert back.parameter_count() == net.parameter_count == ck.parameters.size
    assert np.array_equal(back.parameters, ck.parameters)
    txt = p.read_bytes()
    p.write_bytes(txt.replace(b"width 16", b"widht 16"))
    with pytest.raises(core.TsbError, match="unknown field 'widht'"):
        core.load_deform(p)


def _dataset(tmp_path, w=16, h=12, frames=8, fps=120.0, flow=True):
    root = tmp_path / "ds"
    root.mkdir()
    fr = []
    for k in range(frames):
        name = f"raw_{k:05d}.pfm"
        opfm.write_pfm(root / name, np.full((1, h, w), 0.01 * k, np.float32))
        fr.append({"file": name, "time": k / fps, "phase_index": k % 4})
    m = {"format": "tofsplat_dataset", "tof": {"modulation_frequency": 29.9792458e6},
         "camera": {"fx": 0.9 * w, "fy": 0.9 * w, "cx": w / 2, "cy": h / 2, "width": w, "height": h},
         "raw_fps": fps, "frames": fr}
    if flow:
        m["flow_fwd"] = [{"time": 4 * q / fps, "file": "flow.pfm"} for q in range(frames // 4)]
    (root / "manifest.json").write_text(json.dumps(m))
    return root, m


def test_dataset_info_and_validation(tmp_path):
    root, m = _dataset(tmp_path)
    info = tofsplat.dataset_info(str(root))
    assert info["num_frames"] == 8 and info["num_quartets"] == 2
    assert info["width"] == 16 and info["height"] == 12 and info["has_flow"] and not info["has_color"]
    m["frames"][1]["phase_index"] = 2
    (root / "manifest.json").write_text(json.dumps(m))
    with pytest.raises(core.TsbError, match="quartet ordering"):
        tofsplat.dataset_info(str(root))
    m["frames"][1]["phase_index"] = 1
    m["frames"][2]["time"] = 0.5
    (root / "manifest.json").write_text(json.dumps(m))
    with pytest.raises(core.TsbError, match="off the raw cadence"):
        tofsplat.dataset_info(str(root))


# ---- GPU: renders ----------------------------------------------------------------------------
@pytest.mark.gpu
def test_gradcheck_small():
    """test_smoke.py:48-51."""
    r = tofsplat.gradcheck(seed=7, splats=2, width=6, height=6)
    assert r["max_rel_err"] < 1e-3, r
    assert r["groups"]


@pytest.mark.gpu
def test_gradcheck_default_setup():
    """run_gradcheck's defaults (seed 7, 4 splats, 8 x 8; gradcheck.hpp:27) -- every group the
    reference checks except the DeformNet weights (reported as skipped)."""
    r = tofsplat.gradcheck()
    assert r["max_rel_err"] < 1e-3, r
    assert set(r["groups"]) == {"position", "log_scale", "rotation", "opacity", "reflectivity_sh", "color_sh",
                                "motion_fwd", "motion_bwd", "bg_color", "bg_quad", "bg_phasor"}


@pytest.mark.gpu
@pytest.mark.parametrize("timestep", [0.0, 0.5, 1.0])
def test_render_timestep_matches_oracle(tmp_path, timestep):
    """bindings.cpp:164-203: deformed means interpolated between quartet times, rendered with
    the dataset camera; shapes as test_smoke.py:70-78, values vs the oracle render of the
    oracle-deformed positions (1e-4 relative under a 1e-6*max floor)."""
    from oracle import deform as odf
    from oracle import oracle as orc
    from helpers import rel_err_quantile
    root, _ = _dataset(tmp_path)
    sc = _scene_ckpt(300, 9)
    net, ck = _deform_ckpt(2)
    core.save_scene(tmp_path / "scene.ckpt", sc)
    core.save_deform(tmp_path / "deform.ckpt", ck)
    frame = tofsplat.render_timestep(str(tmp_path / "scene.ckpt"), str(tmp_path / "deform.ckpt"), str(root),
                                     timestep)
    quad = np.asarray(frame["quad"])
    assert quad.shape == (12, 16, 4) and np.isfinite(quad).all()
    weight = np.asarray(frame["weight"])
    assert weight.shape == (12, 16, 1) and (weight >= 0).all() and (weight <= 1 + 1e-9).all()
    assert np.asarray(frame["depth"]).shape == (12, 16, 1)
    # oracle: canonical + net(canonical, t) at the two quartet times, interp_positions
    can = sc.position.astype(np.float64)
    nq = 2
    i1 = math.floor(timestep)
    x1 = can + net.offsets(can, core.quartet_time(i1, nq)).astype(np.float32).astype(np.float64)
    pos = x1
    if timestep != i1:
        x2 = can + net.offsets(can, core.quartet_time(i1 + 1, nq)).astype(np.float32).astype(np.float64)
        pos = odf.interp_positions(x1, x2, i1, i1 + 1.0, timestep)
    osc = orc.OScene(pos, sc.log_scale.astype(np.float64), sc.rotation.astype(np.float64),
                     sc.opacity_logit.astype(np.float64), sc.reflectivity_sh.astype(np.float64), sc.sh_degree,
                     sc.tof.modulation_frequency, sc.tof.source_intensity, sc.tof.speed_of_light)
    cam = core.load_dataset_info(root).camera
    ref = orc.OraclePass(osc, cam, type("O", (), {})()).forward()
    assert rel_err_quantile(quad.transpose(2, 0, 1), ref["quad"], 1e-6, 1.0) < 1e-4
    assert rel_err_quantile(weight[..., 0], ref["weight"], 1e-6, 1.0) < 1e-4


@pytest.mark.gpu
def test_render_timestep_without_deformation(tmp_path):
    root, _ = _dataset(tmp_path)
    sc = _scene_ckpt(200, 4, sh_degree=0)
    core.save_scene(tmp_path / "scene.ckpt", sc)
    frame = tofsplat.render_timestep(str(tmp_path / "scene.ckpt"), "", str(root), 0.0)
    assert frame["quad"].shape == (12, 16, 4) and np.isfinite(frame["quad"]).all()
    assert (frame["weight"] > 0).any()
