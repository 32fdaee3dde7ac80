"""GPU diagnostic (round 2): gradient error per group and upstream channel for the posed
camera case, and the worst pixels of the gradcheck-options forward.  Prints only."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2505_05356_b200 as tsb  # noqa: E402
from paper_2505_05356_b200 import synthetic  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from helpers import app_d, gpu_scene, oracle_scene  # noqa: E402
from test_gpu_parity_shapes import rotation_matrix  # noqa: E402

ctx = tsb.Context(0)


def case(name, g, cam, opts, frame, tof, chans, seed=31):
    scene = gpu_scene(tsb, ctx, g, tof)
    rp = tsb.RenderPass(ctx).prepare(scene, cam, opts, frame).forward()
    out = rp.outputs()
    op = orc.OraclePass(oracle_scene(g, frame, tof), cam, opts)
    ref = op.forward()
    H, W = cam.height, cam.width
    rng = np.random.default_rng(seed)
    shapes = {"d_quad": (4, H, W), "d_phasor": (2, H, W)}
    ups = {c: rng.normal(0, 1e-3, shapes.get(c, (H, W))).astype(np.float32) for c in chans}
    rp.backward_buffers(**ups)
    gr = scene.grads()
    og = op.backward(**{k: v.astype(np.float64) for k, v in ups.items()})
    res = {}
    for nm, a, b in (("pos", gr["d_position"], og["d_position"]), ("ls", gr["d_log_scale"], og["d_log_scale"]),
                     ("rot", gr["d_rotation"], og["d_rotation"]), ("op", gr["d_opacity_logit"], og["d_opacity_logit"]),
                     ("refl", gr["d_reflectivity_dc"], og["d_refl_sh"][:, 0])):
        st = app_d(a, b, 1e-4)
        res[nm] = f"{st['max']:.2e}/{st['p9999']:.2e}"
    print(name, "+".join(c[2:] for c in chans), res, "fixups", rp.debug_fixups(), flush=True)
    scene.close()
    rp.close()
    return out, ref


cfg = synthetic.config("c1")
posed = synthetic.camera(640, 480, 525.0)
posed.rotation = rotation_matrix((0.3, -0.8, 0.2), 0.12)
posed.translation = np.array([0.15, -0.1, 0.4])
tpose = synthetic.camera(640, 480, 525.0)
tpose.translation = np.array([0.15, -0.1, 0.4])
rpose = synthetic.camera(640, 480, 525.0)
rpose.rotation = rotation_matrix((0.3, -0.8, 0.2), 0.12)
bg = dict(bg_quad=(0.01, -0.02, 0.015, 0.005), bg_phasor=(0.02, -0.01))
for cname, cam in (("identity", cfg.camera), ("posed", posed), ("t_only", tpose), ("R_only", rpose)):
    for chans in (("d_quad",), ("d_depth_raw",), ("d_weight",), ("d_transmittance",), ("d_phasor",)):
        case(cname, cfg.scene, cam, tsb.RenderOptions(counts=True, **bg), cfg.frames[0], cfg.tof, chans)
    case(cname + "_nobg", cfg.scene, cam, tsb.RenderOptions(counts=True), cfg.frames[0], cfg.tof, ("d_quad",))

# gradcheck options forward
g = synthetic.gaussians(20_000, 41, n_keyframes=2)
g.opacity_logit[::50] = 40.0
g.log_scale[::50] += np.float32(0.7)
cam = synthetic.camera(320, 240, 262.5)
for variant, kw in (("full", dict(alpha_threshold=0.0, transmittance_floor=0.0, sigma_cutoff=6.0)),
                    ("floor_only", dict(transmittance_floor=0.0)),
                    ("sigma6_only", dict(sigma_cutoff=6.0)),
                    ("alpha0_only", dict(alpha_threshold=0.0))):
    opts = tsb.RenderOptions(counts=True, **kw)
    scene = gpu_scene(tsb, ctx, g, tsb.ToFConfig(30e6))
    rp = tsb.RenderPass(ctx).prepare(scene, cam, opts, (0, 0.3)).forward()
    out = rp.outputs()
    op = orc.OraclePass(oracle_scene(g, (0, 0.3), tsb.ToFConfig(30e6)), cam, opts)
    ref = op.forward()
    q, rq = out["quad"].astype(np.float64), ref["quad"]
    fl = 1e-6 * np.abs(rq).max()
    rel = np.abs(q - rq) / np.maximum(np.maximum(np.abs(q), np.abs(rq)), fl)
    st = app_d(q, rq)
    idx = np.unravel_index(np.argsort(rel.ravel())[-5:], rel.shape)
    print("gradcheck-opts", variant, st, "counts equal", np.array_equal(out["n_contrib"], ref["n_contrib"]),
          "fixups", rp.debug_fixups(), flush=True)
    for c, y, x in zip(*idx):
        print("   worst", c, y, x, "gpu", q[c, y, x], "ref", rq[c, y, x], "nc", out["n_contrib"][y, x],
              ref["n_contrib"][y, x], "T", out["transmittance"][y, x], ref["transmittance"][y, x],
              "fixed", (out["n_contrib"][y, x] >= 0))
    T = out["transmittance"]
    print("   T==0 gpu", int((T == 0).sum()), "ref", int((ref["transmittance"] == 0).sum()),
          "rel(T) max", app_d(T, ref["transmittance"]))
