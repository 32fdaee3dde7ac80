"""GPU diagnostic: the worst d_position elements of the posed-camera parity case (prints only)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2505_05356_b200 as tsb  # noqa: E402
from paper_2505_05356_b200 import synthetic  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from helpers import gpu_scene, oracle_scene  # noqa: E402
from test_gpu_parity_shapes import rotation_matrix  # noqa: E402

ctx = tsb.Context(0)
cfg = synthetic.config("c1")
cam = synthetic.camera(640, 480, 525.0)
cam.rotation = rotation_matrix((0.3, -0.8, 0.2), 0.12)
cam.translation = np.array([0.15, -0.1, 0.4])
opts = tsb.RenderOptions(counts=True, bg_quad=(0.01, -0.02, 0.015, 0.005), bg_phasor=(0.02, -0.01))
frame = cfg.frames[0]
scene = gpu_scene(tsb, ctx, cfg.scene, cfg.tof)
rp = tsb.RenderPass(ctx).prepare(scene, cam, opts, frame)
rp.debug_keep_screen(True)
rp.forward()
H, W = cam.height, cam.width
rng = np.random.default_rng(31)
ups = {"d_quad": rng.normal(0, 1e-3, (4, H, W)), "d_phasor": rng.normal(0, 1e-3, (2, H, W)),
       "d_depth_raw": rng.normal(0, 1e-3, (H, W)), "d_weight": rng.normal(0, 1e-3, (H, W)),
       "d_transmittance": rng.normal(0, 1e-3, (H, W))}
ups = {k: v.astype(np.float32) for k, v in ups.items()}
rp.backward_buffers(**ups)
gr = scene.grads()
sg = rp.debug_screen_grads()
op = orc.OraclePass(oracle_scene(cfg.scene, frame, cfg.tof), cam, opts)
op.forward()
og = op.backward(**{k: v.astype(np.float64) for k, v in ups.items()})
a, b = gr["d_position"].astype(np.float64), og["d_position"]
floor = 1e-4 * np.abs(b).max()
rel = (np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)).max(axis=1)
order = rp.debug_prepared()
rank_of = {int(g): r for r, g in enumerate(order["gidx"])}
fix = set(rp.debug_fixup_list()[0].tolist())
for gi in np.argsort(rel)[-6:]:
    r = rank_of.get(int(gi))
    rc = order["rect"][r]
    npix_fix = sum(1 for y in range(rc[2], rc[3]) for x in range(rc[0], rc[1]) if y * W + x in fix)
    print("g", gi, "rel %.2e" % rel[gi], "gpu", a[gi], "ref", b[gi], "floor %.2e" % floor, "rank", r, "rect", rc,
          "fixed px in rect", npix_fix)
    print("   screen gpu", sg[r])
    print("   screen ref", og["screen"][r])
