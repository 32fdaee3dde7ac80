"""Per-channel backward error vs the oracle, with and without the fp64-fixed pixels' upstream."""
import sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_2505_05356_b200 as tsb
from paper_2505_05356_b200 import synthetic
from oracle import oracle as orc
from helpers import gpu_scene, oracle_scene, rel_err

ctx = tsb.Context(0)
cfg = synthetic.config("c1")
cam, frame, tof = cfg.camera, cfg.frames[0], cfg.tof
H, W = cam.height, cam.width
opts = tsb.RenderOptions(counts=True, distortion=True)
op = orc.OraclePass(oracle_scene(cfg.scene, frame, tof, 0), cam, opts)
op.forward()
for ch in sys.argv[1:] or ["quad", "depth_raw", "weight", "transmittance", "distortion"]:
    for mask_fixed in (False, True):
        scene = gpu_scene(tsb, ctx, cfg.scene, tof)
        rp = tsb.RenderPass(ctx).prepare(scene, cam, opts, frame).forward()
        fl = rp.debug_fixup_list()
        pix = np.asarray(fl, np.int64) & 0xffffff
        rng = np.random.default_rng(77)
        shp = {"quad": (4, H, W), "phasor": (2, H, W)}.get(ch, (H, W))
        up = rng.normal(0.0, 1e-3, shp).astype(np.float32)
        if mask_fixed:
            up.reshape(-1, H * W)[:, pix] = 0
        rp.backward_buffers(**{"d_" + ch: up})
        gr = scene.grads()
        og = op.backward(**{"d_" + ch: up.astype(np.float64)})
        e = {k: rel_err(gr[k], og[k], 1e-4) for k in ("d_position", "d_log_scale", "d_rotation", "d_opacity_logit")}
        print(ch, "mask_fixed" if mask_fixed else "all", len(pix), {k: f"{v:.2e}" for k, v in e.items()})
