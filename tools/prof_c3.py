"""Profiling driver: a few c3 frames (forward) and, optionally, one c4-shaped
train frame (forward_loss + backward).  Used under ncu; never a bench number."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2505_05356_b200 as tsb
from paper_2505_05356_b200 import synthetic

mode = sys.argv[1] if len(sys.argv) > 1 else "fwd"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = synthetic.config("c3")
g = cfg.scene
ctx = tsb.Context(0)
scene = tsb.GaussianScene(ctx, g.n, g.n_keyframes, cfg.tof)
scene.set_params(g.position, g.log_scale, g.rotation, g.opacity_logit, g.reflectivity_dc, g.motion)
rp = tsb.RenderPass(ctx)
opts = tsb.RenderOptions()
tgt = None
for i in range(2 + frames):
    fr = cfg.frames[(i * 53) % 300]
    rp.prepare(scene, cfg.camera, opts, fr)
    if mode == "train":
        if tgt is None:
            rp.forward()
            tgt = rp.outputs()["quad"] * 0.9
        rp.forward_loss(tgt, sync=False)
        rp.backward()
    else:
        rp.forward()
ctx.synchronize()
print("ok", rp.visible_count(), rp.num_keys(), rp.debug_fixups())
