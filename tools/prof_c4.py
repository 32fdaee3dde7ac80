"""Profiling driver: a few c4 train frames (forward_loss + backward) on one pass.
Used under ncu; never a bench number."""
import sys
sys.path.insert(0, '.')
import paper_2505_05356_b200 as tsb
from paper_2505_05356_b200 import synthetic

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = synthetic.config("c4")
g = cfg.scene
ctx = tsb.Context(0)
scene = tsb.GaussianScene(ctx, g.n, g.n_keyframes, cfg.tof)
scene.set_params(g.position, g.log_scale, g.rotation, g.opacity_logit, g.reflectivity_dc, g.motion)
rp = tsb.RenderPass(ctx)
opts = tsb.RenderOptions()
rp.prepare(scene, cfg.camera, opts, cfg.frames[0]).forward()
tgt = rp.outputs()["quad"] * 0.9
for i in range(1 + frames):
    rp.prepare(scene, cfg.camera, opts, cfg.frames[(i * 7) % len(cfg.frames)])
    rp.forward_loss(tgt, sync=False)
    rp.backward()
ctx.synchronize()
print("ok", rp.visible_count(), rp.debug_fixups(), ctx.redo_count())
pix, why = rp.debug_fixup_list()
print("fixup reasons", {b: int(((why & b) != 0).sum()) for b in (1, 2, 4, 8, 16)})
