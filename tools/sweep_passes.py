"""c3 forward throughput vs render passes in flight (timing experiment, not the bench)."""
import sys
import time
sys.path.insert(0, '.')
import torch  # noqa: F401
import paper_2505_05356_b200 as tsb
from paper_2505_05356_b200 import synthetic

cfg = synthetic.config("c3")
g = cfg.scene
ctx = tsb.Context(0)
scene = tsb.GaussianScene(ctx, g.n, g.n_keyframes, cfg.tof)
scene.set_params(g.position, g.log_scale, g.rotation, g.opacity_logit, g.reflectivity_dc, g.motion)
opts = tsb.RenderOptions()
pool = [tsb.RenderPass(ctx) for _ in range(32)]
for npass in [int(a) for a in (sys.argv[1:] or ["1", "2", "3", "4", "6"])]:
    ps = pool[:npass]
    for rep in range(3):
        ctx.synchronize()
        t0 = time.perf_counter()
        for i, fr in enumerate(cfg.frames):
            q = ps[i % npass]
            q.prepare(scene, cfg.camera, opts, fr)
            q.forward()
        ctx.synchronize()
        dt = time.perf_counter() - t0
    print(f"passes={npass} frames/s={len(cfg.frames) / dt:.1f} redo={ctx.redo_count()} launches={ctx.launch_count()}",
          flush=True)
