"""Host-side cost per frame of the public API (prepare + forward) with a tiny scene, so the
device work is negligible (timing experiment, not the bench)."""
import sys
import time
sys.path.insert(0, '.')
import paper_2505_05356_b200 as tsb
from paper_2505_05356_b200 import synthetic

cfg = synthetic.config("c3")
g = synthetic.gaussians(int(sys.argv[1]) if len(sys.argv) > 1 else 1000, 7, n_keyframes=2)
ctx = tsb.Context(0)
scene = tsb.GaussianScene(ctx, g.n, g.n_keyframes, cfg.tof)
scene.set_params(g.position, g.log_scale, g.rotation, g.opacity_logit, g.reflectivity_dc, g.motion)
opts = tsb.RenderOptions()
passes = [tsb.RenderPass(ctx) for _ in range(12)]
for rep in range(3):
    tp = tf = 0.0
    ctx.synchronize()
    t0 = time.perf_counter()
    for i, fr in enumerate(cfg.frames):
        q = passes[i % 12]
        a = time.perf_counter()
        q.prepare(scene, cfg.camera, opts, fr)
        b = time.perf_counter()
        q.forward()
        tf += time.perf_counter() - b
        tp += b - a
    ctx.synchronize()
    dt = time.perf_counter() - t0
n = len(cfg.frames)
print(f"n={g.n} frames/s={n / dt:.0f} host us/frame: prepare {1e6 * tp / n:.1f} forward {1e6 * tf / n:.1f} "
      f"total {1e6 * dt / n:.1f}")
