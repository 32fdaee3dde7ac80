"""c3 e2e (public API, pinned host buffers, D2H of quad/depth/weight) vs passes in flight
(timing experiment, not the bench)."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import os
UPLOAD = os.environ.get('UPLOAD', '1') == '1'
import torch
import paper_2505_05356_b200 as tsb
from paper_2505_05356_b200 import synthetic

cfg = synthetic.config("c3")
g = cfg.scene
ctx = tsb.Context(0)
scene = tsb.GaussianScene(ctx, g.n, g.n_keyframes, cfg.tof)
scene.set_params(g.position, g.log_scale, g.rotation, g.opacity_logit, g.reflectivity_dc, g.motion)
opts = tsb.RenderOptions()
H, W = cfg.camera.height, cfg.camera.width
host = {k: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for k, a in
        [("position", g.position), ("log_scale", g.log_scale), ("rotation", g.rotation),
         ("opacity_logit", g.opacity_logit), ("reflectivity_dc", g.reflectivity_dc), ("motion", g.motion)]}
which = (tsb._abi.OUT_QUAD, tsb._abi.OUT_DEPTH, tsb._abi.OUT_WEIGHT)
for npass in [int(a) for a in (sys.argv[1:] or ["8", "12", "16"])]:
    passes = [tsb.RenderPass(ctx) for _ in range(npass)]
    pins = [[torch.empty(sz, dtype=torch.float32, pin_memory=True).numpy() for sz in (4 * H * W, H * W, H * W)]
            for _ in passes]

    def e2e_step():
        if UPLOAD: scene.set_params(host["position"], host["log_scale"], host["rotation"], host["opacity_logit"],
                         host["reflectivity_dc"], host["motion"])
        for i, fr in enumerate(cfg.frames):
            j = i % npass
            q = passes[j]
            q.prepare(scene, cfg.camera, opts, fr)
            q.forward()
            for w, buf in zip(which, pins[j]):
                q.download_async(w, buf)
        for q in passes:
            q.wait()

    e2e_step()
    e2e_step()
    t0 = time.perf_counter()
    for _ in range(3):
        e2e_step()
    ctx.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"passes={npass} e2e frames/s={len(cfg.frames) / dt:.1f}", flush=True)
    for q in passes:
        q.close()
