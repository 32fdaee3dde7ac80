"""GPU stress (diagnostic): the deterministic training iteration of tests/test_gpu_determinism.py
repeated in one process (run with TSB_PREFIX=256 to force prefix aborts and full-order redos).
Prints the first failing iteration, or OK."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2505_05356_b200 as tsb  # noqa: E402
from paper_2505_05356_b200 import synthetic  # noqa: E402
from helpers import gpu_scene  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
det = (sys.argv[2] != "0") if len(sys.argv) > 2 else True
npass = int(sys.argv[3]) if len(sys.argv) > 3 else 3
fresh_ctx = (sys.argv[4] != "0") if len(sys.argv) > 4 else True
cfg = synthetic.config("c1", n=60_000)
frames = [(0, 0.2), (0, 0.5), (0, 0.8), (0, 0.3), (0, 0.6), (0, 0.9)]
ctx = None
target = np.random.default_rng(4).normal(0, 0.02, (4, cfg.camera.height, cfg.camera.width)).astype(np.float32)
opts = tsb.RenderOptions(deterministic=det)
redos = 0
for it in range(iters):
    try:
        if ctx is None or fresh_ctx:
            ctx = tsb.Context(0)  # fresh: the learned prefix cap resets, so every iteration redoes frames
        scene = gpu_scene(tsb, ctx, cfg.scene, cfg.tof)
        rps = [tsb.RenderPass(ctx) for _ in range(npass)]
        for i, fr in enumerate(frames):
            rp = rps[i % npass]
            rp.prepare(scene, cfg.camera, opts, fr)
            rp.forward_loss(target, sync=False)
            rp.backward()
        g = scene.grads()
        scene.adam_step(tsb.LrTable.uniform(1e-3))
        for rp in rps:
            rp.close()
        scene.close()
        if fresh_ctx:
            redos += ctx.redo_count()
            ctx.close()
    except Exception as e:  # noqa: BLE001
        print("FAIL at", it, e)
        sys.exit(1)
print("OK", iters, "redos", redos if fresh_ctx else ctx.redo_count())
