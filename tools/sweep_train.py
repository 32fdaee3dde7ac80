"""c4 train iters/s vs render passes in flight (timing experiment, not the bench)."""
import sys
import time
sys.path.insert(0, '.')
import torch
import paper_2505_05356_b200 as tsb
from paper_2505_05356_b200 import synthetic
from paper_2505_05356_b200.parallel import FrameShardedTrainer

cfg = synthetic.config("c4")
g, tg = cfg.scene, cfg.target
cam, opts = cfg.camera, tsb.RenderOptions()
ctx = tsb.Context(0)
scene = tsb.GaussianScene(ctx, g.n, g.n_keyframes, cfg.tof)
scene.set_params(g.position, g.log_scale, g.rotation, g.opacity_logit, g.reflectivity_dc, g.motion)
tscene = tsb.GaussianScene(ctx, tg.n, tg.n_keyframes, cfg.tof)
tscene.set_params(tg.position, tg.log_scale, tg.rotation, tg.opacity_logit, tg.reflectivity_dc, tg.motion)
rp = tsb.RenderPass(ctx)
H, W = cam.height, cam.width
targets = torch.empty((len(cfg.frames), 4, H, W), dtype=torch.float32, device="cuda:0")
for i, fr in enumerate(cfg.frames):
    rp.prepare(tscene, cam, opts, fr).forward()
    targets[i].copy_(torch.from_numpy(rp.download(tsb._abi.OUT_QUAD, shape=(4, H, W))))
torch.cuda.synchronize()
for npass in [int(a) for a in (sys.argv[1:] or ["2", "3", "4"])]:
    tr = FrameShardedTrainer(ctx, scene, cam, opts, lr=tsb.LrTable.uniform(cfg.lr), passes=npass)
    tr.step(cfg.frames, lambda i: targets[i].data_ptr())
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        tr.step(cfg.frames, lambda i: targets[i].data_ptr())
    ctx.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"passes={npass} iters/s={1 / dt:.2f} redo={ctx.redo_count()}", flush=True)
    for q in tr.passes:
        q.close()
