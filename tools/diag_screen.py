"""Screen-space gradient components vs the oracle for one upstream channel (worst elements)."""
import sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_2505_05356_b200 as tsb
from paper_2505_05356_b200 import synthetic
from oracle import oracle as orc
from helpers import gpu_scene, oracle_scene

ch = sys.argv[1] if len(sys.argv) > 1 else "distortion"
ctx = tsb.Context(0)
cfg = synthetic.config("c1")
cam, frame, tof = cfg.camera, cfg.frames[0], cfg.tof
H, W = cam.height, cam.width
opts = tsb.RenderOptions(counts=True, distortion=True)
op = orc.OraclePass(oracle_scene(cfg.scene, frame, tof, 0), cam, opts)
op.forward()
scene = gpu_scene(tsb, ctx, cfg.scene, tof)
rp = tsb.RenderPass(ctx).prepare(scene, cam, opts, frame).forward()
tsb._abi.check(tsb._abi.lib().tsb_pass_debug_keep_screen(rp.handle, 1))
pix = np.asarray(rp.debug_fixup_list(), np.int64) & 0xffffff
rng = np.random.default_rng(77)
shp = {"quad": (4, H, W), "phasor": (2, H, W)}.get(ch, (H, W))
up = rng.normal(0.0, 1e-3, shp).astype(np.float32)
up.reshape(-1, H * W)[:, pix] = 0
rp.backward_buffers(**{"d_" + ch: up})
sg = rp.debug_screen_grads().astype(np.float64)
og = op.backward(**{"d_" + ch: up.astype(np.float64)})["screen"]
names = ["dmx", "dmy", "dca", "dcb", "dcc", "dop", "dcoef", "ddep"]
for c in range(8):
    a, b = sg[:, c], og[:, c]
    fl = 1e-4 * np.abs(b).max()
    r = np.abs(a - b) / np.maximum(np.abs(b), fl)
    i = int(np.argmax(r))
    print(f"{names[c]:6s} max|ref| {np.abs(b).max():.3e} worst rel {r[i]:.2e} at rank {i}: gpu {a[i]:.6e} ref {b[i]:.6e}"
          f"  p99.9 {np.quantile(r, 0.999):.2e}")
