"""Diagnostic: fp32 B200 forward vs fp64 oracle error distribution on a config."""
import sys, json
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2505_05356_b200 as tsb
from paper_2505_05356_b200 import synthetic
from oracle import oracle as orc
from helpers import gpu_scene, oracle_scene

name = sys.argv[1] if len(sys.argv) > 1 else "c0"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = synthetic.config(name, n)
ctx = tsb.Context(0)
opts = tsb.RenderOptions(counts=True)
scene = gpu_scene(tsb, ctx, cfg.scene, cfg.tof)
rp = tsb.RenderPass(ctx).prepare(scene, cfg.camera, opts, cfg.frames[0]).forward()
out = rp.outputs()
print("fixups", rp.debug_fixups(), "visible", rp.visible_count(), "keys", rp.num_keys())
op = orc.OraclePass(oracle_scene(cfg.scene, cfg.frames[0], cfg.tof), cfg.camera, opts)
ref = op.forward()
print("n_contrib equal", np.array_equal(out["n_contrib"], ref["n_contrib"]), "mismatch", int((out["n_contrib"] != ref["n_contrib"]).sum()))
for k in ["quad", "depth_raw", "weight", "transmittance", "depth"]:
    a = out[k].astype(np.float64); b = ref[k]
    m = np.isfinite(b)
    a, b = a[m], b[m]
    ab = np.abs(a - b)
    floor = 1e-6 * np.abs(b).max()
    rel = ab / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    i = int(np.argmax(rel))
    print(f"{k:14s} max|ref|={np.abs(b).max():.3e} maxabs={ab.max():.3e} maxrel={rel.max():.3e} p9999={np.quantile(rel, 0.9999):.3e} "
          f"at ref={b[i]:.6e} got={a[i]:.6e}")
# where is the worst quad pixel
a = out["quad"].astype(np.float64); b = ref["quad"]
floor = 1e-6 * np.abs(b).max()
rel = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
c, y, x = np.unravel_index(np.argmax(rel), rel.shape)
print("worst quad pixel", c, y, x, "n_contrib", ref["n_contrib"][y, x], "T", ref["transmittance"][y, x], "vals", a[:, y, x], b[:, y, x])
