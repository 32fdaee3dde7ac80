"""Why are pixels sent to the fp64 fix-up?  Reason histogram + how many of them the
fp32 composite actually got wrong (contributor count differs from the oracle)."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import paper_2505_05356_b200 as tsb
from paper_2505_05356_b200 import synthetic
from helpers import gpu_scene, oracle_scene
from oracle import oracle as orc

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfg = synthetic.config(name)
ctx = tsb.Context(0)
scene = gpu_scene(tsb, ctx, cfg.scene, cfg.tof)
rp = tsb.RenderPass(ctx).prepare(scene, cfg.camera, tsb.RenderOptions(counts=True), cfg.frames[0]).forward()
pix, why = rp.debug_fixup_list()
print("fixups", len(pix), "by reason bits:", {b: int(((why >> i) & 1).sum()) for i, b in enumerate(["maha", "alpha", "T"])})
ref = orc.OraclePass(oracle_scene(cfg.scene, cfg.frames[0], cfg.tof), cfg.camera, tsb.RenderOptions()).forward()
out = rp.outputs()
print("after fixup n_contrib mismatches:", int((out["n_contrib"] != ref["n_contrib"]).sum()))
T = ref["transmittance"].ravel()[pix]
print("T/floor of T-flagged pixels (quantiles):", np.quantile(T[(why & 4) > 0] / 1e-4, [0, .1, .5, .9, 1]) if (why & 4).any() else None)
npr = ref["n_processed"].ravel()[pix]
print("walk length (entries) of flagged pixels: quantiles", np.quantile(npr, [0, .5, .9, .99, 1]))
print("all pixels walk length quantiles", np.quantile(ref["n_processed"], [.5, .9, .99, 1]))
