"""GPU diagnostic: screen-space vs chained gradients for a translated camera (prints only)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2505_05356_b200 as tsb  # noqa: E402
from paper_2505_05356_b200 import synthetic  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from helpers import app_d, gpu_scene, oracle_scene  # noqa: E402

ctx = tsb.Context(0)
cfg = synthetic.config("c1", n=20000)
for tvec in ((0, 0, 0), (0.15, -0.1, 0.4), (0, 0, 0.4), (0.15, 0, 0), (0, 0, -0.3)):
    cam = synthetic.camera(320, 240, 262.5)
    cam.translation = np.array(tvec, float)
    frame = cfg.frames[0]
    scene = gpu_scene(tsb, ctx, cfg.scene, cfg.tof)
    opts = tsb.RenderOptions(counts=True)
    rp = tsb.RenderPass(ctx).prepare(scene, cam, opts, frame)
    rp.debug_keep_screen(True)
    rp.forward()
    rng = np.random.default_rng(3)
    up = rng.normal(0, 1e-3, (4, 240, 320)).astype(np.float32)
    rp.backward(up)
    gr = scene.grads()
    sg = rp.debug_screen_grads()
    op = orc.OraclePass(oracle_scene(cfg.scene, frame, cfg.tof), cam, opts)
    ref = op.forward()
    og = op.backward(d_quad=up.astype(np.float64))
    osg = og["screen"]
    names = ["mx", "my", "ca", "cb", "cc", "op", "coef", "dep"]
    scr = {nm: f"{app_d(sg[:, i], osg[:, i], 1e-4)['max']:.1e}/{app_d(sg[:, i], osg[:, i], 1e-4)['p9999']:.1e}"
           for i, nm in enumerate(names)}
    par = {nm: f"{app_d(a, b, 1e-4)['max']:.1e}/{app_d(a, b, 1e-4)['p9999']:.1e}" for nm, a, b in
           (("pos", gr["d_position"], og["d_position"]), ("ls", gr["d_log_scale"], og["d_log_scale"]),
            ("rot", gr["d_rotation"], og["d_rotation"]), ("op", gr["d_opacity_logit"], og["d_opacity_logit"]))}
    print("t", tvec, "screen", scr, flush=True)
    print("   params", par, "fix", rp.debug_fixups(), flush=True)
    # chain applied to the ORACLE's screen gradients vs the oracle chain: isolates the chain
    d = np.abs(gr["d_position"] - og["d_position"]).max(axis=1)
    worst = np.argsort(d)[-3:]
    order = rp.debug_prepared()["gidx"]
    rank_of = {int(g): r for r, g in enumerate(order)}
    for gi in worst:
        r = rank_of.get(int(gi))
        print("   worst g", gi, "rank", r, "gpu", gr["d_position"][gi], "ref", og["d_position"][gi],
              "scr gpu", None if r is None else sg[r], "scr ref", None if r is None else osg[r], flush=True)
