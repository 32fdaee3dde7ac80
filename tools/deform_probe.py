"""Locate DeformNet gradient errors vs batch size (debug aid)."""
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
import paper_2505_05356_b200 as tsb
from oracle import deform as od
from test_gpu_deform import _nets

ctx = tsb.Context(0)
cfg = od.DeformConfig()
for n in [int(a) for a in (sys.argv[1:] or ["3000", "5000", "8192", "20000", "70000"])]:
    onet, gnet, pos, rng = _nets(tsb, ctx, cfg, 5, n=n)
    ref, cache = onet.offsets(pos.astype(np.float64), 0.8, with_cache=True)
    off = gnet.offsets(pos, 0.8)
    up = rng.normal(size=pos.shape).astype(np.float32)
    dW, db, _ = onet.backward(cache, up.astype(np.float64), want_positions=False)
    gnet.zero_grads()
    gnet.backward(up, want_positions=False)
    g = gnet.grads()
    k = 0
    errs = []
    for w, b in zip(dW, db):
        for part in (w.ravel(), b):
            e = np.abs(g[k:k + part.size] - part).max() / np.abs(part).max()
            errs.append(f"{e:.1e}")
            k += part.size
    print(n, "offsets", f"{np.abs(off - ref).max() / np.abs(ref).max():.1e}", "blocks(W,b per layer):", errs,
          flush=True)
