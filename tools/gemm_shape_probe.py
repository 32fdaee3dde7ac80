"""d_below-shaped GEMMs (delta W, transposed B, ReLU mask) at growing M (debug aid)."""
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
import paper_2505_05356_b200 as tsb
from test_gpu_deform import gemm

ctx = tsb.Context(0)
rng = np.random.default_rng(1)
for n in [8192, 20000, 70000]:
    for O, K in [(3, 128), (128, 128), (128, 84)]:
        delta = rng.normal(size=(n, O)).astype(np.float32)
        W = rng.normal(size=(O, K)).astype(np.float32)
        mask = (rng.random((n, K)) > 0.5).astype(np.float32)
        got = gemm(tsb, ctx, delta, O, 1, W, 1, K, n, K, O, mask=mask)
        ref = (delta.astype(np.float64) @ W.astype(np.float64)) * mask
        bad = np.abs(got - ref) > 1e-4 * np.abs(ref).max()
        rows = np.unique(np.nonzero(bad)[0])
        print(n, O, K, "max err", f"{np.abs(got - ref).max() / np.abs(ref).max():.1e}", "bad rows", rows.size,
              rows[:8], flush=True)
