"""Accuracy of long tensor-core K-reductions (dW-like): error vs split-K slice length."""
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
import paper_2505_05356_b200 as tsb
from test_gpu_deform import gemm

ctx = tsb.Context(0)
rng = np.random.default_rng(0)
n, o, k = 65536, 128, 128
delta = rng.normal(size=(n, o)).astype(np.float32)
H = np.abs(rng.normal(size=(n, k))).astype(np.float32)
ref = delta.astype(np.float64).T @ H.astype(np.float64)
for kps in [256, 1024, 4096, 16384, 65536]:
    slices = n // kps
    got = gemm(tsb, ctx, delta, 1, o, H, 1, k, o, k, n, slices=slices)
    err = np.abs(got - ref)
    print(f"rows/slice={kps:6d} normwise={err.max() / np.abs(ref).max():.2e} "
          f"mean_signed={(got - ref).mean() / np.abs(ref).mean():.2e}", flush=True)
