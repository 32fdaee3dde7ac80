"""DeformNet forward/backward throughput on the tensor cores (timing tool; the bench leg
is in bench.py).  Scene-coupled: offsets of N canonical positions into a keyframe plane,
backward from that keyframe's gradient (no host copies)."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2505_05356_b200 as tsb
from paper_2505_05356_b200 import synthetic

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
ctx = tsb.Context(0)
g = synthetic.gaussians(n, 0, n_keyframes=2)
scene = tsb.GaussianScene(ctx, g.n, g.n_keyframes, tsb.ToFConfig(30e6))
scene.set_params(g.position, g.log_scale, g.rotation, g.opacity_logit, g.reflectivity_dc, g.motion)
net = tsb.DeformNet(ctx)
rng = np.random.default_rng(0)
net.set_parameters(rng.normal(size=net.parameter_count).astype(np.float32) * 0.05)
stream = torch.cuda.ExternalStream(ctx.stream)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for _ in range(2):
    net.scene_offsets(scene, 0, 0.3)
    net.scene_backward(scene, 0)
ctx.synchronize()
reps = 5
ev[0].record(stream)
for _ in range(reps):
    net.scene_offsets(scene, 0, 0.3)
ev[1].record(stream)
for _ in range(reps):
    net.scene_backward(scene, 0)
ev[2].record(stream)
ctx.synchronize()
fwd = ev[0].elapsed_time(ev[1]) / reps
bwd = ev[1].elapsed_time(ev[2]) / reps
din, w, L = net.input_dim, net.width, net.hidden_layers
mac = din * w + (L - 1) * w * w + w * 3
f_fwd = 2.0 * mac * n
f_bwd = 2.0 * f_fwd  # weight gradients + input gradients
print(f"n={n} fwd {fwd:.3f} ms ({f_fwd / fwd / 1e9:.1f} TFLOP/s algorithmic, x3 issued for 3xTF32) "
      f"bwd {bwd:.3f} ms ({f_bwd / bwd / 1e9:.1f} TFLOP/s)", flush=True)
