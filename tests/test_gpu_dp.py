"""Frame-sharded data parallelism on the GPUs of this node: world =
min(#GPUs, 8) ranks, each renders its share of 16 frames, gradients summed by the library's
NCCL allreduce (tsb_scene_allreduce_grads, trainer.cpp:123-131), identical fused Adam on
every rank.  The reduced gradients must equal a single-GPU pass over all frames (summation
order only) and every rank must hold bit-identical parameters after the step.  Skipped with
fewer than two GPUs (NCCL cannot give two ranks one device)."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from helpers import rel_err

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs (NCCL ranks need distinct devices)")
def test_frame_sharded_allreduce_matches_single_gpu(tmp_path):
    world = min(_gpus(), 8)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(HERE / "dp_worker.py"), str(tmp_path)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    ranks = [np.load(tmp_path / f"rank{k}.npz") for k in range(world)]
    for k in range(1, world):  # replicas stay identical: the allreduce result is the same everywhere
        assert np.array_equal(ranks[0]["position"], ranks[k]["position"])
    # the same iteration on one GPU, all frames, no communicator
    sys.path.insert(0, str(HERE))
    import dp_worker
    import paper_2505_05356_b200 as tsb
    g, cam, frames, targets = dp_worker.setup()
    ctx = tsb.Context(0)
    scene = tsb.GaussianScene(ctx, g.n, g.n_keyframes, tsb.ToFConfig(30e6))
    scene.set_params(g.position, g.log_scale, g.rotation, g.opacity_logit, g.reflectivity_dc, g.motion)
    rp = tsb.RenderPass(ctx)
    for i, fr in enumerate(frames):
        rp.prepare(scene, cam, tsb.RenderOptions(), fr)
        rp.forward_loss(targets[i], sync=False)
        rp.backward()
    gr = scene.grads()
    for name in ("d_position", "d_motion", "d_log_scale"):
        assert rel_err(ranks[0][name], gr[name], 1e-4) < 1e-5 * 10, name
    assert float(ranks[0]["loss"]) == pytest.approx(gr["loss"], rel=1e-9)


def test_nccl_allreduce_single_rank_runs_the_product_path():
    """The library's NCCL path on a 1-GPU box: a one-rank communicator (tsb_comm_create),
    the gradient + statistics allreduce (tsb_scene_allreduce_grads) after a training frame --
    the sum over one rank leaves every gradient bit-identical; the communicator is destroyed
    cleanly.  (The multi-rank case needs >= 2 GPUs: test above.)"""
    sys.path.insert(0, str(HERE))
    import dp_worker
    import paper_2505_05356_b200 as tsb
    g, cam, frames, targets = dp_worker.setup()
    ctx = tsb.Context(0)
    scene = tsb.GaussianScene(ctx, g.n, g.n_keyframes, tsb.ToFConfig(30e6))
    scene.set_params(g.position, g.log_scale, g.rotation, g.opacity_logit, g.reflectivity_dc, g.motion)
    rp = tsb.RenderPass(ctx)
    rp.prepare(scene, cam, tsb.RenderOptions(), frames[0])
    rp.forward_loss(targets[0], sync=False)
    rp.backward()
    before = scene.grads()
    comm = tsb.Comm(ctx, tsb.Comm.unique_id(), 1, 0)
    scene.allreduce_grads(comm)
    after = scene.grads()
    comm.close()
    for name in before:
        assert np.array_equal(np.asarray(before[name]), np.asarray(after[name])), name
