"""World-size-2 data parallelism on CPU (gloo): frames sharded with the product's
shard_frames, per-rank gradients from the oracle, summed with all_reduce, must equal
the single-process sum over all frames (trainer.cpp:123-131 semantics)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_05356_b200.parallel import shard_frames, shard_indices


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def frame_grads(gset, frames, idxs, cam, tof):
    """Oracle gradients of sum_f L_f over the given frames, chained to the canonical
    means and keyframe offsets as trainer.cpp:313-331 does."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__)))
    from helpers import oracle_scene
    from oracle import oracle as orc
    n, nk = gset.n, gset.n_keyframes
    flat = np.zeros(n * 3 * (1 + nk) + n * 8 + 1)
    for i in idxs:
        fr = frames[i]
        op = orc.OraclePass(oracle_scene(gset, fr, tof), cam, type("O", (), {})())
        out = op.forward()
        rng = np.random.default_rng(100 + i)
        target = out["quad"] + rng.normal(0, 0.01, out["quad"].shape)
        d_quad = np.zeros_like(target)
        loss = 0.0
        for m in range(4):
            v, d = orc.mse(out["quad"][m], target[m])
            loss += 0.25 * v
            d_quad[m] = 0.25 * d
        g = op.backward(d_quad=d_quad)
        k, w = fr
        dP = g["d_position"]
        canon = flat[: 3 * n].reshape(n, 3)
        motion = flat[3 * n: 3 * n * (1 + nk)].reshape(nk, n, 3)
        canon += dP
        motion[k] += (1 - w) * dP
        motion[k + 1] += w * dP
        rest = flat[3 * n * (1 + nk):]
        rest[: 3 * n] += g["d_log_scale"].ravel()
        rest[3 * n: 7 * n] += g["d_rotation"].ravel()
        rest[7 * n: 8 * n] += g["d_opacity_logit"]
        rest[-1] += loss
    return flat


def _setup():
    from paper_2505_05356_b200 import synthetic
    g = synthetic.gaussians(300, 4, n_keyframes=2)
    cam = synthetic.camera(64, 48, 55.0)
    frames = [synthetic.frame_for_time(t, 2) for t in (0.0, 0.2, 0.45, 0.7, 1.0)]
    return g, cam, frames, synthetic.ToFConfig(30e6)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, cam, frames, tof = _setup()
    mine = shard_indices(len(frames), rank, world)
    local = torch.from_numpy(frame_grads(g, frames, mine, cam, tof))
    dist.all_reduce(local)
    if rank == 0:
        q.put(local.numpy())
    dist.destroy_process_group()


def test_shard_frames_partition():
    frames = list(range(17))
    for world in (1, 2, 4, 8):
        got = sorted(sum((shard_frames(frames, r, world) for r in range(world)), []))
        assert got == frames
        sizes = [len(shard_frames(frames, r, world)) for r in range(world)]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_frames(frames, 2, 2)


def test_gloo_world2_grad_sum_matches_single_process():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    reduced = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g, cam, frames, tof = _setup()
    single = frame_grads(g, frames, range(len(frames)), cam, tof)
    assert np.allclose(reduced, single, rtol=1e-10, atol=1e-14)
