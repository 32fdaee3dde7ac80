"""Rank worker of tests/test_gpu_dp.py (launched by torch.distributed.run, one rank per GPU):
one FrameShardedTrainer iteration -- this rank's frames, NCCL allreduce of the gradient
buffer through the library's own communicator (tsb_scene_allreduce_grads), fused Adam --
then the reduced gradients and the parameters after the step are saved for the test."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2505_05356_b200 as tsb  # noqa: E402
from paper_2505_05356_b200 import synthetic  # noqa: E402
from paper_2505_05356_b200.parallel import FrameShardedTrainer  # noqa: E402


def setup():
    g = synthetic.gaussians(30_000, 12, n_keyframes=2)
    cam = synthetic.camera(320, 240, 262.5)
    rng = np.random.default_rng(7)
    frames = [tsb.frame_for_time(t, 2) for t in rng.uniform(0, 1, 16)]
    targets = [rng.normal(0, 0.03, (4, 240, 320)).astype(np.float32) for _ in frames]
    return g, cam, frames, targets


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    out = Path(sys.argv[1])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    g, cam, frames, targets = setup()
    ctx = tsb.Context(local)
    scene = tsb.GaussianScene(ctx, g.n, g.n_keyframes, tsb.ToFConfig(30e6))
    scene.set_params(g.position, g.log_scale, g.rotation, g.opacity_logit, g.reflectivity_dc, g.motion)
    obj = [tsb.Comm.unique_id() if rank == 0 else b""]
    dist.broadcast_object_list(obj, src=0)
    comm = tsb.Comm(ctx, obj[0], world, rank)
    trainer = FrameShardedTrainer(ctx, scene, cam, tsb.RenderOptions(), lr=tsb.LrTable.uniform(1e-3), comm=comm,
                                  rank=rank, world=world, passes=4)
    for k, i in enumerate(range(rank, len(frames), world)):  # this rank's frames, then the allreduce
        rp = trainer.passes[k % len(trainer.passes)]
        rp.prepare(scene, cam, tsb.RenderOptions(), frames[i])
        rp.forward_loss(targets[i], sync=False)
        rp.backward()
    scene.allreduce_grads(comm)
    gr = scene.grads()
    scene.adam_step(tsb.LrTable.uniform(1e-3))
    prm = scene.get_params()
    np.savez(out / f"rank{rank}.npz", d_position=gr["d_position"], d_motion=gr["d_motion"],
             d_log_scale=gr["d_log_scale"], loss=np.array(gr["loss"]), position=prm["position"])
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
