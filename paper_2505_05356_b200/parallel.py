"""Frame-sharded data parallelism for the training step.

The reference fit() renders a batch of frames sequentially against one set of
Gaussians and sums the per-render SceneGrads before one Adam step
(trainer.cpp:123-131, 256, 312, 339-378).  Frames are independent, so on N GPUs
each rank renders its share of the frames against replicated parameters,
gradients are summed with one NCCL allreduce of the flat per-Gaussian gradient
buffer (tsb_scene_allreduce_grads), and every rank applies the identical fused
Adam step -- replicas stay bitwise identical because the allreduce result is.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

from .render import AdamParams, CameraModel, Comm, Context, GaussianScene, LrTable, RenderOptions, RenderPass


def shard_frames(frames: Sequence, rank: int, world: int) -> List:
    """Round-robin frame assignment: rank r gets frames r, r+world, ... (every frame
    exactly once across ranks, shares differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_frames: bad rank/world")
    return list(frames[rank::world])


def shard_indices(n: int, rank: int, world: int) -> List[int]:
    return list(range(rank, n, world))


class FrameShardedTrainer:
    """One optimisation step = for my frames: prepare -> forward + fused L2 loss ->
    backward (accumulates into the scene); allreduce; fused Adam + densify statistic."""

    def __init__(self, ctx: Context, scene: GaussianScene, camera: CameraModel,
                 options: Optional[RenderOptions] = None, lr: Optional[LrTable] = None,
                 adam: AdamParams = AdamParams(), comm: Optional[Comm] = None, rank: int = 0, world: int = 1,
                 channel_weight: Optional[Sequence[float]] = None, passes: int = 3, ssim_mix: float = 0.0):
        self.ctx, self.scene, self.camera = ctx, scene, camera
        self.options = options or RenderOptions()
        self.lr = lr or LrTable()
        self.adam = adam
        self.comm, self.rank, self.world = comm, rank, world
        self.channel_weight = list(channel_weight or [0.25] * (4 * scene.n_freq))
        self.ssim_mix = ssim_mix  # LossWeights::ssim_mix (trainer.hpp:49; BASELINE configs use 0)
        # render passes (one stream each) rotate over frames: frame i's backward overlaps the
        # preprocess/sort/binning of the next frames; nothing waits for the device until a pass
        # is reused (it settles its previous frame) and at the allreduce / Adam step.  Gradient
        # writes are serialised by the scene's event chain inside the library.
        self.passes = [RenderPass(ctx) for _ in range(max(1, passes))]
        self.rp = self.passes[0]

    def step(self, frames: Sequence, target: Callable[[int], object]) -> None:
        """frames: the iteration's (key, w) frames (all ranks pass the same list);
        target(i) -> host array (4*n_freq, H, W) or an int device pointer for frame i."""
        for k, i in enumerate(shard_indices(len(frames), self.rank, self.world)):
            rp = self.passes[k % len(self.passes)]
            rp.prepare(self.scene, self.camera, self.options, frames[i])
            t = target(i)
            if isinstance(t, int):
                rp.forward_loss(None, self.channel_weight, sync=False, device_ptr=t, ssim_mix=self.ssim_mix)
            else:
                rp.forward_loss(t, self.channel_weight, sync=False, ssim_mix=self.ssim_mix)
            rp.backward()
        if self.comm is not None and self.world > 1:
            self.scene.allreduce_grads(self.comm)
        self.scene.adam_step(self.lr, self.adam)
