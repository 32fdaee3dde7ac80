"""Seeded synthetic inputs for the BASELINE.json configurations.

No dataset or checkpoint is available (and none is named), so every config is
generated here with the distributions BASELINE.json states.  Arrays are fp32
SoA; the CPU oracle reads the same fp32 values promoted to double, so GPU and
oracle see bit-identical inputs.

c0  N=20k static, 320x240 f300, 30 MHz                      (forward parity / CPU ref)
c1  N=100k + 2 keyframe offsets ~N(0,0.05), t=0.5, 640x480 f525; L2 vs seed-1 target + N(0,0.01^2)
c2  N=500k, 9 keyframes, 30+60 MHz (8 channels), 640x576 f525; 8 frames/iter; rotating 20k rod target
c3  N=1M dynamic (2 keyframes), z~U[0.5,8], 640x480 f525; 300 frames at t=i/299 (forward sweep)
c4  N=2M at 1024x1024 f840; 64 frames/iter, t~U[0,1]; 18 floats/Gaussian of gradients
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .render import SH_C0, CameraModel, ToFConfig, frame_for_time

F30 = 30e6


@dataclass
class GaussianSet:
    position: np.ndarray       # (n,3) f32 canonical mean
    log_scale: np.ndarray      # (n,3) f32
    rotation: np.ndarray       # (n,4) f32 (w,x,y,z)
    opacity_logit: np.ndarray  # (n,) f32
    reflectivity_dc: np.ndarray  # (n,) f32  (= amplitude / SH_C0)
    motion: Optional[np.ndarray] = None  # (k, n, 3) f32 keyframe offsets

    @property
    def n(self):
        return int(self.position.shape[0])

    @property
    def n_keyframes(self):
        return 0 if self.motion is None else int(self.motion.shape[0])

    def rendered_means(self, frame) -> np.ndarray:
        """fp64 rendered means (trainer.cpp:259-279), same op order as the kernels."""
        x = self.position.astype(np.float64)
        if self.motion is None:
            return x
        k, w = frame
        xi = x + self.motion[k].astype(np.float64)
        xip1 = x + self.motion[k + 1].astype(np.float64)
        return xi if w == 0.0 else (1.0 - w) * xi + w * xip1


def gaussians(n: int, seed: int, *, z_range=(1.0, 5.0), n_keyframes: int = 0, motion_std: float = 0.05,
              xy_range=(-1.0, 1.0)) -> GaussianSet:
    rng = np.random.default_rng(seed)
    pos = np.empty((n, 3), np.float64)
    pos[:, 0] = rng.uniform(xy_range[0], xy_range[1], n)
    pos[:, 1] = rng.uniform(xy_range[0], xy_range[1], n)
    pos[:, 2] = rng.uniform(z_range[0], z_range[1], n)
    log_scale = rng.normal(-3.0, 0.3, (n, 3))
    q = rng.normal(0.0, 1.0, (n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = rng.normal(0.0, 1.0, n)
    amp = np.exp(rng.normal(-1.0, 0.5, n))
    motion = None
    if n_keyframes:
        motion = rng.normal(0.0, motion_std, (n_keyframes, n, 3)).astype(np.float32)
    return GaussianSet(pos.astype(np.float32), log_scale.astype(np.float32), q.astype(np.float32),
                       op.astype(np.float32), (amp / SH_C0).astype(np.float32), motion)


def concat(a: GaussianSet, b: GaussianSet) -> GaussianSet:
    mo = None
    if a.motion is not None:
        mo = np.concatenate([a.motion, b.motion], axis=1)
    return GaussianSet(*(np.concatenate([getattr(a, k), getattr(b, k)]) for k in
                         ("position", "log_scale", "rotation", "opacity_logit", "reflectivity_dc")), mo)


def rotating_rod(n: int, seed: int, n_keyframes: int, omega: float = 10.0, length: float = 1.2,
                 ratio: float = 20.0, center=(0.0, 0.0, 3.0)) -> GaussianSet:
    """A 'bat-like' rod of anisotropic Gaussians (scale ratio 20:1) whose centres rotate
    about the view axis at omega rad per unit t; keyframe offsets sample the rotation."""
    rng = np.random.default_rng(seed)
    s = rng.uniform(-0.5, 0.5, n) * length
    base = np.zeros((n, 3))
    base[:, 0] = s
    base += np.asarray(center)
    small = 0.01
    log_scale = np.log(np.stack([np.full(n, small * ratio), np.full(n, small), np.full(n, small)], 1))
    log_scale += rng.normal(0, 0.05, (n, 3))
    q = np.zeros((n, 4))
    q[:, 0] = 1.0
    op = rng.normal(2.0, 0.5, n)
    amp = np.exp(rng.normal(-0.5, 0.3, n))
    K = n_keyframes - 1
    motion = np.zeros((n_keyframes, n, 3))
    for k in range(n_keyframes):
        th = omega * (k / K)
        c, sn = np.cos(th), np.sin(th)
        rot = np.stack([c * s, sn * s, np.zeros(n)], 1) + np.asarray(center)
        motion[k] = rot - base
    return GaussianSet(base.astype(np.float32), log_scale.astype(np.float32), q.astype(np.float32),
                       op.astype(np.float32), (amp / SH_C0).astype(np.float32), motion.astype(np.float32))


@dataclass
class Config:
    name: str
    scene: GaussianSet
    camera: CameraModel
    tof: ToFConfig
    frames: List[tuple]                 # (key, w) per rendered frame
    frames_per_iter: int = 1
    target: Optional[GaussianSet] = None  # scene whose render is the L2 target
    noise_std: float = 0.0
    lr: float = 1e-3
    iterations: int = 1
    notes: str = ""


def camera(w, h, f, cx=None, cy=None) -> CameraModel:
    return CameraModel(fx=f, fy=f, cx=w / 2 if cx is None else cx, cy=h / 2 if cy is None else cy, width=w,
                       height=h)


def config(name: str, n: Optional[int] = None) -> Config:
    """Build a BASELINE config; `n` overrides the Gaussian count (parity tests use
    smaller instances of the same distributions)."""
    if name == "c0":
        n = n or 20_000
        return Config("c0", gaussians(n, 0), camera(320, 240, 300.0), ToFConfig(F30), [(0, 0.0)],
                      notes="static forward, seed 0")
    if name == "c1":
        n = n or 100_000
        return Config("c1", gaussians(n, 0, n_keyframes=2), camera(640, 480, 525.0), ToFConfig(F30), [(0, 0.5)],
                      target=gaussians(n, 1, n_keyframes=2), noise_std=0.01, lr=1e-3,
                      notes="one training step at t=0.5 vs seed-1 target + N(0,0.01^2)")
    if name == "c2":
        n = n or 500_000
        nk = 9
        rod_n = min(20_000, max(n // 25, 16))
        rng = np.random.default_rng(7)
        ts = rng.uniform(0.0, 1.0, 8)
        return Config("c2", gaussians(n, 0, n_keyframes=nk), camera(640, 576, 525.0, 320, 288),
                      ToFConfig(F30, second_frequency=60e6), [frame_for_time(t, nk) for t in ts],
                      frames_per_iter=8,
                      target=concat(gaussians(n, 1, n_keyframes=nk), rotating_rod(rod_n, 2, nk)),
                      lr=1e-3, iterations=200, notes="2 frequencies, 8 frames/iter, rotating rod target")
    if name == "c3":
        n = n or 1_000_000
        return Config("c3", gaussians(n, 0, z_range=(0.5, 8.0), n_keyframes=2), camera(640, 480, 525.0),
                      ToFConfig(F30), [frame_for_time(i / 299, 2) for i in range(300)],
                      notes="forward sweep, 300 frames at t=i/299")
    if name == "c4":
        n = n or 2_000_000
        rng = np.random.default_rng(11)
        ts = rng.uniform(0.0, 1.0, 64)
        return Config("c4", gaussians(n, 0, n_keyframes=2), camera(1024, 1024, 840.0, 512, 512), ToFConfig(F30),
                      [frame_for_time(t, 2) for t in ts], frames_per_iter=64,
                      target=gaussians(n, 1, n_keyframes=2), lr=1e-3,
                      notes="data-parallel training, 64 frames/iter")
    raise KeyError(name)
