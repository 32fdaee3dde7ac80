"""Python mirror of the reference renderer / optimiser API over the C ABI.

Reference names are kept: ``CameraModel`` (camera.hpp:9-49), ``ToFConfig``
(tof.hpp:13-21), ``RenderOptions`` (splat.hpp:28-37), ``RenderPass`` with
``forward`` / ``backward`` / ``visible_count`` (splat.hpp:97-112),
``AdamParams`` / ``LrTable`` (trainer.hpp:14-44).  The Gaussian parameters
live on the GPU in a ``GaussianScene`` (the device counterpart of
``CanonicalScene`` + the trainer's ``Params`` / ``GroupGrads`` / ``AdamState``,
trainer.cpp:63-132), so a training loop never copies them to the host.

Every method calls libtsb.so; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _abi
from ._abi import check, lib

SH_C0 = 0.28209479177387814


@dataclass
class ToFConfig:
    """tof.hpp:13-21; a second frequency renders a second quad sharing geometry."""
    modulation_frequency: float = 29.9792458e6
    source_intensity: float = 1.0
    speed_of_light: float = 299792458.0
    second_frequency: Optional[float] = None

    @property
    def frequencies(self):
        f = [self.modulation_frequency]
        if self.second_frequency:
            f.append(self.second_frequency)
        return f


@dataclass
class CameraModel:
    """Pinhole camera, pixel centres at +0.5, p_cam = R p + t (camera.hpp:9-49)."""
    fx: float = 1.0
    fy: float = 1.0
    cx: float = 0.0
    cy: float = 0.0
    width: int = 0
    height: int = 0
    near_plane: float = 0.2
    far_plane: float = 100.0
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def valid(self) -> bool:
        return (self.fx > 0 and self.fy > 0 and self.width > 0 and self.height > 0 and self.near_plane > 0
                and self.far_plane > self.near_plane)

    def to_abi(self) -> _abi.Camera:
        c = _abi.Camera()
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        c.width, c.height = int(self.width), int(self.height)
        c.near_plane, c.far_plane = float(self.near_plane), float(self.far_plane)
        R = np.asarray(self.rotation, dtype=np.float64).reshape(9)
        t = np.asarray(self.translation, dtype=np.float64).reshape(3)
        for i in range(9):
            c.R[i] = R[i]
        for i in range(3):
            c.t[i] = t[i]
        return c


@dataclass
class RenderOptions:
    """splat.hpp:13-37 (+ Backgrounds::quad / ::phasor, 4 resp. 2 values per frequency)."""
    alpha_threshold: float = 1.0 / 255.0
    transmittance_floor: float = 1e-4
    dilation: float = 0.3
    sigma_cutoff: float = 3.0
    coverage_eps: float = 1e-12
    tile_size: int = 16
    bg_quad: Sequence[float] = (0.0, 0.0, 0.0, 0.0)
    bg_phasor: Sequence[float] = (0.0, 0.0)
    distortion: bool = False  # RenderChannels::distortion (needed for a distortion upstream)
    counts: bool = False      # also emit per-pixel n_contrib / n_processed (parity diagnostics)
    full_lists: bool = False  # bin every tile's complete list (parity); default stops binning a tile
                              # once all its pixels have terminated (identical outputs)
    color: bool = False       # RenderChannels::color (scene created with color=True)
    flow: bool = False        # RenderChannels::flow (motions via RenderPass.set_motion)
    bg_color: Sequence[float] = (0.0, 0.0, 0.0)
    exact: bool = False       # reference-exact mode (TSB_CH_EXACT): every pixel in fp64, fp64 output planes
    deterministic: bool = False  # bit-reproducible ToF gradients / loss (TSB_CH_DETERMINISTIC)

    def to_abi(self) -> _abi.RenderOptions:
        o = _abi.RenderOptions()
        o.alpha_threshold = float(self.alpha_threshold)
        o.transmittance_floor = float(self.transmittance_floor)
        o.dilation = float(self.dilation)
        o.sigma_cutoff = float(self.sigma_cutoff)
        o.coverage_eps = float(self.coverage_eps)
        o.tile_size = int(self.tile_size)
        o.channels = _abi.CH_QUAD | _abi.CH_DEPTH | _abi.CH_WEIGHT | _abi.CH_TRANSM | (
            _abi.CH_COUNTS if self.counts else 0) | (_abi.CH_FULL_LISTS if self.full_lists else 0) | (
            _abi.CH_PHASOR) | (_abi.CH_DISTORTION if self.distortion else 0) | (
            _abi.CH_COLOR if self.color else 0) | (_abi.CH_FLOW if self.flow else 0) | (
            _abi.CH_EXACT if self.exact else 0) | (_abi.CH_DETERMINISTIC if self.deterministic else 0)
        bq = np.zeros(8)
        b = np.asarray(self.bg_quad, dtype=np.float64).reshape(-1)[:8]
        bq[: b.size] = b
        for i in range(8):
            o.bg_quad[i] = bq[i]
        bp = np.zeros(4)
        b = np.asarray(self.bg_phasor, dtype=np.float64).reshape(-1)[:4]
        bp[: b.size] = b
        for i in range(4):
            o.bg_phasor[i] = bp[i]
        bc = np.asarray(self.bg_color, dtype=np.float64).reshape(-1)
        for i in range(3):
            o.bg_color[i] = float(bc[i]) if bc.size > i else 0.0
        return o


@dataclass
class AdamParams:
    """trainer.hpp:14-18."""
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15


@dataclass
class LrTable:
    """Per-group learning rates, already resolved (trainer.cpp:339-366: position lr
    is multiplied by the scene extent there; reflectivity uses appearance/10)."""
    position: float = 1.6e-4
    log_scale: float = 5e-3
    rotation: float = 1e-3
    opacity: float = 0.05
    reflectivity: float = 1.6e-4
    motion: float = 1.6e-4
    color: float = 1.6e-3

    @staticmethod
    def uniform(lr: float) -> "LrTable":
        return LrTable(lr, lr, lr, lr, lr, lr, lr)


def scene_extent(positions) -> float:
    """scene_extent_of (trainer.cpp:140-147): max distance from the centroid (>= 1e-9; 1 when empty)."""
    p = np.asarray(positions, np.float64).reshape(-1, 3)
    if p.shape[0] == 0:
        return 1.0
    return max(float(np.linalg.norm(p - p.mean(axis=0), axis=1).max()), 1e-9)


def frame_for_time(t: float, n_keyframes: int):
    """Keyframe segment and weight for normalised time t in [0, 1]: i = floor(t K),
    w = t K - i with K = n_keyframes - 1 (the trajectory lerp of trainer.cpp:259-279 /
    deform.cpp:248-251 between tick offsets)."""
    if n_keyframes < 2:
        return 0, 0.0
    K = n_keyframes - 1
    i = min(int(math.floor(t * K)), K - 1)
    return i, t * K - i


class Context:
    """One CUDA stream on one GPU (tsb_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().tsb_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return int(lib().tsb_ctx_stream(self._h) or 0)

    def synchronize(self):
        check(lib().tsb_ctx_synchronize(self._h))

    def join(self):
        """Make the context stream wait for all work enqueued on this context's passes."""
        check(lib().tsb_ctx_join(self._h))

    def launch_count(self) -> int:
        return int(lib().tsb_ctx_launch_count(self._h))

    def redo_count(self) -> int:
        """Frames redone after a device-side abort (list overflow / long tie run)."""
        return int(lib().tsb_ctx_redo_count(self._h))

    def set_profiling(self, on: bool):
        check(lib().tsb_ctx_set_profiling(self._h, 1 if on else 0))

    def raster_counts(self):
        """(evaluations, contributions) of the forward raster since the last call (profiling mode)."""
        e, c = C.c_int64(), C.c_int64()
        check(lib().tsb_ctx_raster_counts(self._h, C.byref(e), C.byref(c)))
        return e.value, c.value

    def scan_counts(self):
        """(ranks, super-tile list entries) of the frames' orders since the last call (profiling mode)."""
        r, e = C.c_int64(), C.c_int64()
        check(lib().tsb_ctx_scan_counts(self._h, C.byref(r), C.byref(e)))
        return r.value, e.value

    def stage_times(self):
        """{stage: (ms_total, calls)} since the last call (synchronises)."""
        ms = (C.c_double * len(_abi.STAGES))()
        calls = (C.c_int64 * len(_abi.STAGES))()
        check(lib().tsb_ctx_stage_times(self._h, ms, calls))
        return {name: (ms[i], calls[i]) for i, name in enumerate(_abi.STAGES)}

    def close(self):
        if getattr(self, "_h", None):
            lib().tsb_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _f32(a, n, comps):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    if a.size != n * comps:
        raise RuntimeError(f"render: parameter count mismatch (expected {n}x{comps}, got {a.shape})")
    return a


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_abi._fp)


class GaussianScene:
    """Device-resident Gaussian parameters, gradients and Adam moments."""

    def __init__(self, ctx: Context, n: int, n_keyframes: int = 0, tof: Optional[ToFConfig] = None,
                 sh_degree: int = 0, color: bool = False):
        tof = tof or ToFConfig()
        d = _abi.SceneDesc()
        d.n, d.n_keyframes, d.sh_degree = int(n), int(n_keyframes), int(sh_degree)
        d.color = 1 if color else 0
        self.color = bool(color)
        fr = tof.frequencies
        d.n_freq = len(fr)
        for i, f in enumerate(fr):
            d.frequency[i] = float(f)
        d.source_intensity = float(tof.source_intensity)
        d.speed_of_light = float(tof.speed_of_light)
        h = C.c_void_p()
        check(lib().tsb_scene_create(ctx.handle, C.byref(d), C.byref(h)))
        self._h, self.ctx, self.n, self.n_keyframes, self.tof = h, ctx, int(n), int(n_keyframes), tof
        self.n_freq = d.n_freq

    @property
    def handle(self):
        return self._h

    def densify(self, scene_extent: float, grad_threshold: float = 5e-5, opacity_floor: float = 5e-3,
                split_scale_fraction: float = 0.01, split_shrink: float = 1.6, min_count: int = 16) -> int:
        """Densification surgery + Adam reindex on the device (trainer.cpp:385-470, DensifyConfig
        defaults trainer.hpp:68-78); returns the new Gaussian count."""
        cfg = _abi.DensifyConfigC(grad_threshold, opacity_floor, split_scale_fraction, split_shrink, min_count)
        n = C.c_int32()
        check(lib().tsb_scene_densify(self._h, C.byref(cfg), float(scene_extent), C.byref(n)))
        self.n = int(n.value)
        return self.n

    def set_params(self, position, log_scale, rotation, opacity_logit, reflectivity_dc, motion=None):
        """Host numpy arrays (float32 SoA: position (n,3), log_scale (n,3), rotation (n,4) wxyz,
        opacity_logit (n,), reflectivity_dc (n,), motion (n_keyframes, n, 3))."""
        n = self.n
        arrs = [_f32(position, n, 3), _f32(log_scale, n, 3), _f32(rotation, n, 4), _f32(opacity_logit, n, 1),
                _f32(reflectivity_dc, n, 1)]
        mo = None
        if motion is not None and self.n_keyframes > 0:
            mo = _f32(motion, n, 3 * self.n_keyframes)
        check(lib().tsb_scene_set_params(self._h, _abi.TSB_HOST, *[a.ctypes.data for a in arrs],
                                         mo.ctypes.data if mo is not None else None))

    def set_sh(self, refl_sh):
        """All 16 reflectivity SH coefficients per Gaussian, (n, 16) (sh_degree > 0)."""
        a = _f32(refl_sh, self.n, 16)
        check(lib().tsb_scene_set_sh(self._h, _abi.TSB_HOST, a.ctypes.data))

    def get_sh(self, grads: bool = False):
        out = np.zeros((self.n, 16), np.float32)
        check(lib().tsb_scene_get_sh(self._h, _ptr(out), 1 if grads else 0))
        return out

    def set_color(self, color_sh):
        """Colour SH per Gaussian, (n, 16, 3) -- Gaussian::color_sh, coefficient k of channel c
        at [i, k, c] (scene created with color=True)."""
        a = np.ascontiguousarray(np.asarray(color_sh, np.float32).reshape(self.n, 16, 3).transpose(0, 2, 1))
        check(lib().tsb_scene_set_color(self._h, _abi.TSB_HOST, a.ctypes.data))

    def get_color(self, grads: bool = False):
        """(n, 16, 3) colour SH parameters, or SceneGrads::d_color_sh when grads."""
        out = np.zeros((self.n, 3, 16), np.float32)
        check(lib().tsb_scene_get_color(self._h, _ptr(out), 1 if grads else 0))
        return out.transpose(0, 2, 1).copy()

    def set_params_device(self, position, log_scale, rotation, opacity_logit, reflectivity_dc, motion=None):
        """Device pointers (ints) in the same SoA layout."""
        check(lib().tsb_scene_set_params(self._h, _abi.TSB_DEVICE, position, log_scale, rotation, opacity_logit,
                                         reflectivity_dc, motion))

    def get_params(self):
        n, k = self.n, self.n_keyframes
        out = {"position": np.zeros((n, 3), np.float32), "log_scale": np.zeros((n, 3), np.float32),
               "rotation": np.zeros((n, 4), np.float32), "opacity_logit": np.zeros(n, np.float32),
               "reflectivity_dc": np.zeros(n, np.float32), "motion": np.zeros((k, n, 3), np.float32)}
        check(lib().tsb_scene_get_params(self._h, _ptr(out["position"]), _ptr(out["log_scale"]),
                                         _ptr(out["rotation"]), _ptr(out["opacity_logit"]),
                                         _ptr(out["reflectivity_dc"]), _ptr(out["motion"]) if k else None))
        return out

    def grads(self):
        """Accumulated GroupGrads (+ d_bg_quad, loss sum)."""
        n, k = self.n, self.n_keyframes
        g = {"d_position": np.zeros((n, 3), np.float32), "d_log_scale": np.zeros((n, 3), np.float32),
             "d_rotation": np.zeros((n, 4), np.float32), "d_opacity_logit": np.zeros(n, np.float32),
             "d_reflectivity_dc": np.zeros(n, np.float32), "d_motion": np.zeros((k, n, 3), np.float32),
             "d_bg_quad": np.zeros(8), }
        loss = C.c_double()
        check(lib().tsb_scene_get_grads(self._h, _ptr(g["d_position"]), _ptr(g["d_log_scale"]),
                                        _ptr(g["d_rotation"]), _ptr(g["d_opacity_logit"]),
                                        _ptr(g["d_reflectivity_dc"]), _ptr(g["d_motion"]) if k else None,
                                        g["d_bg_quad"].ctypes.data_as(_abi._dp), C.byref(loss)))
        g["d_bg_quad"] = g["d_bg_quad"][: 4 * self.n_freq]
        g["loss"] = loss.value
        bq, bp = np.zeros(8), np.zeros(4)
        check(lib().tsb_scene_get_bg_grads(self._h, bq.ctypes.data_as(_abi._dp), bp.ctypes.data_as(_abi._dp)))
        g["d_bg_phasor"] = bp[: 2 * self.n_freq]
        bc = np.zeros(3)
        check(lib().tsb_scene_get_bg_color_grad(self._h, bc.ctypes.data_as(_abi._dp)))
        g["d_bg_color"] = bc
        return g

    def zero_grads(self):
        check(lib().tsb_scene_zero_grads(self._h))

    def adam_step(self, lr: LrTable, adam: AdamParams = AdamParams()):
        cfg = _abi.AdamConfig(lr.position, lr.log_scale, lr.rotation, lr.opacity, lr.reflectivity, lr.motion,
                              adam.beta1, adam.beta2, adam.eps, lr.color)
        check(lib().tsb_scene_adam_step(self._h, C.byref(cfg)))

    def adam_moments_position(self):
        m = np.zeros((self.n, 3), np.float32)
        v = np.zeros((self.n, 3), np.float32)
        check(lib().tsb_scene_get_adam_state(self._h, _ptr(m), _ptr(v)))
        return m, v

    def densify_stat(self):
        s = np.zeros(self.n, np.float32)
        c = C.c_int64()
        check(lib().tsb_scene_get_densify_stat(self._h, _ptr(s), C.byref(c)))
        return s, c.value

    def allreduce_grads(self, comm: "Comm"):
        check(lib().tsb_scene_allreduce_grads(self._h, comm.handle))

    def close(self):
        # after the context is gone (interpreter teardown, GC cycles) the handle is dropped, not freed
        if getattr(self, "_h", None) and getattr(getattr(self, "ctx", None), "_h", None):
            lib().tsb_scene_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RenderPass:
    """Reusable per-frame workspace; ``prepare`` is the reference RenderPass ctor
    (prepare + depth sort + build_tiles, splat.cpp:90-200)."""

    def __init__(self, ctx: Context):
        h = C.c_void_p()
        check(lib().tsb_pass_create(ctx.handle, C.byref(h)))
        self._h, self.ctx = h, ctx
        self.scene = None
        self.camera = None

    @property
    def handle(self):
        return self._h

    def prepare(self, scene: GaussianScene, camera: CameraModel, options: Optional[RenderOptions] = None,
                frame=None):
        options = options or RenderOptions()
        cam = camera.to_abi() if hasattr(camera, "to_abi") else camera
        fr = None
        if frame is not None:
            fr = _abi.Frame()
            fr.key, fr.w = int(frame[0]), float(frame[1])
        self._cam, self._opt = cam, options.to_abi()
        check(lib().tsb_pass_prepare(self._h, scene.handle, C.byref(self._cam), C.byref(self._opt),
                                     C.byref(fr) if fr is not None else None))
        self.scene, self.camera, self.options = scene, camera, options
        return self

    def visible_count(self) -> int:
        v = C.c_int32()
        check(lib().tsb_pass_visible_count(self._h, C.byref(v)))
        return v.value

    def num_keys(self) -> int:
        v = C.c_int64()
        check(lib().tsb_pass_num_keys(self._h, C.byref(v)))
        return v.value

    def forward(self):
        check(lib().tsb_pass_forward(self._h))
        return self

    def forward_loss(self, target, channel_weight=None, sync=True, device_ptr=None, ssim_mix: float = 0.0):
        """Forward + the trainer's image loss per quad channel, sum_c w_c [(1 - ssim_mix) mse_c +
        ssim_mix (1 - SSIM_c)] (losses.cpp:148-166; weight quad/4 per channel, trainer.cpp:210-219;
        ssim_mix 0 = pure L2, fused into the raster epilogue).  target: host array
        (4*n_freq, H, W) or a device pointer."""
        nf = self.scene.n_freq
        if channel_weight is None:
            channel_weight = [0.25] * (4 * nf)
        w = (C.c_double * 8)(*([float(x) for x in channel_weight] + [0.0] * (8 - len(channel_weight))))
        loss = C.c_double()
        if device_ptr is not None:
            check(lib().tsb_pass_forward_image_loss(self._h, _abi.TSB_DEVICE, C.c_void_p(device_ptr), w,
                                                    float(ssim_mix), C.byref(loss) if sync else None))
        else:
            t = np.ascontiguousarray(np.asarray(target, dtype=np.float32))
            self._target_keep = t
            check(lib().tsb_pass_forward_image_loss(self._h, _abi.TSB_HOST, t.ctypes.data, w, float(ssim_mix),
                                                    C.byref(loss) if sync else None))
        return loss.value if sync else None

    def backward(self, d_quad=None, device_ptr=None):
        """Accumulate gradients into the scene (uses the loss residual when d_quad is None)."""
        if device_ptr is not None:
            check(lib().tsb_pass_backward(self._h, _abi.TSB_DEVICE, C.c_void_p(device_ptr)))
        elif d_quad is not None:
            up = np.ascontiguousarray(np.asarray(d_quad, dtype=np.float32))
            self._up_keep = up
            check(lib().tsb_pass_backward(self._h, _abi.TSB_HOST, up.ctypes.data))
        else:
            check(lib().tsb_pass_backward(self._h, _abi.TSB_HOST, None))
        return self

    def backward_ext(self, **upstreams):
        """RenderPass::backward(BufferGrads) with any of the BufferGrads images (alias of
        backward_buffers, whose keyword names it takes)."""
        return self.backward_buffers(**upstreams)

    def backward_buffers(self, d_quad=None, d_phasor=None, d_depth_raw=None, d_weight=None,
                         d_distortion=None, d_transmittance=None, d_color=None, d_motion_fwd_acc=None,
                         d_motion_bwd_acc=None):
        """RenderPass::backward(BufferGrads) (splat.cpp:347-650): None skips a channel."""
        keep = []

        def arr(a):
            if a is None:
                return None
            a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
            keep.append(a)
            return a.ctypes.data

        ptrs = [arr(a) for a in (d_quad, d_phasor, d_depth_raw, d_weight, d_distortion, d_transmittance,
                                 d_color, d_motion_fwd_acc, d_motion_bwd_acc)]
        self._up_keep = keep
        check(lib().tsb_pass_backward_ext(self._h, _abi.TSB_HOST, *ptrs))
        return self

    def set_motion(self, motion_fwd=None, motion_bwd=None):
        """RenderInput::motion_fwd / motion_bwd (splat.hpp:46-47): (n, 3) per-Gaussian motions of
        this frame for the flow channel; None = zero.  Call after prepare()."""
        n = self.scene.n
        a = None if motion_fwd is None else _f32(motion_fwd, n, 3)
        b = None if motion_bwd is None else _f32(motion_bwd, n, 3)
        check(lib().tsb_pass_set_motion(self._h, _abi.TSB_HOST, a.ctypes.data if a is not None else None,
                                        b.ctypes.data if b is not None else None))
        return self

    def flow_loss(self, target_fwd=None, target_bwd=None, weight: float = 1.0):
        """flow_loss (losses.cpp:168-251) of the last forward (flow channel): targets (3, H, W) =
        (u, v, valid) or None.  Returns (value, valid_pixels); the motion-accumulator gradients
        (x weight) stay on the device for backward_flow()."""
        H, W = self.camera.height, self.camera.width
        keep = []

        def arr(a):
            if a is None:
                return None
            a = np.ascontiguousarray(np.asarray(a, np.float32))
            if a.shape != (3, H, W):
                raise RuntimeError("flow_loss: target shape mismatch")
            keep.append(a)
            return a.ctypes.data

        v, n, g = C.c_double(), C.c_int64(), C.c_int32()
        check(lib().tsb_pass_flow_loss(self._h, _abi.TSB_HOST, arr(target_fwd), arr(target_bwd), float(weight),
                                       C.byref(v), C.byref(n), C.byref(g)))
        self._flow_grads = g.value
        return v.value, n.value

    def flow_loss_grads(self):
        """(d_motion_fwd_acc, d_motion_bwd_acc) of the last flow_loss, (3, H, W) or None."""
        H, W = self.camera.height, self.camera.width
        g = getattr(self, "_flow_grads", 0)
        return tuple(self.download(w, shape=(3, H, W)) if g & (1 << k) else None
                     for k, w in enumerate((_abi.OUT_D_MOTION_FWD_ACC, _abi.OUT_D_MOTION_BWD_ACC)))

    def backward_flow(self, with_image_loss: bool = True):
        """Backward of the trainer's combined loss for this frame: the image-loss residual (the
        forward_loss d_quad, when with_image_loss) + the flow-loss motion upstreams, all on the
        device (trainer.cpp:296-310)."""
        g = getattr(self, "_flow_grads", 0)
        ptr = lambda w: C.c_void_p(self.output_ptr(w)[0])
        dq = ptr(_abi.OUT_D_QUAD) if with_image_loss else None
        mf = ptr(_abi.OUT_D_MOTION_FWD_ACC) if g & 1 else None
        mb = ptr(_abi.OUT_D_MOTION_BWD_ACC) if g & 2 else None
        check(lib().tsb_pass_backward_ext(self._h, _abi.TSB_DEVICE, dq, None, None, None, None, None, None, mf, mb))
        return self

    def write_render_stack(self, directory, quartet: int):
        """One render stack of write_render_stacks (eval.cpp:96-121, 165-185) from the last forward
        (options.distortion required; colour written when options.color): quad planes, gated
        depth, d_ToF, distortion (and colour) as PFM files named as the reference names them."""
        check(lib().tsb_pass_render_stack(self._h, str(directory).encode(), int(quartet)))
        return self

    def motion_grads(self):
        """SceneGrads::d_motion_fwd / d_motion_bwd of the last backward, (n, 3) each."""
        n = self.scene.n
        a, b = np.zeros((n, 3), np.float32), np.zeros((n, 3), np.float32)
        check(lib().tsb_pass_get_motion_grads(self._h, _ptr(a), _ptr(b)))
        return a, b

    def output_ptr(self, which: int):
        p = C.c_void_p()
        nb = C.c_size_t()
        check(lib().tsb_pass_output(self._h, which, C.byref(p), C.byref(nb)))
        return p.value, nb.value

    def download(self, which: int, dtype=np.float32, shape=None):
        _, nb = self.output_ptr(which)
        a = np.empty(nb // np.dtype(dtype).itemsize, dtype=dtype)
        check(lib().tsb_pass_download(self._h, which, a.ctypes.data, nb))
        return a.reshape(shape) if shape is not None else a

    def download_async(self, which: int, host: np.ndarray):
        """Enqueue a device->host copy of output `which` into `host` (ideally pinned);
        valid after wait() / Context.synchronize() (prepare() of the next frame does not wait for it)."""
        check(lib().tsb_pass_download_async(self._h, which, host.ctypes.data, host.nbytes))
        return self

    def wait(self):
        check(lib().tsb_pass_wait(self._h))
        return self

    def outputs(self):
        """RenderedBuffers (splat.hpp:51-66), ToF channels: quad, phasor, depth_raw, depth, weight,
        transmittance (+ distortion when enabled)."""
        H, W, nf = self.camera.height, self.camera.width, self.scene.n_freq
        out = {"quad": self.download(_abi.OUT_QUAD, shape=(4 * nf, H, W)),
               "depth_raw": self.download(_abi.OUT_DEPTH_RAW, shape=(H, W)),
               "depth": self.download(_abi.OUT_DEPTH, shape=(H, W)),
               "weight": self.download(_abi.OUT_WEIGHT, shape=(H, W)),
               "transmittance": self.download(_abi.OUT_TRANSM, shape=(H, W)),
               "phasor": self.download(_abi.OUT_PHASOR, shape=(2 * nf, H, W))}
        if self.options.distortion:
            out["distortion"] = self.download(_abi.OUT_DISTORTION, shape=(H, W))
        if self.options.color:
            out["color"] = self.download(_abi.OUT_COLOR, shape=(3, H, W))
        if self.options.flow:
            out["motion_fwd_acc"] = self.download(_abi.OUT_MOTION_FWD_ACC, shape=(3, H, W))
            out["motion_bwd_acc"] = self.download(_abi.OUT_MOTION_BWD_ACC, shape=(3, H, W))
            out["flow_fwd"] = self.download(_abi.OUT_FLOW_FWD, shape=(2, H, W))
            out["flow_bwd"] = self.download(_abi.OUT_FLOW_BWD, shape=(2, H, W))
            out["flow_valid"] = self.download(_abi.OUT_FLOW_VALID, shape=(2, H, W))
        if self.options.exact:
            out["f64"] = self.download(_abi.OUT_F64, np.float64, (6 * nf + 5, H, W))
            if self.options.color or self.options.flow:
                out["ext_f64"] = self.download(_abi.OUT_EXT_F64, np.float64, (9, H, W))
        if self.options.counts:
            out["n_contrib"] = self.download(_abi.OUT_N_CONTRIB, np.int32, (H, W))
            out["n_processed"] = self.download(_abi.OUT_N_PROCESSED, np.int32, (H, W))
        return out

    # ---- parity diagnostics ----
    def debug_prepared(self):
        v = self.visible_count()
        g = np.zeros(max(v, 1), np.int32)
        r = np.zeros((max(v, 1), 4), np.int32)
        check(lib().tsb_pass_debug_prepared(self._h, g.ctypes.data_as(_abi._ip), r.ctypes.data_as(_abi._ip)))
        return {"gidx": g[:v], "rect": r[:v]}

    def debug_tiles(self):
        tx, ty = C.c_int32(), C.c_int32()
        check(lib().tsb_pass_debug_tiles(self._h, C.byref(tx), C.byref(ty), None, None))
        k = self.num_keys()
        off = np.zeros(tx.value * ty.value + 1, np.int64)
        ids = np.zeros(max(k, 1), np.int32)
        check(lib().tsb_pass_debug_tiles(self._h, None, None, off.ctypes.data_as(_abi._lp),
                                         ids.ctypes.data_as(_abi._ip)))
        return off, ids[:k]

    def debug_records(self):
        v = self.visible_count()
        r = np.zeros((max(v, 1), 12), np.float32)
        check(lib().tsb_pass_debug_records(self._h, _ptr(r)))
        return r[:v]

    def debug_keep_screen(self, enabled: bool = True):
        """Keep a copy of every following backward's screen-space gradients (the chain
        kernel consumes them); needed before debug_screen_grads."""
        check(lib().tsb_pass_debug_keep_screen(self._h, 1 if enabled else 0))
        return self

    def debug_screen_grads(self):
        """Per-rank screen-space gradients of the last backward (d_mean2d x/y, d_conic a/b/c,
        d_opacity, d_coef, d_depth), in prepared (rank) order."""
        v = self.visible_count()
        g = np.zeros((max(v, 1), 8), np.float32)
        check(lib().tsb_pass_debug_screen_grads(self._h, _ptr(g)))
        return g[:v]

    def debug_set_list_capacity(self, entries: int):
        """Test hook (call between prepare and forward): shrink the tile-list storage so the
        frame overflows and takes the device-side abort + redo path."""
        check(lib().tsb_pass_debug_set_list_capacity(self._h, int(entries)))
        return self

    def debug_fixups(self) -> int:
        c = C.c_int32()
        check(lib().tsb_pass_debug_fixups(self._h, C.byref(c)))
        return c.value

    def debug_fixup_list(self):
        """(pixel index, reason bits) of the pixels recomposited in fp64."""
        n = self.debug_fixups()
        a = np.zeros(max(n, 1), np.int32)
        c = C.c_int32()
        check(lib().tsb_pass_debug_fixup_list(self._h, a.ctypes.data_as(_abi._ip), int(a.size), C.byref(c)))
        a = a[:n]
        return a & 0xFFFFFF, (a >> 24) & 31  # reasons: 1 maha, 2 alpha, 4 T band, 8 T error bound, 16 exact mode

    def close(self):
        # after the context is gone (interpreter teardown, GC cycles) the handle is dropped, not freed
        if getattr(self, "_h", None) and getattr(getattr(self, "ctx", None), "_h", None):
            lib().tsb_pass_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Comm:
    """NCCL communicator for frame-sharded data parallelism (tsb_comm)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_char * 128)()
        check(lib().tsb_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, ctx: Context, uid: bytes, nranks: int, rank: int):
        h = C.c_void_p()
        buf = (C.c_char * 128).from_buffer_copy(uid)
        check(lib().tsb_comm_create(ctx.handle, buf, int(nranks), int(rank), C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().tsb_comm_destroy(self._h)
            self._h = None


# ---- Python _core surface (bindings.cpp:43-63) ----
def write_pfm(path, img) -> None:
    """write_pfm (pfm.cpp:51-75): planar (C, H, W) or (H, W) float image, C in {1, 3}."""
    a = np.ascontiguousarray(np.asarray(img, np.float32))
    if a.ndim == 2:
        a = a[None]
    c, h, w = a.shape
    check(lib().tsb_write_pfm(str(path).encode(), a.ctypes.data, w, h, c))


def read_pfm(path) -> np.ndarray:
    """read_pfm (pfm.cpp:77-114) -> planar (C, H, W) float32."""
    w, h, c = C.c_int32(), C.c_int32(), C.c_int32()
    p = str(path).encode()
    check(lib().tsb_read_pfm(p, None, 0, C.byref(w), C.byref(h), C.byref(c)))
    out = np.empty((c.value, h.value, w.value), np.float32)
    check(lib().tsb_read_pfm(p, out.ctypes.data, out.size, C.byref(w), C.byref(h), C.byref(c)))
    return out


def unambiguous_range(frequency: float = 0.0) -> float:
    return float(lib().tsb_unambiguous_range(float(frequency)))


def quad_to_depth(q0, q90, q180, q270, frequency: float = 0.0) -> float:
    return float(lib().tsb_quad_to_depth(float(q0), float(q90), float(q180), float(q270), float(frequency)))


def quad_basis(depth: float, frequency: float = 0.0):
    out = (C.c_double * 4)()
    lib().tsb_quad_basis(float(depth), float(frequency), out)
    return list(out)


class DeformNet:
    """The reference's DeformNet (deform.hpp:19-66) on the tensor cores: positional
    encodings -> `hidden_layers` ReLU layers -> 3 offsets; each layer a tcgen05 GEMM
    (3xTF32).  Parameters are the flat get_parameters order (W row-major, then b)."""

    def __init__(self, ctx: Context, hidden_layers: int = 4, width: int = 128, l_x: int = 10, l_t: int = 10,
                 coord_scale: float = 1.0):
        self.ctx = ctx
        cfg = _abi.DeformConfigC(hidden_layers, width, l_x, l_t, coord_scale)
        h = C.c_void_p()
        check(lib().tsb_deform_create(ctx.handle, C.byref(cfg), C.byref(h)))
        self._h = h
        self.hidden_layers, self.width, self.l_x, self.l_t, self.coord_scale = hidden_layers, width, l_x, l_t, \
            coord_scale

    @property
    def handle(self):
        return self._h

    @property
    def input_dim(self) -> int:
        return 3 * (1 + 2 * self.l_x) + 1 + 2 * self.l_t

    @property
    def parameter_count(self) -> int:
        return int(lib().tsb_deform_param_count(self._h))

    def set_parameters(self, flat):
        a = np.ascontiguousarray(flat, np.float32)
        if a.size != self.parameter_count:
            raise ValueError("DeformNet::set_parameters: size mismatch")
        check(lib().tsb_deform_set_params(self._h, _abi.TSB_HOST, a.ctypes.data))

    def get_parameters(self) -> np.ndarray:
        out = np.empty(self.parameter_count, np.float32)
        check(lib().tsb_deform_get_params(self._h, out.ctypes.data))
        return out

    def grads(self) -> np.ndarray:
        out = np.empty(self.parameter_count, np.float32)
        check(lib().tsb_deform_get_grads(self._h, out.ctypes.data))
        return out

    def zero_grads(self):
        check(lib().tsb_deform_zero_grads(self._h))

    def offsets(self, positions, t: float, slot: int = 0) -> np.ndarray:
        """positions (n, 3) -> offsets (n, 3); caches the forward in `slot` for backward()."""
        p = np.ascontiguousarray(positions, np.float32).reshape(-1, 3)
        out = np.empty_like(p)
        check(lib().tsb_deform_offsets(self._h, slot, _abi.TSB_HOST, p.ctypes.data, p.shape[0], float(t),
                                       out.ctypes.data))
        return out

    def backward(self, d_offsets, slot: int = 0, want_positions: bool = True):
        """Accumulates dW/db for the slot's forward; returns d(positions) (n, 3) or None."""
        d = np.ascontiguousarray(d_offsets, np.float32).reshape(-1, 3)
        dp = np.empty_like(d) if want_positions else None
        check(lib().tsb_deform_backward(self._h, slot, _abi.TSB_HOST, d.ctypes.data,
                                        dp.ctypes.data if want_positions else None))
        return dp

    def scene_offsets(self, scene: "GaussianScene", keyframe: int, t: float, slot: int = 0):
        check(lib().tsb_deform_scene_offsets(self._h, slot, scene.handle, keyframe, float(t)))

    def scene_backward(self, scene: "GaussianScene", keyframe: int, slot: int = 0):
        check(lib().tsb_deform_scene_backward(self._h, slot, scene.handle, keyframe))

    def debug_activation(self, layer: int, n: int, slot: int = 0) -> np.ndarray:
        out = np.empty((n, self.width), np.float32)
        check(lib().tsb_deform_debug_activation(self._h, slot, layer, out.ctypes.data))
        return out

    def adam_step(self, lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-15):
        check(lib().tsb_deform_adam_step(self._h, lr, beta1, beta2, eps))

    def close(self):
        # after the context is gone (interpreter teardown, GC cycles) the handle is dropped, not freed
        if getattr(self, "_h", None) and getattr(getattr(self, "ctx", None), "_h", None):
            lib().tsb_deform_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
