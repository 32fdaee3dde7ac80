"""ctypes wrapper of the CPU oracle (oracle/tofsplat_oracle.c).

TEST INFRASTRUCTURE ONLY -- the parity checker for the B200 path and the
"port" CPU baseline of bench.py.  Only tests/, __graft_entry__.smoke() and
bench.py's CPU legs may import this module; the product package
(paper_2505_05356_b200) never does.

Everything here is double precision and mirrors the reference's
RenderPass / mse / AdamState semantics (see tofsplat_oracle.h for citations).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "liboracle.so"


def build() -> Path:
    subprocess.run(["make", "-C", str(_HERE)], check=True, stdout=subprocess.DEVNULL)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = C.CDLL(str(_LIB_PATH))
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int32)
        lp = C.POINTER(C.c_int64)
        L.orc_last_error.restype = C.c_char_p
        L.orc_pass_create.restype = C.c_void_p
        L.orc_pass_create.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_pass_destroy.argtypes = [C.c_void_p]
        L.orc_pass_visible_count.argtypes = [C.c_void_p]
        L.orc_pass_tiles.argtypes = [C.c_void_p, ip, ip]
        L.orc_pass_num_keys.argtypes = [C.c_void_p]
        L.orc_pass_num_keys.restype = C.c_int64
        L.orc_pass_prepared.argtypes = [C.c_void_p, ip, ip, dp]
        L.orc_pass_tile_lists.argtypes = [C.c_void_p, lp, ip]
        L.orc_pass_forward.argtypes = [C.c_void_p] + [dp] * 7 + [ip, ip]
        L.orc_pass_backward.argtypes = [C.c_void_p] + [dp] * 14
        L.orc_pass_forward_ext.argtypes = [C.c_void_p] + [dp] * 6
        L.orc_pass_backward_ext.argtypes = [C.c_void_p] + [dp] * 21
        L.orc_mse.restype = C.c_double
        L.orc_mse.argtypes = [dp, dp, C.c_size_t, dp]
        L.orc_adam_step.argtypes = [dp, dp, dp, dp, C.c_size_t, C.c_int64, C.c_double, C.c_double,
                                    C.c_double, C.c_double]
        L.orc_interp_positions.argtypes = [dp, dp, dp, C.c_double, C.c_size_t, dp]
        L.orc_quat_to_rotation.argtypes = [dp, dp]
        L.orc_sh_basis.argtypes = [dp, C.c_int, dp]
        L.orc_sh_basis_jacobian.argtypes = [dp, C.c_int, dp]
        L.orc_num_threads.restype = C.c_int
        L.orc_set_num_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


class _Camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("near_plane", C.c_double),
                ("far_plane", C.c_double), ("R", C.c_double * 9), ("t", C.c_double * 3)]


class _Options(C.Structure):
    _fields_ = [("alpha_threshold", C.c_double), ("transmittance_floor", C.c_double),
                ("dilation", C.c_double), ("sigma_cutoff", C.c_double), ("coverage_eps", C.c_double),
                ("tile_size", C.c_int32), ("_pad", C.c_int32), ("bg_quad", C.c_double * 4),
                ("bg_phasor", C.c_double * 2), ("bg_color", C.c_double * 3)]


class _Scene(C.Structure):
    _fields_ = [("n", C.c_int32), ("sh_degree", C.c_int32), ("modulation_frequency", C.c_double),
                ("source_intensity", C.c_double), ("speed_of_light", C.c_double),
                ("position", C.c_void_p), ("log_scale", C.c_void_p), ("rotation", C.c_void_p),
                ("opacity_logit", C.c_void_p), ("refl_sh", C.c_void_p), ("color_sh", C.c_void_p),
                ("motion_fwd", C.c_void_p), ("motion_bwd", C.c_void_p)]


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int32))


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


@dataclass
class OScene:
    """Gaussian parameters (reference Gaussian fields, SoA, double)."""
    position: np.ndarray          # (n, 3) rendered means
    log_scale: np.ndarray         # (n, 3)
    rotation: np.ndarray          # (n, 4) (w, x, y, z)
    opacity_logit: np.ndarray     # (n,)
    refl_sh: np.ndarray           # (n, 16)
    sh_degree: int = 0
    modulation_frequency: float = 29.9792458e6
    source_intensity: float = 1.0
    speed_of_light: float = 299792458.0
    color_sh: Optional[np.ndarray] = None    # (n, 48): [16 c + k] = Gaussian::color_sh(k, c)
    motion_fwd: Optional[np.ndarray] = None  # (n, 3) RenderInput::motion_fwd
    motion_bwd: Optional[np.ndarray] = None

    @property
    def n(self):
        return int(self.position.shape[0])


def scene_from_dc(position, log_scale, rotation, opacity_logit, reflectivity_dc, *, frequency=29.9792458e6,
                  source_intensity=1.0, speed_of_light=299792458.0):
    n = len(opacity_logit)
    refl = np.zeros((n, 16))
    refl[:, 0] = np.asarray(reflectivity_dc, dtype=np.float64)
    return OScene(_f64(position, (n, 3)), _f64(log_scale, (n, 3)), _f64(rotation, (n, 4)),
                  _f64(opacity_logit, (n,)), refl, 0, frequency, source_intensity, speed_of_light)


def _camera(cam) -> _Camera:
    c = _Camera()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    c.near_plane = float(getattr(cam, "near_plane", 0.2))
    c.far_plane = float(getattr(cam, "far_plane", 100.0))
    R = np.asarray(getattr(cam, "rotation", np.eye(3)), dtype=np.float64).reshape(9)
    t = np.asarray(getattr(cam, "translation", np.zeros(3)), dtype=np.float64).reshape(3)
    for i in range(9):
        c.R[i] = R[i]
    for i in range(3):
        c.t[i] = t[i]
    return c


def _options(opt) -> _Options:
    o = _Options()
    o.alpha_threshold = float(getattr(opt, "alpha_threshold", 1.0 / 255.0))
    o.transmittance_floor = float(getattr(opt, "transmittance_floor", 1e-4))
    o.dilation = float(getattr(opt, "dilation", 0.3))
    o.sigma_cutoff = float(getattr(opt, "sigma_cutoff", 3.0))
    o.coverage_eps = float(getattr(opt, "coverage_eps", 1e-12))
    o.tile_size = int(getattr(opt, "tile_size", 16))
    bq = np.zeros(4)
    b = np.asarray(getattr(opt, "bg_quad", np.zeros(4)), dtype=np.float64).reshape(-1)
    bq[: min(4, b.size)] = b[:4]
    for i in range(4):
        o.bg_quad[i] = bq[i]
    bp = np.asarray(getattr(opt, "bg_phasor", np.zeros(2)), dtype=np.float64).reshape(-1)
    for i in range(2):
        o.bg_phasor[i] = bp[i] if bp.size > i else 0.0
    bc = np.asarray(getattr(opt, "bg_color", np.zeros(3)), dtype=np.float64).reshape(-1)
    for i in range(3):
        o.bg_color[i] = bc[i] if bc.size > i else 0.0
    return o


class OraclePass:
    """RenderPass restated on the CPU (splat.cpp:83-650)."""

    def __init__(self, scene: OScene, camera, options):
        L = lib()
        self.scene = scene
        self._keep = [_f64(scene.position, (scene.n, 3)), _f64(scene.log_scale, (scene.n, 3)),
                      _f64(scene.rotation, (scene.n, 4)), _f64(scene.opacity_logit, (scene.n,)),
                      _f64(scene.refl_sh, (scene.n, 16))]
        s = _Scene()
        s.n = scene.n
        s.sh_degree = scene.sh_degree
        s.modulation_frequency = scene.modulation_frequency
        s.source_intensity = scene.source_intensity
        s.speed_of_light = scene.speed_of_light
        s.position, s.log_scale, s.rotation, s.opacity_logit, s.refl_sh = [a.ctypes.data for a in self._keep]
        for name, comps in (("color_sh", 48), ("motion_fwd", 3), ("motion_bwd", 3)):
            a = getattr(scene, name, None)
            if a is not None:
                a = _f64(a, (scene.n, comps))
                self._keep.append(a)
                setattr(s, name, a.ctypes.data)
        self._s, self._c, self._o = s, _camera(camera), _options(options)
        self.width, self.height = int(camera.width), int(camera.height)
        h = L.orc_pass_create(C.byref(self._s), C.byref(self._c), C.byref(self._o))
        if not h:
            raise RuntimeError(L.orc_last_error().decode())
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_pass_destroy(h)
            self._h = None

    def visible_count(self) -> int:
        return int(lib().orc_pass_visible_count(self._h))

    def tiles(self):
        tx, ty = C.c_int32(), C.c_int32()
        lib().orc_pass_tiles(self._h, C.byref(tx), C.byref(ty))
        return tx.value, ty.value

    def num_keys(self) -> int:
        return int(lib().orc_pass_num_keys(self._h))

    def prepared(self):
        v = self.visible_count()
        g = np.zeros(max(v, 1), np.int32)
        r = np.zeros((max(v, 1), 4), np.int32)
        rec = np.zeros((max(v, 1), 10), np.float64)
        lib().orc_pass_prepared(self._h, _ip(g), _ip(r), _dp(rec))
        return {"gidx": g[:v], "rect": r[:v], "rec": rec[:v]}

    def tile_lists(self):
        tx, ty = self.tiles()
        off = np.zeros(tx * ty + 1, np.int64)
        ids = np.zeros(max(self.num_keys(), 1), np.int32)
        lib().orc_pass_tile_lists(self._h, off.ctypes.data_as(C.POINTER(C.c_int64)), _ip(ids))
        return off, ids[: self.num_keys()]

    def forward(self):
        W, H = self.width, self.height
        out = {k: np.zeros((c, H, W)) for k, c in
               [("quad", 4), ("phasor", 2), ("depth_raw", 1), ("depth", 1), ("weight", 1),
                ("transmittance", 1), ("distortion", 1)]}
        nc = np.zeros((H, W), np.int32)
        npr = np.zeros((H, W), np.int32)
        lib().orc_pass_forward(self._h, _dp(out["quad"]), _dp(out["phasor"]), _dp(out["depth_raw"]),
                               _dp(out["depth"]), _dp(out["weight"]), _dp(out["transmittance"]),
                               _dp(out["distortion"]), _ip(nc), _ip(npr))
        for k in ("depth_raw", "depth", "weight", "transmittance", "distortion"):
            out[k] = out[k][0]
        out["n_contrib"] = nc
        out["n_processed"] = npr
        return out

    def forward_ext(self):
        """Colour and flow channels (splat.cpp:273-294, 301-334)."""
        W, H = self.width, self.height
        out = {k: np.zeros((c, H, W)) for k, c in
               [("color", 3), ("motion_fwd_acc", 3), ("motion_bwd_acc", 3), ("flow_fwd", 2), ("flow_bwd", 2),
                ("flow_valid", 2)]}
        lib().orc_pass_forward_ext(self._h, *[_dp(out[k]) for k in ("color", "motion_fwd_acc", "motion_bwd_acc",
                                                                     "flow_fwd", "flow_bwd", "flow_valid")])
        return out

    def backward(self, d_quad=None, d_phasor=None, d_depth_raw=None, d_weight=None, d_distortion=None,
                 d_transmittance=None, d_color=None, d_motion_fwd_acc=None, d_motion_bwd_acc=None):
        n, v = self.scene.n, self.visible_count()
        W, H = self.width, self.height

        def up(a, c):
            return None if a is None else _f64(a, (c, H, W))

        ups = [up(d_quad, 4), up(d_phasor, 2), up(d_depth_raw, 1), up(d_weight, 1), up(d_distortion, 1),
               up(d_transmittance, 1), up(d_color, 3), up(d_motion_fwd_acc, 3), up(d_motion_bwd_acc, 3)]
        g = {"d_position": np.zeros((n, 3)), "d_log_scale": np.zeros((n, 3)), "d_rotation": np.zeros((n, 4)),
             "d_opacity_logit": np.zeros(n), "d_refl_sh": np.zeros((n, 16)), "d_bg_quad": np.zeros(4),
             "d_bg_phasor": np.zeros(2), "d_color_sh": np.zeros((n, 48)), "d_motion_fwd": np.zeros((n, 3)),
             "d_motion_bwd": np.zeros((n, 3)), "d_bg_color": np.zeros(3), "screen": np.zeros((max(v, 1), 8))}
        lib().orc_pass_backward_ext(self._h, *[_dp(a) for a in ups], _dp(g["d_position"]), _dp(g["d_log_scale"]),
                                    _dp(g["d_rotation"]), _dp(g["d_opacity_logit"]), _dp(g["d_refl_sh"]),
                                    _dp(g["d_bg_quad"]), _dp(g["d_bg_phasor"]), _dp(g["d_color_sh"]),
                                    _dp(g["d_motion_fwd"]), _dp(g["d_motion_bwd"]), _dp(g["d_bg_color"]),
                                    _dp(g["screen"]))
        g["screen"] = g["screen"][:v]
        return g


def mse(pred, target, want_grad=True):
    p = _f64(pred).reshape(-1)
    t = _f64(target).reshape(-1)
    if p.size != t.size:
        raise RuntimeError("mse: shape mismatch")
    d = np.zeros_like(p) if want_grad else None
    v = lib().orc_mse(_dp(p), _dp(t), p.size, _dp(d))
    return (v, d.reshape(np.shape(pred))) if want_grad else v


def adam_step(params, grads, m, v, t, lr, beta1=0.9, beta2=0.999, eps=1e-15):
    """In place on float64 contiguous arrays (AdamState::step, trainer.cpp:18-31)."""
    for a in (params, grads, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    lib().orc_adam_step(_dp(params), _dp(grads), _dp(m), _dp(v), params.size, int(t), lr, beta1, beta2, eps)


def interp_positions(x, d_i, d_ip1, w):
    x, d_i, d_ip1 = _f64(x), _f64(d_i), _f64(d_ip1)
    out = np.zeros_like(x)
    lib().orc_interp_positions(_dp(x), _dp(d_i), _dp(d_ip1), float(w), x.size // 3, _dp(out))
    return out


def quat_to_rotation(q):
    q = _f64(q, (4,))
    R = np.zeros(9)
    lib().orc_quat_to_rotation(_dp(q), _dp(R))
    return R.reshape(3, 3)


def sh_basis(d, degree):
    d = _f64(d, (3,))
    b = np.zeros(16)
    lib().orc_sh_basis(_dp(d), int(degree), _dp(b))
    return b


def sh_basis_jacobian(d, degree):
    d = _f64(d, (3,))
    J = np.zeros(48)
    lib().orc_sh_basis_jacobian(_dp(d), int(degree), _dp(J))
    return J.reshape(16, 3)


def set_threads(n: int):
    lib().orc_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().orc_num_threads())
