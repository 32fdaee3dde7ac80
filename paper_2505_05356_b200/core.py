"""The reference's Python `_core` surface (proj/python/bindings.cpp:40-204,
proj/python/tofsplat/__init__.py:3-27) over the B200 path.

Same function names, argument names, defaults and return shapes as the pybind11
bindings, so the reference's own smoke tests (proj/tests/python/test_smoke.py) read
the same against it:

  unambiguous_range(frequency=0.0)                  bindings.cpp:43-47  (tof.hpp:36-38)
  quad_to_depth(q0, q90, q180, q270, frequency=0.0) bindings.cpp:49-56  (tof.hpp:59-65)
  quad_basis(depth, frequency=0.0)                  bindings.cpp:58-65  (tof.hpp:75-79)
  dataset_info(dataset_dir)                         bindings.cpp:90-104 (dataset.cpp:44-116)
  render_timestep(scene_path, deform_path, dataset_dir, timestep=0.0)
                                                    bindings.cpp:164-203
  gradcheck(seed=7, splats=4, width=8, height=8)    bindings.cpp:150-162 (gradcheck.cpp:155-247)

Every render runs on the GPU through libtsb.so (checkpoint deformation on the
tcgen05 DeformNet, preprocess / sort / binning / composite / backward in the
sm_100a kernels); this module only parses files and moves arrays.  The functions
outside the render/optimise path -- dataset simulation, the training driver and the
evaluation report (components 11, 14, 15) -- raise TsbError
(TSB_ERR_UNSUPPORTED) naming what they belong to.
"""
from __future__ import annotations

import json
import math
import struct
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Dict, List, Optional

import numpy as np

from . import _abi
from ._abi import TsbError
from .render import (CameraModel, Context, DeformNet, GaussianScene, RenderOptions, RenderPass, ToFConfig,
                     quad_basis as _quad_basis, quad_to_depth as _quad_to_depth,
                     unambiguous_range as _unambiguous_range, read_pfm)

SH_C0 = 0.28209479177387814
GAUSSIAN_FLOATS = 75  # scene.hpp:40-42: position 3, log_scale 3, rotation 4, opacity 1, refl SH 16, colour SH 48

_CTX: Optional[Context] = None


def _context() -> Context:
    global _CTX
    if _CTX is None:
        _CTX = Context(0)
    return _CTX


# ---- tof.hpp helpers ---------------------------------------------------------------------
def unambiguous_range(frequency: float = 0.0) -> float:
    """Maximum depth before phase wraps, c / (2 f); frequency <= 0 uses the default sensor."""
    return _unambiguous_range(frequency)


def quad_to_depth(q0: float, q90: float, q180: float, q270: float, frequency: float = 0.0) -> float:
    """Depth decoded from one raw quartet sample (NaN if flat)."""
    return _quad_to_depth(q0, q90, q180, q270, frequency)


def quad_basis(depth: float, frequency: float = 0.0) -> List[float]:
    """The four phase-offset modulation values {sin, cos, -sin, -cos} at this depth."""
    return _quad_basis(depth, frequency)


# ---- scene / deformation checkpoints (scene.cpp:114-218, deform.cpp:189-246) -------------
@dataclass
class SceneCheckpoint:
    """CanonicalScene (scene.hpp:44-52) as float32 SoA."""
    position: np.ndarray      # (n, 3)
    log_scale: np.ndarray     # (n, 3)
    rotation: np.ndarray      # (n, 4) w, x, y, z
    opacity_logit: np.ndarray  # (n,)
    reflectivity_sh: np.ndarray  # (n, 16)
    color_sh: np.ndarray      # (n, 16, 3)
    sh_degree: int = 3
    tof: ToFConfig = field(default_factory=ToFConfig)
    bg_quad: tuple = (0.0, 0.0, 0.0, 0.0)
    bg_color: tuple = (0.0, 0.0, 0.0)

    @property
    def n(self) -> int:
        return int(self.position.shape[0])


def _read_header(f, magic: str, what: str):
    """`magic 1` line, then `key value...` lines up to `data`; returns [(key, [values])]."""
    first = f.readline().split()
    if len(first) != 2 or first[0].decode() != magic or first[1] != b"1":
        raise TsbError(_abi.TSB_ERR_INVALID, f"{what}: bad header in {f.name}")
    fields = []
    while True:
        line = f.readline()
        if not line:
            raise TsbError(_abi.TSB_ERR_INVALID, f"{what}: expected data section")
        parts = line.split()
        if not parts:
            continue
        if parts[0] == b"data":
            return fields
        fields.append((parts[0].decode(), [p.decode() for p in parts[1:]]))


def load_scene(path) -> SceneCheckpoint:
    """load_scene (scene.cpp:176-216): text header, then n x 75 little-endian float32."""
    try:
        f = open(path, "rb")
    except OSError:
        raise TsbError(_abi.TSB_ERR_INVALID, f"load_scene: cannot open {path}") from None
    with f:
        fields = dict(_read_header(f, "tofsplat_scene", "load_scene"))
        order = ["gaussians", "sh_degree", "modulation_frequency", "source_intensity", "speed_of_light", "bg_quad",
                 "bg_color"]
        for k in order:
            if k not in fields:
                raise TsbError(_abi.TSB_ERR_INVALID, f"scene checkpoint: expected header field '{k}'")
        n = int(fields["gaussians"][0])
        if n < 0:
            raise TsbError(_abi.TSB_ERR_INVALID, "load_scene: negative gaussian count")
        raw = f.read(4 * n * GAUSSIAN_FLOATS)
        if len(raw) != 4 * n * GAUSSIAN_FLOATS:
            raise TsbError(_abi.TSB_ERR_INVALID, "scene checkpoint: truncated parameter block")
    flat = np.frombuffer(raw, "<f4").reshape(n, GAUSSIAN_FLOATS).astype(np.float32)
    tof = ToFConfig(float(fields["modulation_frequency"][0]), float(fields["source_intensity"][0]),
                    float(fields["speed_of_light"][0]))
    # pack order (scene.cpp:130-139): colour SH is coefficient-major, (16, 3)
    return SceneCheckpoint(flat[:, 0:3].copy(), flat[:, 3:6].copy(), flat[:, 6:10].copy(), flat[:, 10].copy(),
                           flat[:, 11:27].copy(), flat[:, 27:75].reshape(n, 16, 3).copy(),
                           int(fields["sh_degree"][0]), tof, tuple(float(v) for v in fields["bg_quad"][:4]),
                           tuple(float(v) for v in fields["bg_color"][:3]))


def save_scene(path, sc: SceneCheckpoint) -> None:
    """save_scene (scene.cpp:153-174): the same header fields and float32 block."""
    n = sc.n
    flat = np.zeros((n, GAUSSIAN_FLOATS), np.float32)
    flat[:, 0:3], flat[:, 3:6], flat[:, 6:10] = sc.position, sc.log_scale, sc.rotation
    flat[:, 10] = sc.opacity_logit
    flat[:, 11:27] = sc.reflectivity_sh
    flat[:, 27:75] = np.asarray(sc.color_sh, np.float32).reshape(n, 48)
    hdr = (f"tofsplat_scene 1\ngaussians {n}\nsh_degree {sc.sh_degree}\n"
           f"modulation_frequency {sc.tof.modulation_frequency!r}\nsource_intensity {sc.tof.source_intensity!r}\n"
           f"speed_of_light {sc.tof.speed_of_light!r}\n"
           f"bg_quad {' '.join(repr(float(v)) for v in sc.bg_quad)}\n"
           f"bg_color {' '.join(repr(float(v)) for v in sc.bg_color)}\ndata\n")
    with open(path, "wb") as f:
        f.write(hdr.encode())
        f.write(flat.astype("<f4").tobytes())


@dataclass
class DeformCheckpoint:
    hidden_layers: int
    width: int
    l_x: int
    l_t: int
    coord_scale: float
    parameters: np.ndarray  # flat float32, DeformNet::get_parameters order

    def parameter_count(self) -> int:
        d_in = 3 * (1 + 2 * self.l_x) + 1 + 2 * self.l_t
        sizes = [d_in] + [self.width] * self.hidden_layers + [3]
        return sum(sizes[i] * sizes[i + 1] + sizes[i + 1] for i in range(len(sizes) - 1))


def load_deform(path) -> DeformCheckpoint:
    """DeformNet::load (deform.cpp:212-246)."""
    try:
        f = open(path, "rb")
    except OSError:
        raise TsbError(_abi.TSB_ERR_INVALID, f"DeformNet::load: cannot open {path}") from None
    with f:
        cfg = {"hidden_layers": 4, "width": 128, "l_x": 10, "l_t": 10, "coord_scale": 1.0, "parameters": 0}
        for k, v in _read_header(f, "tofsplat_deform", "DeformNet::load"):
            if k not in cfg:
                raise TsbError(_abi.TSB_ERR_INVALID, f"DeformNet::load: unknown field '{k}'")
            if not v:
                raise TsbError(_abi.TSB_ERR_INVALID, "DeformNet::load: malformed header")
            cfg[k] = float(v[0]) if k == "coord_scale" else int(v[0])
        ck = DeformCheckpoint(cfg["hidden_layers"], cfg["width"], cfg["l_x"], cfg["l_t"], cfg["coord_scale"],
                              np.zeros(0, np.float32))
        if cfg["parameters"] != ck.parameter_count():
            raise TsbError(_abi.TSB_ERR_INVALID, "DeformNet::load: parameter count mismatch")
        raw = f.read(4 * cfg["parameters"])
        if len(raw) != 4 * cfg["parameters"]:
            raise TsbError(_abi.TSB_ERR_INVALID, "DeformNet::load: truncated parameter block")
    ck.parameters = np.frombuffer(raw, "<f4").astype(np.float32)
    return ck


def save_deform(path, ck: DeformCheckpoint) -> None:
    """DeformNet::save (deform.cpp:189-210)."""
    hdr = (f"tofsplat_deform 1\nhidden_layers {ck.hidden_layers}\nwidth {ck.width}\nl_x {ck.l_x}\nl_t {ck.l_t}\n"
           f"coord_scale {ck.coord_scale!r}\nparameters {ck.parameter_count()}\ndata\n")
    with open(path, "wb") as f:
        f.write(hdr.encode())
        f.write(np.asarray(ck.parameters, "<f4").tobytes())


# ---- datasets (dataset.cpp:18-153) ----------------------------------------------------------
@dataclass
class DatasetInfo:
    root: str
    tof: ToFConfig
    camera: CameraModel
    raw_fps: float
    frames: list          # (file, time, phase_index, color_file or None)
    has_color: bool
    has_flow: bool

    @property
    def num_quartets(self) -> int:
        return len(self.frames) // 4


def _camera_from_json(j) -> CameraModel:
    try:
        cam = CameraModel(fx=float(j["fx"]), fy=float(j["fy"]), cx=float(j["cx"]), cy=float(j["cy"]),
                          width=int(j["width"]), height=int(j["height"]), near_plane=float(j.get("near", 0.2)),
                          far_plane=float(j.get("far", 100.0)))
    except KeyError as e:
        raise TsbError(_abi.TSB_ERR_INVALID, f"dataset: camera field {e} missing") from None
    if "world_to_camera" in j:
        m = [float(v) for v in j["world_to_camera"]]
        if len(m) != 16:
            raise TsbError(_abi.TSB_ERR_INVALID, "dataset: world_to_camera must have 16 entries")
        cam.rotation = np.array([[m[r * 4 + c] for c in range(3)] for r in range(3)])
        cam.translation = np.array([m[r * 4 + 3] for r in range(3)])
    if not cam.valid():
        raise TsbError(_abi.TSB_ERR_INVALID, "dataset: invalid camera parameters")
    return cam


def _pfm_shape(path):
    import ctypes as C
    w, h, c = C.c_int32(), C.c_int32(), C.c_int32()
    _abi.check(_abi.lib().tsb_read_pfm(str(path).encode(), None, 0, C.byref(w), C.byref(h), C.byref(c)))
    return w.value, h.value, c.value


def load_dataset_info(dataset_dir) -> DatasetInfo:
    """load_dataset (dataset.cpp:44-116) + Dataset::validate (:118-151) without keeping the
    raw frames in memory: manifest, camera, ToF, cadence / quartet order and frame shapes."""
    root = Path(dataset_dir)
    mp = root / "manifest.json"
    try:
        text = mp.read_text()
    except OSError:
        raise TsbError(_abi.TSB_ERR_INVALID, f"dataset: cannot open {mp}") from None
    try:
        m = json.loads(text)
    except json.JSONDecodeError as e:
        raise TsbError(_abi.TSB_ERR_INVALID, f"dataset: malformed manifest: {e}") from None
    if m.get("format", "") != "tofsplat_dataset":
        raise TsbError(_abi.TSB_ERR_INVALID, "dataset: not a tofsplat_dataset manifest")
    tj = m["tof"]
    tof = ToFConfig(float(tj["modulation_frequency"]), float(tj.get("source_intensity", 1.0)),
                    float(tj.get("speed_of_light", 299792458.0)))
    if not (tof.modulation_frequency > 0 and tof.speed_of_light > 0):
        raise TsbError(_abi.TSB_ERR_INVALID, "dataset: invalid tof config")
    cam = _camera_from_json(m["camera"])
    raw_fps = float(m["raw_fps"])
    frames = [(f["file"], float(f["time"]), int(f["phase_index"]), f.get("color_file")) for f in m["frames"]]
    if not frames:
        raise TsbError(_abi.TSB_ERR_INVALID, "dataset: no raw frames")
    if len(frames) % 4:
        raise TsbError(_abi.TSB_ERR_INVALID, "dataset: raw frame count must be a multiple of 4")
    if raw_fps <= 0.0:
        raise TsbError(_abi.TSB_ERR_INVALID, "dataset: raw_fps must be positive")
    dt = 1.0 / raw_fps
    for k, (file, t, ph, _) in enumerate(frames):
        if ph != k % 4:
            raise TsbError(_abi.TSB_ERR_INVALID, f"dataset: frame {k} breaks the 0/90/180/270 quartet ordering")
        if abs(t - k * dt) > 1e-6 * max(1.0, t):
            raise TsbError(_abi.TSB_ERR_INVALID, f"dataset: frame {k} is off the raw cadence")
        if _pfm_shape(root / file) != (cam.width, cam.height, 1):
            raise TsbError(_abi.TSB_ERR_INVALID, f"dataset: frame {k} has the wrong shape")
    nq = len(frames) // 4
    has_flow = False
    for key in ("flow_fwd", "flow_bwd"):  # matched by time against the quartet base times
        for f in m.get(key, []):
            t = float(f["time"])
            if any(abs(4.0 * q / raw_fps - t) < 0.25 / raw_fps for q in range(nq)):
                has_flow = True
    return DatasetInfo(str(root), tof, cam, raw_fps, frames, any(f[3] for f in frames), has_flow)


def dataset_info(dataset_dir) -> Dict:
    ds = load_dataset_info(dataset_dir)
    return {"num_quartets": ds.num_quartets, "num_frames": len(ds.frames), "width": ds.camera.width,
            "height": ds.camera.height, "raw_fps": ds.raw_fps, "modulation_frequency": ds.tof.modulation_frequency,
            "has_color": ds.has_color, "has_flow": ds.has_flow}


def quartet_time(i: int, num_quartets: int) -> float:
    """trainer.hpp:123-125."""
    return float(i) / (num_quartets - 1) if num_quartets > 1 else 0.0


# ---- rendering ---------------------------------------------------------------------------
def _gpu_scene(ctx, sc: SceneCheckpoint, n_keyframes: int, color: bool = False) -> GaussianScene:
    g = GaussianScene(ctx, sc.n, n_keyframes, sc.tof, sh_degree=sc.sh_degree, color=color)
    motion = np.zeros((n_keyframes, sc.n, 3), np.float32) if n_keyframes else None
    g.set_params(sc.position, sc.log_scale, sc.rotation, sc.opacity_logit, sc.reflectivity_sh[:, 0], motion)
    if sc.sh_degree > 0:
        g.set_sh(sc.reflectivity_sh)
    if color:
        g.set_color(sc.color_sh)
    return g


def _hwc(planar: np.ndarray) -> np.ndarray:
    """planar (C, H, W) -> image_to_numpy's (H, W, C) float64 (bindings.cpp:24-31)."""
    return np.ascontiguousarray(np.asarray(planar, np.float64).transpose(1, 2, 0))


def render_timestep(scene_path: str, deform_path: str, dataset_dir: str, timestep: float = 0.0) -> Dict:
    """Render quads + depth at a (fractional) timestep (bindings.cpp:164-203): the canonical
    means deformed by the checkpoint's DeformNet at the quartet times floor(t) and
    floor(t) + 1, blended by interp_positions (deform.cpp:248-251), rendered with the
    dataset's camera.  Returns {"quad": (H, W, 4), "depth": (H, W, 1), "weight": (H, W, 1)}."""
    sc = load_scene(scene_path)
    ds = load_dataset_info(dataset_dir)
    ctx = _context()
    frame = (0, 0.0)
    if deform_path:
        ck = load_deform(deform_path)
        net = DeformNet(ctx, ck.hidden_layers, ck.width, ck.l_x, ck.l_t, ck.coord_scale)
        net.set_parameters(ck.parameters)
        nq = ds.num_quartets
        i1 = math.floor(timestep)
        scene = _gpu_scene(ctx, sc, 2)
        # x1 = canonical + net(canonical, t(i1)) -> keyframe 0; x2 -> keyframe 1 (trainer.hpp:123)
        net.scene_offsets(scene, 0, quartet_time(int(i1), nq))
        if timestep != i1:
            net.scene_offsets(scene, 1, quartet_time(int(i1) + 1, nq))
            frame = (0, float(timestep - i1))  # (i2 - j) x1 + (j - i1) x2
        net.close()
    else:
        scene = _gpu_scene(ctx, sc, 0)
    rp = RenderPass(ctx).prepare(scene, ds.camera, RenderOptions(), frame).forward()
    out = rp.outputs()
    res = {"quad": _hwc(out["quad"][:4]), "depth": _hwc(out["depth"][None]), "weight": _hwc(out["weight"][None])}
    rp.close()
    scene.close()
    return res


# ---- gradient check (gradcheck.cpp) --------------------------------------------------------
class MT19937_64:
    """std::mt19937_64 (the published 64-bit Mersenne Twister) + libstdc++'s
    uniform_real_distribution<double> (generate_canonical with one 64-bit draw), the
    generator gradcheck.cpp's make_setup uses."""
    _N, _M = 312, 156
    _MASK = (1 << 64) - 1

    def __init__(self, seed: int):
        self.mt = [0] * self._N
        self.mt[0] = seed & self._MASK
        for i in range(1, self._N):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & self._MASK
        self.idx = self._N

    def _twist(self):
        mt, N, M = self.mt, self._N, self._M
        upper, lower = 0xFFFFFFFF80000000, 0x7FFFFFFF
        for i in range(N):
            x = (mt[i] & upper) | (mt[(i + 1) % N] & lower)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + M) % N] ^ xa
        self.idx = 0

    def next_u64(self) -> int:
        if self.idx >= self._N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self._MASK

    def uniform(self, lo: float, hi: float) -> float:
        r = float(self.next_u64()) / 18446744073709551616.0
        if r >= 1.0:
            r = math.nextafter(1.0, 0.0)
        return r * (hi - lo) + lo


def _gradcheck_setup(seed: int, n: int, w: int, h: int):
    """make_setup (gradcheck.cpp:38-99).  Draw order follows the source; where the reference
    draws several values inside one expression (the position vector) C++ leaves the order to
    the compiler -- the setup is then the same distribution, not necessarily the same bits."""
    rng = MT19937_64(seed)
    u = rng.uniform
    cam = CameraModel(fx=0.75 * w, fy=0.75 * w, cx=0.5 * w, cy=0.5 * h, width=w, height=h)
    pos = np.zeros((n, 3))
    ls = np.zeros((n, 3))
    rot = np.zeros((n, 4))
    op = np.zeros(n)
    refl = np.zeros((n, 16))
    col = np.zeros((n, 16, 3))
    mf = np.zeros((n, 3))
    mb = np.zeros((n, 3))
    for i in range(n):
        z = 1.0 + 0.45 * i + u(0.05, 0.25)
        pos[i] = (u(-0.25, 0.25) * z, u(-0.2, 0.2) * z, z)
        for k in range(3):
            ls[i, k] = math.log(u(0.08, 0.3))
        for k in range(4):
            rot[i, k] = u(-1.0, 1.0)
        if np.linalg.norm(rot[i]) < 0.3:
            rot[i, 0] += 1.0
        op[i] = u(-1.0, 1.5)
        refl[i, 0] = u(0.3, 0.7) / SH_C0
        for c in range(3):
            col[i, 0, c] = u(0.3, 0.7) / SH_C0
        for k in range(1, 16):
            refl[i, k] = u(-0.05, 0.05)
            for c in range(3):
                col[i, k, c] = u(-0.05, 0.05)
        for k in range(3):
            mf[i, k] = u(-0.05, 0.05)
            mb[i, k] = u(-0.05, 0.05)
    bg_color = [u(0, 1), u(0, 1), u(0, 1)]
    bg_quad = [u(-1, 1) for _ in range(4)]
    bg_phasor = [u(-1, 1), u(-1, 1)]

    def image(c):  # random_image: planar data, channel-major
        return np.array([u(-1.0, 1.0) for _ in range(c * w * h)]).reshape(c, h, w)

    ups = {}
    for name, c in (("d_color", 3), ("d_quad", 4), ("d_phasor", 2), ("d_depth_raw", 1), ("d_weight", 1),
                    ("d_distortion", 1), ("d_transmittance", 1), ("d_motion_fwd_acc", 3), ("d_motion_bwd_acc", 3)):
        ups[name] = image(c)
    params = {"position": pos, "log_scale": ls, "rotation": rot, "opacity_logit": op, "reflectivity_sh": refl,
              "color_sh": col, "motion_fwd": mf, "motion_bwd": mb, "bg_color": np.array(bg_color),
              "bg_quad": np.array(bg_quad), "bg_phasor": np.array(bg_phasor)}
    return cam, params, ups


class _ExactRenderer:
    """The gradcheck objective sum_c <rendered_c, up_c> (gradcheck.cpp:112-121) from the GPU's
    reference-exact mode (TSB_CH_EXACT: every pixel composited in fp64, outputs read back as
    fp64 planes), and the analytic gradients from the GPU backward of the same mode."""

    def __init__(self, ctx, cam, p, ups):
        self.ctx, self.cam, self.ups = ctx, cam, ups
        n = p["position"].shape[0]
        self.scene = GaussianScene(ctx, n, 0, ToFConfig(), sh_degree=3, color=True)
        self.rp = RenderPass(ctx)
        self.p = {k: (np.asarray(v, np.float32) if k not in ("bg_color", "bg_quad", "bg_phasor") else
                      np.asarray(v, np.float64)) for k, v in p.items()}
        self.upload()

    def upload(self):
        p = self.p
        self.scene.set_params(p["position"], p["log_scale"], p["rotation"], p["opacity_logit"],
                              p["reflectivity_sh"][:, 0])
        self.scene.set_sh(p["reflectivity_sh"])
        self.scene.set_color(p["color_sh"])

    def options(self):
        p = self.p
        return RenderOptions(alpha_threshold=0.0, transmittance_floor=0.0, sigma_cutoff=6.0, distortion=True,
                             color=True, flow=True, exact=True, bg_quad=tuple(p["bg_quad"]),
                             bg_phasor=tuple(p["bg_phasor"]), bg_color=tuple(p["bg_color"]))

    def prepare(self):
        self.rp.prepare(self.scene, self.cam, self.options())
        self.rp.set_motion(self.p["motion_fwd"], self.p["motion_bwd"])
        return self.rp

    def objective(self) -> float:
        rp = self.prepare().forward()
        H, W = self.cam.height, self.cam.width
        tof = rp.download(_abi.OUT_F64, dtype=np.float64, shape=(11, H, W))
        ext = rp.download(_abi.OUT_EXT_F64, dtype=np.float64, shape=(9, H, W))
        u = self.ups
        # planes: quad 0-3, depth_raw 4, depth 5, weight 6, T 7, phasor 8-9, distortion 10 (one frequency)
        return float(np.sum(ext[0:3] * u["d_color"]) + np.sum(tof[0:4] * u["d_quad"]) +
                     np.sum(tof[8:10] * u["d_phasor"]) + np.sum(tof[4] * u["d_depth_raw"][0]) +
                     np.sum(tof[6] * u["d_weight"][0]) + np.sum(tof[10] * u["d_distortion"][0]) +
                     np.sum(tof[7] * u["d_transmittance"][0]) + np.sum(ext[3:6] * u["d_motion_fwd_acc"]) +
                     np.sum(ext[6:9] * u["d_motion_bwd_acc"]))

    def analytic(self):
        self.scene.zero_grads()
        rp = self.prepare().forward()
        f32 = {k: np.asarray(v, np.float32) for k, v in self.ups.items()}
        rp.backward_ext(**f32)
        g = self.scene.grads()
        mf, mb = rp.motion_grads()
        return {"position": g["d_position"], "log_scale": g["d_log_scale"], "rotation": g["d_rotation"],
                "opacity_logit": g["d_opacity_logit"], "reflectivity_sh": self.scene.get_sh(grads=True),
                "color_sh": self.scene.get_color(grads=True), "motion_fwd": mf, "motion_bwd": mb,
                "bg_color": g["d_bg_color"], "bg_quad": g["d_bg_quad"][:4], "bg_phasor": g["d_bg_phasor"][:2]}

    def close(self):
        self.rp.close()
        self.scene.close()


def gradcheck(seed: int = 7, splats: int = 4, width: int = 8, height: int = 8) -> Dict:
    """run_gradcheck (gradcheck.cpp:155-247) with the B200 renderer: the analytic gradients of
    every parameter group from the GPU backward against central finite differences
    (h = 1e-4) of the objective rendered by the GPU in reference-exact (fp64) mode, thresholds
    disabled (alpha 0, transmittance floor 0, sigma 6).  Parameters live in fp32 on the
    device, so each probe's step is the exact difference of the two stored fp32 values.
    The reference's last group, the DeformNet weights, runs on the 3xTF32 tensor-core MLP
    whose ~1e-7 relative offsets a 1e-4 probe cannot resolve to 1e-3; it is checked against
    the fp64 oracle in tests/test_gpu_deform.py and reported here under `skipped`."""
    t0 = time.perf_counter()
    cam, params, ups = _gradcheck_setup(seed, splats, width, height)
    ctx = _context()
    r = _ExactRenderer(ctx, cam, params, ups)
    try:
        an = r.analytic()
        groups = {}
        hstep = 1e-4

        def rel(a, b):
            return abs(a - b) / max(abs(a), abs(b), 1e-6)

        order = ["position", "log_scale", "rotation", "opacity_logit", "reflectivity_sh", "color_sh", "motion_fwd",
                 "motion_bwd", "bg_color", "bg_quad", "bg_phasor"]
        names = {"opacity_logit": "opacity"}
        for key in order:
            arr = r.p[key]
            a = np.asarray(an[key], np.float64).reshape(arr.shape)
            worst = 0.0
            for idx in np.ndindex(arr.shape):
                orig = arr[idx]
                hi = arr.dtype.type(orig + hstep)
                lo = arr.dtype.type(orig - hstep)
                arr[idx] = hi
                r.upload()
                jp = r.objective()
                arr[idx] = lo
                r.upload()
                jm = r.objective()
                arr[idx] = orig
                fd = (jp - jm) / (float(hi) - float(lo))
                worst = max(worst, rel(a[idx], fd))
            r.upload()
            groups[names.get(key, key)] = worst
    finally:
        r.close()
    return {"max_rel_err": max(groups.values()), "seconds": time.perf_counter() - t0, "groups": groups,
            "skipped": {"net_weights": "DeformNet runs in 3xTF32 on the tensor cores; checked against the fp64 "
                                       "oracle (tests/test_gpu_deform.py)"}}


# ---- outside the render / optimise path ---------------------------------------------------
def _unsupported(name: str, what: str):
    def f(*args, **kwargs):
        raise TsbError(_abi.TSB_ERR_UNSUPPORTED,
                       f"{name}: {what} is outside the B200 render/optimise path (SURVEY.md section 2)")
    f.__name__ = name
    return f


builtin_scene_names = _unsupported("builtin_scene_names", "the C-ToF simulator (synthcam.cpp)")
simulate_dataset = _unsupported("simulate_dataset", "the C-ToF simulator (synthcam.cpp)")
fit_dataset = _unsupported("fit_dataset", "the dataset-driven training driver (trainer.cpp fit())")
evaluate = _unsupported("evaluate", "the evaluation report (eval.cpp)")
