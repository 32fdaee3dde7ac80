"""CPU restatement of the reference's PFM I/O and render-stack planes (numpy).

TEST INFRASTRUCTURE ONLY -- the checker for tsb_write_pfm / tsb_read_pfm
(paper_2505_05356_b200/csrc/tsb_io.cpp) and tsb_pass_render_stack.  Only tests/ may
import it.

Follows /root/reference/proj:
  write_pfm / read_pfm          pfm.cpp:51-114 ("Pf" 1 ch / "PF" 3 ch interleaved, rows bottom
                                to top, scale -1.0 little-endian on write, either order on read,
                                '#' comments in the header)
  quad_to_depth                 tof.hpp:47-65 (phase of (q90 - q270, q0 - q180) in [0, 2 pi))
  decode_quad_depth             eval.cpp:22-33
  render_stack depth gating     eval.cpp:115-118 (weight > 0.5, NaN elsewhere)
  stack file names              eval.cpp:78-82, 168-184
Images are planar (C, H, W) float arrays like tofsplat::Image.
"""
from __future__ import annotations

import numpy as np


def write_pfm(path, img) -> None:
    img = np.asarray(img, np.float32)
    if img.ndim == 2:
        img = img[None]
    c, h, w = img.shape
    if c not in (1, 3):
        raise RuntimeError(f"pfm: {path}: only 1- or 3-channel images can be written")
    if w <= 0 or h <= 0:
        raise RuntimeError(f"pfm: {path}: empty image")
    rows = np.transpose(img, (1, 2, 0))[::-1]  # (H, W, C), bottom row first
    with open(path, "wb") as f:
        f.write(f"{'Pf' if c == 1 else 'PF'}\n{w} {h}\n-1.0\n".encode())
        f.write(np.ascontiguousarray(rows).astype("<f4").tobytes())


def _tokens(data: bytes, n: int):
    """n header tokens (whitespace separated, '#' comments) and the offset after the byte that
    follows the last one."""
    toks, i = [], 0
    while len(toks) < n:
        while i < len(data) and (chr(data[i]).isspace() or data[i] == ord("#")):
            if data[i] == ord("#"):
                while i < len(data) and data[i] != ord("\n"):
                    i += 1
            else:
                i += 1
        j = i
        while j < len(data) and not chr(data[j]).isspace():
            j += 1
        toks.append(data[i:j].decode(errors="replace"))
        i = j
    return toks, i + 1


def read_pfm(path) -> np.ndarray:
    try:
        data = open(path, "rb").read()
    except OSError:
        raise RuntimeError(f"pfm: {path}: cannot open")
    (magic,), _ = _tokens(data, 1)
    if magic not in ("Pf", "PF"):
        raise RuntimeError(f"pfm: {path}: bad magic '{magic}'")
    c = 1 if magic == "Pf" else 3
    (_, ws, hs, ss), off = _tokens(data, 4)
    try:
        w, h, scale = int(ws), int(hs), float(ss)
    except ValueError:
        raise RuntimeError(f"pfm: {path}: malformed header")
    if w <= 0 or h <= 0:
        raise RuntimeError(f"pfm: {path}: bad dimensions")
    if scale == 0.0:
        raise RuntimeError(f"pfm: {path}: zero scale")
    n = w * h * c
    body = data[off:off + 4 * n]
    if len(body) < 4 * n:
        raise RuntimeError(f"pfm: {path}: truncated pixel data")
    px = np.frombuffer(body, dtype="<f4" if scale < 0 else ">f4").astype(np.float32)
    return np.ascontiguousarray(np.transpose(px.reshape(h, w, c)[::-1], (2, 0, 1)))


def quad_to_depth(quad, frequency: float, speed_of_light: float = 299792458.0):
    """tof.hpp:47-65 per pixel; quad (4, ...) -> depth, NaN where both differences vanish."""
    q = np.asarray(quad, np.float64)
    re, im = q[1] - q[3], q[0] - q[2]
    psi = np.arctan2(im, re)
    psi = np.where(psi < 0.0, psi + 2.0 * np.pi, psi)
    d = psi * speed_of_light / (4.0 * np.pi * frequency)
    return np.where((re == 0.0) & (im == 0.0), np.nan, d)


def stack_depth(depth, weight):
    """eval.cpp:115-118: mean depth where the coverage weight exceeds 0.5."""
    return np.where(np.asarray(weight) > 0.5, np.asarray(depth, np.float64), np.nan)


def stack_names(q: int, color: bool = False):
    """eval.cpp:78-82, 168-184."""
    names = [f"quad_{q:05d}{s}.pfm" for s in ("_p0", "_p90", "_p180", "_p270")]
    names += [f"depth_{q:05d}.pfm", f"dtof_{q:05d}.pfm", f"dd_{q:05d}.pfm"]
    if color:
        names.append(f"color_{q:05d}.pfm")
    return names
