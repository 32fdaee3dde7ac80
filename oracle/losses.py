"""CPU restatement of the reference image losses (numpy, float64).

TEST INFRASTRUCTURE ONLY -- the parity checker for the B200 SSIM / image_loss
kernels (paper_2505_05356_b200/csrc/tsb_ssim.cu).  Only tests/ may import it.

Follows /root/reference/proj/src/losses.cpp:
  mse                       :9-25
  11-tap Gaussian window    :29-47   (sigma 1.5, normalised)
  conv_same                 :51-75   (separable, zero padded, self-adjoint)
  ssim (+ gradient, scale)  :79-145
  image_loss                :148-166 ((1 - lambda) mse + lambda (1 - ssim))
  flow_loss                 :168-251 (mean squared flow error over pixels valid in target and
                                      render, pulled back to the motion accumulators through
                                      the projection at the frozen backprojected point)
Images are planar (C, H, W) like tofsplat::Image.
"""
from __future__ import annotations

import numpy as np

WIN = 11
SIGMA = 1.5
C1 = 0.01 * 0.01
C2 = 0.03 * 0.03


def window1d() -> np.ndarray:
    d = np.arange(WIN, dtype=np.float64) - WIN // 2
    w = np.exp(-d * d / (2.0 * SIGMA * SIGMA))
    return w / w.sum()


def conv_same(plane: np.ndarray) -> np.ndarray:
    """Separable zero-padded 'same' convolution of one (H, W) plane (rows first, then columns)."""
    w = window1d()
    r = WIN // 2
    H, W = plane.shape
    pad = np.zeros((H, W + 2 * r))
    pad[:, r:r + W] = plane
    tmp = np.zeros((H, W))
    for k in range(WIN):
        tmp += w[k] * pad[:, k:k + W]
    pad = np.zeros((H + 2 * r, W))
    pad[r:r + H, :] = tmp
    out = np.zeros((H, W))
    for k in range(WIN):
        out += w[k] * pad[k:k + H, :]
    return out


def mse(pred, target, want_grad=False):
    pred, target = np.asarray(pred, np.float64), np.asarray(target, np.float64)
    n = pred.size
    if n == 0:
        return (0.0, np.zeros_like(pred)) if want_grad else 0.0
    d = pred - target
    v = float((d * d).sum() / n)
    return (v, 2.0 / n * d) if want_grad else v


def ssim(pred, target, want_grad=False, scale=1.0):
    """Mean SSIM over channels and pixels; gradient (scaled) w.r.t. pred when want_grad."""
    pred, target = np.asarray(pred, np.float64), np.asarray(target, np.float64)
    C, H, W = pred.shape
    npx = H * W
    if npx == 0:
        return (1.0, np.zeros_like(pred)) if want_grad else 1.0
    grad = np.zeros_like(pred)
    total = 0.0
    for c in range(C):
        x, y = pred[c], target[c]
        mu1, mu2 = conv_same(x), conv_same(y)
        p11, p22, p12 = conv_same(x * x), conv_same(y * y), conv_same(x * y)
        s1 = p11 - mu1 * mu1
        s2 = p22 - mu2 * mu2
        s12 = p12 - mu1 * mu2
        A1 = 2.0 * mu1 * mu2 + C1
        A2 = 2.0 * s12 + C2
        B1 = mu1 * mu1 + mu2 * mu2 + C1
        B2 = s1 + s2 + C2
        S = (A1 * A2) / (B1 * B2)
        total += S.sum() / npx
        if want_grad:
            dS_dsig1 = -S / B2
            dS_dsig12 = 2.0 * A1 / (B1 * B2)
            g_mu1 = 2.0 * mu2 * A2 / (B1 * B2) - 2.0 * mu1 * S / B1 - 2.0 * mu1 * dS_dsig1 - mu2 * dS_dsig12
            norm = scale / (npx * C)
            grad[c] = norm * (conv_same(g_mu1) + 2.0 * x * conv_same(dS_dsig1) + y * conv_same(dS_dsig12))
    value = total / C
    return (value, grad) if want_grad else value


def image_loss(pred, target, lam, want_grad=False):
    """(1 - lambda) mse + lambda (1 - ssim) (losses.cpp:148-166)."""
    pred, target = np.asarray(pred, np.float64), np.asarray(target, np.float64)
    value = 0.0
    grad = np.zeros_like(pred)
    if lam < 1.0:
        m, dm = mse(pred, target, True)
        value += (1.0 - lam) * m
        grad += (1.0 - lam) * dm
    if lam > 0.0:
        s, ds = ssim(pred, target, True, -lam)
        value += lam * (1.0 - s)
        grad += ds
    return (value, grad) if want_grad else value


def _cam(cam):
    R = np.asarray(getattr(cam, "rotation", np.eye(3)), np.float64).reshape(3, 3)
    t = np.asarray(getattr(cam, "translation", np.zeros(3)), np.float64).reshape(3)
    return float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy), R, t


def backproject(cam, px, py, depth):
    """camera.hpp:34-43: optical centre + depth * normalize(R^T ((px - cx)/fx, (py - cy)/fy, 1))."""
    fx, fy, cx, cy, R, t = _cam(cam)
    d = np.stack([(px - cx) / fx, (py - cy) / fy, np.ones_like(px)], axis=-1)
    w = d @ R  # rows: R^T d
    w = w / np.linalg.norm(w, axis=-1, keepdims=True)
    center = -(R.T @ t)
    return center + np.asarray(depth)[..., None] * w


def flow_loss(buf, cam, target_fwd=None, target_bwd=None):
    """losses.cpp:168-251.  buf: dict with flow_fwd / flow_bwd (2, H, W), flow_valid (2, H, W),
    depth (H, W), motion_fwd_acc / motion_bwd_acc (3, H, W).  Targets (3, H, W): (u, v, valid).
    Returns dict(value, valid_pixels, d_motion_fwd_acc, d_motion_bwd_acc) (None = no gradient)."""
    if buf.get("flow_fwd") is None:
        raise RuntimeError("flow_loss: render lacks flow channels")
    fx, fy, cx, cy, R, t = _cam(cam)
    H, W = np.asarray(buf["depth"]).shape
    res = {"value": 0.0, "valid_pixels": 0, "d_motion_fwd_acc": None, "d_motion_bwd_acc": None}
    dirs = []
    if target_fwd is not None:
        dirs.append(("fwd", np.asarray(target_fwd, np.float64), 0))
    if target_bwd is not None:
        dirs.append(("bwd", np.asarray(target_bwd, np.float64), 1))
    if not dirs:
        return res
    ys, xs = np.mgrid[0:H, 0:W]
    pcx, pcy = xs + 0.5, ys + 0.5
    out = {}
    value, used = 0.0, 0
    for name, tgt, vch in dirs:
        if tgt.shape != (3, H, W):
            raise RuntimeError("flow_loss: target shape mismatch")
        flow = np.asarray(buf["flow_" + name], np.float64)
        macc = np.asarray(buf["motion_" + name + "_acc"], np.float64)
        mask = (tgt[2] > 0.5) & (np.asarray(buf["flow_valid"])[vch] > 0.5)
        count = int(mask.sum())
        d = np.zeros((3, H, W))
        out[name] = d
        if count == 0:
            continue
        ru = np.where(mask, flow[0] - tgt[0], 0.0)
        rv = np.where(mask, flow[1] - tgt[1], 0.0)
        sse = float((ru * ru + rv * rv)[mask].sum())
        du, dv = 2.0 * ru / count, 2.0 * rv / count
        depth = np.where(mask, np.asarray(buf["depth"], np.float64), 1.0)
        xd = backproject(cam, pcx, pcy, depth)
        P = (xd + np.moveaxis(macc, 0, -1)) @ R.T + t
        z = P[..., 2]
        dp = np.stack([fx * du / z, fy * dv / z, -(fx * P[..., 0] * du + fy * P[..., 1] * dv) / (z * z)], axis=-1)
        dm = dp @ R  # R^T dp
        d[:] = np.where(mask[None], np.moveaxis(dm, -1, 0), 0.0)
        value += sse / count
        res["valid_pixels"] += count
        used += 1
    if used == 0:
        return res
    res["value"] = value / used
    for name, _, _ in dirs:
        res["d_motion_%s_acc" % name] = out[name] / used
    return res
