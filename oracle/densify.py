"""CPU restatement of the reference densification surgery and Adam reindex (numpy).

TEST INFRASTRUCTURE ONLY -- the parity checker for tsb_scene_densify
(paper_2505_05356_b200/csrc/tsb_densify.cu).

Follows /root/reference/proj/src/trainer.cpp:
  prune loop with the min_count floor       :392-400
  split / clone decisions and children      :401-440
  new order (kept, then extras)             :442-469
  AdamState::reindex                        :33-47
Inputs are the fp32 parameters the device holds (promoted to float64); split
children are computed in float64 and rounded to float32, as on the device.
"""
from __future__ import annotations

import numpy as np


def quat_to_rotation(q):
    q = np.asarray(q, np.float64)
    n = np.sqrt((q * q).sum())
    w, x, y, z = q / n if n > 0 else q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def densify(params: dict, grad_sum, count, extent, grad_threshold=5e-5, opacity_floor=5e-3,
            split_scale_fraction=0.01, split_shrink=1.6, min_count=16):
    """params: position (n,3), log_scale (n,3), rotation (n,4), opacity_logit (n,), reflectivity_dc (n,),
    motion (k,n,3) or None, optional refl_sh (n,16) / color_sh (n,16,3) (fp32).  Returns (new params dict (fp32), src list: old index or -1)."""
    n = params["position"].shape[0]
    logit = params["opacity_logit"].astype(np.float64)
    drop = np.zeros(n, bool)
    alive = n
    for i in range(n):
        if not alive > min_count:
            break
        if 1.0 / (1.0 + np.exp(-logit[i])) < opacity_floor:
            drop[i] = True
            alive -= 1
    extras = []  # (parent, position, log_scale)
    for i in range(n):
        if drop[i] or count <= 0:
            continue
        if float(grad_sum[i]) / count > grad_threshold:
            ls = params["log_scale"][i].astype(np.float64)
            max_scale = np.exp(ls).max()
            if max_scale > split_scale_fraction * extent:
                axis = int(np.argmax(ls))
                R = quat_to_rotation(params["rotation"][i])
                d = R[:, axis] * 0.25 * max_scale
                for sgn in (-1.0, 1.0):
                    extras.append((i, params["position"][i].astype(np.float64) + sgn * d, ls - np.log(split_shrink)))
                drop[i] = True
            else:
                extras.append((i, None, None))
    keep = [i for i in range(n) if not drop[i]]
    order = keep + [e[0] for e in extras]
    out = {}
    for key in ("position", "log_scale", "rotation", "opacity_logit", "reflectivity_dc"):
        out[key] = params[key][order].copy()
    if params.get("motion") is not None:
        out["motion"] = params["motion"][:, order].copy()
    for key in ("refl_sh", "color_sh"):  # per-Gaussian appearance follows its parent (trainer.cpp:429-474)
        if params.get(key) is not None:
            out[key] = params[key][order].copy()
    for j, (i, pos, ls) in enumerate(extras):
        if pos is not None:
            out["position"][len(keep) + j] = pos.astype(np.float32)
            out["log_scale"][len(keep) + j] = ls.astype(np.float32)
    src = keep + [-1] * len(extras)
    return out, src


def adam_reindex(m, v, src):
    """AdamState::reindex: copied moments for kept Gaussians, zeros for new ones."""
    m2 = np.zeros((len(src),) + m.shape[1:], m.dtype)
    v2 = np.zeros((len(src),) + v.shape[1:], v.dtype)
    for j, i in enumerate(src):
        if i >= 0:
            m2[j], v2[j] = m[i], v[i]
    return m2, v2
