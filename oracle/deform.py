"""CPU restatement of the reference DeformNet (numpy, float64).

TEST INFRASTRUCTURE ONLY -- the parity checker for the B200 DeformNet
(paper_2505_05356_b200/csrc/tsb_mlp.cu).  Only tests/ and bench.py's CPU legs
may import it; the product package never does.

Follows /root/reference/proj:
  positional_encode / positional_encode_derivative   deform.cpp:10-26
  DeformNet layer layout, input_dim                  deform.hpp:19-66, deform.cpp:56-58
  encode_batch                                       deform.cpp:60-78
  offsets (ReLU hidden layers, linear output)        deform.cpp:80-102
  backward (dW, db, d_positions via the encoding)    deform.cpp:124-159
  get/set_parameters flat order (W row-major, b)     deform.cpp:167-186
  interp_positions                                   deform.cpp:248-251
The reference initialises with std::mt19937_64 + std::normal_distribution
(deform.cpp:28-54), which numpy cannot reproduce bit for bit; parity tests set
the parameters explicitly (set_parameters), as the reference's own tests do.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np


def encoding_size(levels: int) -> int:
    return 1 + 2 * levels


def positional_encode(v, levels: int) -> np.ndarray:
    """gamma(v) = [v, sin(2^0 pi v), cos(2^0 pi v), ...] along a new last axis."""
    v = np.asarray(v, np.float64)
    out = np.empty(v.shape + (encoding_size(levels),))
    out[..., 0] = v
    freq = np.pi
    for lv in range(levels):
        out[..., 1 + 2 * lv] = np.sin(freq * v)
        out[..., 2 + 2 * lv] = np.cos(freq * v)
        freq *= 2.0
    return out


def positional_encode_derivative(v, levels: int) -> np.ndarray:
    v = np.asarray(v, np.float64)
    out = np.empty(v.shape + (encoding_size(levels),))
    out[..., 0] = 1.0
    freq = np.pi
    for lv in range(levels):
        out[..., 1 + 2 * lv] = freq * np.cos(freq * v)
        out[..., 2 + 2 * lv] = -freq * np.sin(freq * v)
        freq *= 2.0
    return out


@dataclass
class DeformConfig:
    hidden_layers: int = 4
    width: int = 128
    l_x: int = 10
    l_t: int = 10
    coord_scale: float = 1.0
    final_std: float = 1e-5


@dataclass
class Cache:
    input: np.ndarray                 # (n, input_dim)
    h: List[np.ndarray]               # post-ReLU activations per hidden layer, (n, width)
    scaled: np.ndarray                # (n, 3) positions / coord_scale


@dataclass
class DeformNet:
    cfg: DeformConfig
    W: List[np.ndarray] = field(default_factory=list)  # [0]: width x in, hidden: width x width, last: 3 x width
    b: List[np.ndarray] = field(default_factory=list)

    @staticmethod
    def init(cfg: DeformConfig, seed: int) -> "DeformNet":
        """Xavier-normal hidden layers, zero biases, N(0, final_std) output layer (deform.cpp:28-54),
        drawn from numpy's generator (not the reference's stream)."""
        rng = np.random.default_rng(seed)
        net = DeformNet(cfg)
        prev = net.input_dim
        for _ in range(cfg.hidden_layers):
            std = np.sqrt(2.0 / (cfg.width + prev))
            net.W.append(std * rng.normal(size=(cfg.width, prev)))
            net.b.append(np.zeros(cfg.width))
            prev = cfg.width
        net.W.append(cfg.final_std * rng.normal(size=(3, prev)))
        net.b.append(np.zeros(3))
        return net

    @property
    def input_dim(self) -> int:
        return 3 * encoding_size(self.cfg.l_x) + encoding_size(self.cfg.l_t)

    @property
    def parameter_count(self) -> int:
        return sum(w.size + b.size for w, b in zip(self.W, self.b))

    def get_parameters(self) -> np.ndarray:
        return np.concatenate([np.concatenate([w.ravel(), b]) for w, b in zip(self.W, self.b)])

    def set_parameters(self, flat) -> None:
        flat = np.asarray(flat, np.float64)
        if flat.size != self.parameter_count:
            raise ValueError("DeformNet::set_parameters: size mismatch")
        k = 0
        for i, (w, b) in enumerate(zip(self.W, self.b)):
            self.W[i] = flat[k:k + w.size].reshape(w.shape)
            k += w.size
            self.b[i] = flat[k:k + b.size].copy()
            k += b.size

    def encode_batch(self, scaled: np.ndarray, t: float) -> np.ndarray:
        n = scaled.shape[0]
        ex = encoding_size(self.cfg.l_x)
        x = np.empty((n, self.input_dim))
        for c in range(3):
            x[:, c * ex:(c + 1) * ex] = positional_encode(scaled[:, c], self.cfg.l_x)
        x[:, 3 * ex:] = positional_encode(np.float64(t), self.cfg.l_t)[None, :]
        return x

    def offsets(self, positions, t: float, with_cache: bool = False):
        """positions (n, 3) -> offsets (n, 3) at normalised time t."""
        scaled = np.asarray(positions, np.float64) / self.cfg.coord_scale
        x = self.encode_batch(scaled, t)
        hs = []
        prev = x
        for lv in range(self.cfg.hidden_layers):
            a = prev @ self.W[lv].T + self.b[lv]
            hs.append(np.maximum(a, 0.0))
            prev = hs[-1]
        out = prev @ self.W[-1].T + self.b[-1]
        if with_cache:
            return out, Cache(x, hs, scaled)
        return out

    def backward(self, cache: Cache, d_offsets, want_positions: bool = True, gates=None):
        """Returns (dW list, db list, d_positions (n, 3) or None) for one cached forward.
        gates (test aid): per hidden layer, boolean ReLU gates to use instead of h > 0."""
        delta = np.asarray(d_offsets, np.float64)
        layers = len(self.W)
        dW = [None] * layers
        db = [None] * layers
        d_pos = None
        for lv in range(layers - 1, -1, -1):
            below = cache.input if lv == 0 else cache.h[lv - 1]
            dW[lv] = delta.T @ below
            db[lv] = delta.sum(axis=0)
            if lv == 0:
                if want_positions:
                    d_input = delta @ self.W[0]
                    ex = encoding_size(self.cfg.l_x)
                    d_pos = np.empty((delta.shape[0], 3))
                    for c in range(3):
                        der = positional_encode_derivative(cache.scaled[:, c], self.cfg.l_x)
                        d_pos[:, c] = (der * d_input[:, c * ex:(c + 1) * ex]).sum(axis=1) / self.cfg.coord_scale
                break
            d_below = delta @ self.W[lv]
            delta = d_below * (cache.h[lv - 1] > 0.0 if gates is None else gates[lv - 1])
        return dW, db, d_pos

    def flat_grads(self, dW, db) -> np.ndarray:
        return np.concatenate([np.concatenate([w.ravel(), b]) for w, b in zip(dW, db)])


def interp_positions(x_i1, x_i2, i1: float, i2: float, j: float):
    """deform.cpp:248-251."""
    return (i2 - j) * np.asarray(x_i1) + (j - i1) * np.asarray(x_i2)
