"""Seeded synthetic workloads for the BASELINE configs.

No dataset or checkpoint is available, so inputs follow the reference's own
synthetic recipe with the BASELINE shapes and distributions:

  X pool  standard normal [128 + M, K]; a seeded column permutation picks
          round(f*K) outlier channels scaled by m (tensorio.py:157-168);
          calibration = pool[:128], X = pool[128:]
  W       default_rng(1).standard_normal((K, N)) * 0.02 (reference [in, out])
  SAF     s = amax_calib^a / wmax^(1-a), a = 0.5 (flatten.py:34-51); W~ = s*W, X~ = X/s
  plan    top-r rows of |W~| (stable, ties to the lower index, saliency.py:77-92),
          permuted to the front: W~p = W~[P], X~p = X~[:, P]  ->  salient_idx = arange(r)
  X~p is rounded to bf16 (the device input); weight artefacts are built from f64 W~p.

This is input preparation (host NumPy + the device encoders), not the
oracle; tests check the artefacts against the oracle separately.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

CONFIGS = {
    # name: (fmt, M, K, N, r, outlier_frac, outlier_mag, act_bits, act_symmetric, r_mode)
    "c1": ("int", 512, 4096, 4096, 64, 0.01, 50.0, 4, True, "dense"),
    "c2": ("mx", 4096, 4096, 4096, 64, 0.01, 50.0, 4, True, None),
    "c3": ("int", 2048, 4096, 11008, 128, 0.005, 100.0, 8, False, "int"),
}

# Llama-2-7B decoder-block linears (C4) and Llama-3-70B (C5): (name, K, N)
LLAMA7B = [("q_proj", 4096, 4096), ("k_proj", 4096, 4096), ("v_proj", 4096, 4096), ("o_proj", 4096, 4096),
           ("gate_proj", 4096, 11008), ("up_proj", 4096, 11008), ("down_proj", 11008, 4096)]
LLAMA70B = [("q_proj", 8192, 8192), ("k_proj", 8192, 1024), ("v_proj", 8192, 1024), ("o_proj", 8192, 8192),
            ("gate_proj", 8192, 28672), ("up_proj", 8192, 28672), ("down_proj", 28672, 8192)]


def synthetic_pool(rows, cols, frac, mag, seed=0) -> np.ndarray:
    g = np.random.default_rng(seed)
    x = g.standard_normal((rows, cols))
    n = int(round(frac * cols))
    if n:
        x[:, g.permutation(cols)[:n]] *= mag
    return x


def smoothing(calib: np.ndarray, w: np.ndarray, alpha=0.5) -> np.ndarray:
    amax = np.abs(calib).max(axis=0)
    wmax = np.abs(w).max(axis=1)
    with np.errstate(divide="ignore", invalid="ignore"):
        s = amax**alpha / wmax ** (1.0 - alpha)
    return np.where(np.isfinite(s) & (s > 0), s, 1.0)


def salient_permutation(w: np.ndarray, r: int) -> np.ndarray:
    order = np.argsort(-np.abs(w).max(axis=1), kind="stable")
    sal = order[:r]
    rest = np.setdiff1d(np.arange(w.shape[0]), sal)
    return np.concatenate([sal, rest]).astype(np.intp)


def bf16(x: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


@dataclass
class LinearWorkload:
    name: str
    x: np.ndarray        # bf16-valued f64 [M, K] (permuted, flattened)
    w: np.ndarray        # f64 [K, N] folded + permuted weight
    r: int
    fmt: str


def make_linear(K, N, M, r, frac=0.01, mag=50.0, fmt="mx", saf=True, x_seed=0, w_seed=1, name="linear",
                with_x=True) -> LinearWorkload:
    w = np.random.default_rng(w_seed).standard_normal((K, N)) * 0.02
    pool = synthetic_pool(128 + (M if with_x else 0), K, frac, mag, x_seed)
    calib, x = pool[:128], pool[128:]
    if saf:
        s = smoothing(calib, w)
        w = s[:, None] * w
        x = x / s
    perm = salient_permutation(w, r)
    w = np.ascontiguousarray(w[perm])
    x = bf16(x[:, perm]) if with_x else None
    return LinearWorkload(name, x, w, r, fmt)


def make_config(name: str):
    fmt, M, K, N, r, frac, mag, bits, sym, r_mode = CONFIGS[name]
    return make_linear(K, N, M, r, frac, mag, fmt, name=name), dict(bits=bits, symmetric=sym, r_mode=r_mode)
