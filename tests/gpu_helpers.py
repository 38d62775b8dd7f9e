"""Shared helpers for the GPU parity tests: build a layer from the oracle's synthetic recipe,
feed the oracle the GPU's exact inputs, and the stated tolerances.

Tolerances (stated once, used everywhere):
  * codes / unpacked slices / permutations / bucket counts: bit-exact
  * router scores: |S_gpu - S_oracle| <= SCORE_ATOL + SCORE_RTOL*|S|   (fp32 accumulation of
    bf16 products vs fp64, identical bf16/fp32 parameters on both sides)
  * masks: identical for every token whose routed scores are all farther than MASK_MARGIN
    from delta (tokens inside the margin may flip; the count is reported)
  * layer outputs Y (bf16, fp32 accumulation, fp16 folded weights) vs the fp64 oracle on the
    same bf16 inputs: per-token relative L2 <= Y_REL_L2 and max |dY| <= Y_MAX_ABS * rms(Y)
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as O

SCORE_ATOL = 2e-3
SCORE_RTOL = 1e-4
MASK_MARGIN = 1e-2
Y_REL_L2 = 4e-3   # ~2.5x the measured noise (1.6-1.8e-3); a 5% error in slice 3's scale gives 7e-3
Y_MAX_ABS = 3e-2    # outlier guard; bf16 rounding of the largest |y| alone reaches ~1e-2, measured <= 2.4e-2 (toy)


def bf16_round(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(torch.bfloat16).to(torch.float64).numpy()


def make_layer(out, inn, *, gs=128, hidden=0, seed=1, slice_bits=(2, 2, 2, 2), device=0):
    from paper_2602_20191_b200 import MobiLayer
    L = O.synthetic_layer(out, inn, seed=seed, group_size=gs, hidden=hidden, slice_bits=slice_bits)
    layer = MobiLayer.from_stack(L["codes"], L["slice_bits"], L["scale"], L["zero"], gs, L["w1"], L["b1"],
                                 L["w2"], L["b2"], device=device)
    return L, layer


def make_x(T, inn, seed=11, device="cuda"):
    x, _ = O.gen_calibset(1, T, inn, 0.05, 8.0, seed)
    xb = torch.from_numpy(x[0]).to(torch.bfloat16)
    return xb.to(device), xb.to(torch.float64).numpy()


def oracle_scores(orc, layer, x64):
    w1, b1, w2, b2 = layer.export_router()
    return orc.score(x64, w1.astype(np.float64), b1.astype(np.float64), w2.astype(np.float64),
                     b2.astype(np.float64))


def gates_from_masks(masks: np.ndarray, n_routed: int) -> np.ndarray:
    m = np.asarray(masks).astype(np.int64)
    return np.stack([((m >> (j + 1)) & 1).astype(np.float64) for j in range(n_routed)], axis=1)


def assert_y_close(y_gpu: torch.Tensor, y_ref: np.ndarray, what=""):
    yg = y_gpu.float().cpu().numpy().astype(np.float64)
    assert yg.shape == y_ref.shape, (yg.shape, y_ref.shape)
    assert np.all(np.isfinite(yg)), what + " non-finite output"
    d = yg - y_ref
    rms = np.sqrt(np.mean(y_ref ** 2)) + 1e-30
    rel = np.linalg.norm(d, axis=1) / (np.linalg.norm(y_ref, axis=1) + 1e-30 * rms)
    maxabs = np.max(np.abs(d)) / rms
    assert rel.max() <= Y_REL_L2, f"{what} per-token rel-L2 {rel.max():.3e} > {Y_REL_L2}"
    assert maxabs <= Y_MAX_ABS, f"{what} max|dY|/rms {maxabs:.3e} > {Y_MAX_ABS}"
    return float(rel.max()), float(maxabs)
