"""Slice layouts outside the folded-weight kernels: non-uniform widths and up to eight slices (any widths
with sum <= 8 bits, config.hpp:143-182; forward_elastic has no uniformity requirement, router.hpp:105-132).
Such layers run the generic path (CUDA-core router with up to 7 routed scores, mask decision over all 2^E
keys, per-slice CUDA-core GEMM: gemm_generic.cu) and must match the oracle like the fast path does:
codes bit-exact through the device layout, scores / masks / Y within the stated tolerances, the stable
permutation exact."""
import numpy as np
import pytest
import torch

from gpu_helpers import (MASK_MARGIN, SCORE_ATOL, SCORE_RTOL, assert_y_close, gates_from_masks, make_x,
                         oracle_scores)
from oracle import oracle as O

pytestmark = pytest.mark.gpu

LAYOUTS = [(4, 2, 2), (2, 3, 3), (3, 3, 2), (1, 1, 1, 1, 1, 1, 1, 1), (2, 2, 2, 1, 1), (3, 5)]


def _layer(sb, out=192, inn=320, gs=64, seed=3):
    from paper_2602_20191_b200 import MobiLayer
    L = O.synthetic_layer(out, inn, seed=seed, group_size=gs, slice_bits=sb)
    layer = MobiLayer.from_stack(L["codes"], L["slice_bits"], L["scale"], L["zero"], gs, L["w1"], L["b1"],
                                 L["w2"], L["b2"], device=0)
    return L, layer


@pytest.mark.parametrize("sb", LAYOUTS)
@pytest.mark.parametrize("T", [1, 37, 300])
def test_generic_layout_matches_oracle(orc, sb, T):
    from paper_2602_20191_b200 import avg_bits_from_masks, calibrate_threshold
    L, layer = _layer(sb, seed=T + len(sb))
    assert np.array_equal(layer.unpack_codes(), L["codes"]), "merged-code layout not bit-exact"
    xb, x64 = make_x(T, 320, seed=T + 9)
    s_gpu = layer.score(xb).cpu().numpy().astype(np.float64)
    s_ref = oracle_scores(orc, layer, x64)
    assert s_ref.shape == (T, len(sb) - 1)
    err = np.abs(s_gpu - s_ref)
    assert np.all(err <= SCORE_ATOL + SCORE_RTOL * np.abs(s_ref)), f"max score err {err.max():.3e}"
    rho = orc.ratio_from_target_bits(sb[0] + 0.5 * sum(sb[1:]), list(sb))
    delta = orc.calibrate_threshold(s_ref, rho)
    y, m = layer.forward(xb, delta, return_masks=True)
    assert layer.last_plan()["gemm"] == "gemm_generic"
    masks = m.cpu().numpy()
    near = np.any(np.abs(s_ref - delta) <= MASK_MARGIN, axis=1)
    m_ref = O.masks_from_gates(orc.gate_hard(s_ref, delta))
    assert np.array_equal(masks[~near], m_ref[~near])
    g = gates_from_masks(masks, len(sb) - 1)
    y_ref = orc.forward_elastic(x64, L["codes"], list(sb), L["scale"], L["zero"], 64, g)
    assert_y_close(y, y_ref, f"{sb} T={T}")
    assert abs(avg_bits_from_masks(m, list(sb)) - orc.avg_bits(g, list(sb))) < 1e-9


@pytest.mark.parametrize("sb", [(4, 2, 2), (1, 1, 1, 1, 1, 1, 1, 1)])
def test_generic_masked_and_route(orc, sb):
    L, layer = _layer(sb, seed=11)
    T = 200
    xb, x64 = make_x(T, 320, seed=5)
    rng = np.random.default_rng(4)
    E = len(sb)
    masks = (rng.integers(0, 1 << (E - 1), T) * 2 + 1).astype(np.uint8)  # every bucket, slice 1 always on
    y = layer.forward_masked(xb, torch.from_numpy(masks).cuda())
    y_ref = orc.forward_elastic(x64, L["codes"], list(sb), L["scale"], L["zero"], 64, gates_from_masks(masks, E - 1))
    assert_y_close(y, y_ref, f"masked {sb}")
    # all slices on == X reconstruct(E)^T: the all-on bucket against the oracle's dense reconstruction
    full = np.full(T, (1 << E) - 1, np.uint8)
    y_all = layer.forward_masked(xb, torch.from_numpy(full).cuda())
    W = orc.reconstruct(L["codes"], list(sb), L["scale"], L["zero"], 64, E)
    assert_y_close(y_all, x64 @ W.T, f"all-on {sb}")
    # route(): stable permutation over the 2^E keys equals the oracle's permute_by_slice
    delta = float(np.median(oracle_scores(orc, layer, x64)))
    s, m, perm, inv, cnt = layer.route(xb, delta)
    mh = m.cpu().numpy()
    _, pr_perm, pr_inv, _ = orc.permute_by_slice(np.zeros((T, 1)), mh)
    assert np.array_equal(perm.cpu().numpy(), pr_perm) and np.array_equal(inv.cpu().numpy(), pr_inv)
    assert np.array_equal(cnt.cpu().numpy(), np.bincount(mh, minlength=1 << E))
