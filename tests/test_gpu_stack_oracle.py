"""The model-level loop of the reference, ``bench::eval_at_ratio`` (pipeline.hpp:146-189), at LLaMA3-8B
linear dimensions (d = 4096, kv = 1024, ffn = 14336), two blocks, T = 16 tokens, checked layer by layer
against the oracle.

For every linear the reference pools the layer's router scores, sets the threshold with
``calibrate_threshold(pooled, rho)`` (router.hpp:167-174), gates with ``gate_hard`` (router.hpp:93-97),
runs ``forward_elastic`` (router.hpp:105-132) and feeds ``silu(y)`` to the next layer (pipeline.hpp:188-189);
realized bits are averaged over tokens (router.hpp:135-150), then over layers (pipeline.hpp:191-213).

The chain here is q -> o -> up -> down per block (the dimensions that compose); k, v and gate read the
same input as q / up (side layers: checked, not chained).  Both sides get identical inputs at every
layer (the GPU's bf16 silu(y), exactly representable in fp64), so the comparison isolates each layer:
  * delta: the device radix-select on the device scores vs the oracle's sort on the oracle scores
    (scores agree to SCORE_ATOL + SCORE_RTOL |S|, so the deltas agree to the same bound);
  * masks: identical for tokens whose routed scores are farther than MASK_MARGIN from delta;
  * y: the stated tolerance against forward_elastic with the device's masks;
  * realized bits: the per-layer mean equals avg_bits of the oracle's gates for the same masks.
"""
import numpy as np
import pytest
import torch

from gpu_helpers import MASK_MARGIN, SCORE_ATOL, SCORE_RTOL, assert_y_close, gates_from_masks
from oracle import oracle as O

pytestmark = pytest.mark.gpu

D, KV, FFN, BLOCKS, T = 4096, 1024, 14336, 2, 16
SLICE_BITS = (2, 2, 2, 2)
GS = 128


def _random_stack_layer(out, inn, rng):
    """Random-init slices (uniform 2-bit codes, group scales for unit gain) and a router per
    RouterState::init with w2 = 0.3 N(0,1), b2 = 0.1 N(0,1) (tools/mobi.cpp:211-212)."""
    from paper_2602_20191_b200 import MobiLayer
    codes = rng.integers(0, 4, size=(4, out, inn), dtype=np.uint8)
    G = -(-inn // GS)
    s0 = 1.0 / (np.sqrt(inn) * 4.0 / np.sqrt(12.0))
    scale = s0 * (0.8 + 0.4 * rng.random(out * G))
    zero = 2.0 + 0.1 * rng.standard_normal(out * G)
    h = inn // 4
    w1 = rng.standard_normal((inn, h)) / np.sqrt(inn)
    w2 = 0.3 * rng.standard_normal((h, 3))
    b2 = 0.1 * rng.standard_normal(3)
    layer = MobiLayer.from_stack(codes, list(SLICE_BITS), scale, zero, GS, w1, np.zeros(h), w2, b2, device=0)
    return dict(layer=layer, codes=codes, scale=scale, zero=zero)


def _check_layer(orc, L, x, rho, name):
    from paper_2602_20191_b200 import avg_bits_from_masks, calibrate_threshold
    layer = L["layer"]
    x64 = x.double().cpu().numpy()
    s_gpu = layer.score(x)
    delta = calibrate_threshold(s_gpu, rho)  # device radix select over the pooled T x 3 scores
    y, m = layer.forward(x, delta, return_masks=True)
    w1, b1, w2, b2 = (a.astype(np.float64) for a in layer.export_router())
    s_ref = orc.score(x64, w1, b1, w2, b2)
    err = np.abs(s_gpu.double().cpu().numpy() - s_ref)
    assert np.all(err <= SCORE_ATOL + SCORE_RTOL * np.abs(s_ref)), f"{name}: max score err {err.max():.3e}"
    delta_ref = orc.calibrate_threshold(s_ref, rho)
    tol = SCORE_ATOL + SCORE_RTOL * abs(delta_ref)
    assert abs(delta - delta_ref) <= tol, f"{name}: delta {delta} vs oracle {delta_ref}"
    masks = m.cpu().numpy()
    m_ref = O.masks_from_gates(orc.gate_hard(s_ref, delta_ref))
    near = np.any(np.abs(s_ref - delta_ref) <= MASK_MARGIN + tol, axis=1)
    assert np.array_equal(masks[~near], m_ref[~near]), f"{name}: masks differ outside the margin"
    y_ref = orc.forward_elastic(x64, L["codes"], list(SLICE_BITS), L["scale"], L["zero"], GS,
                                gates_from_masks(masks, 3))
    assert_y_close(y, y_ref, name)
    bits = avg_bits_from_masks(m, SLICE_BITS)
    assert abs(bits - orc.avg_bits(gates_from_masks(masks, 3), list(SLICE_BITS))) < 1e-9
    return y, bits


@pytest.mark.parametrize("target", [3.0])
def test_eval_at_ratio_chain_matches_oracle(orc, target):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(2026)
    rho = orc.ratio_from_target_bits(target, list(SLICE_BITS))
    x0, _ = O.gen_calibset(1, T, D, 0.05, 8.0, 7)  # calibset.hpp:20-47 recipe
    h = torch.from_numpy(x0[0]).to(torch.bfloat16).cuda()
    realized = []
    for blk in range(BLOCKS):
        shapes = [("q", D, D, True), ("k", KV, D, False), ("v", KV, D, False), ("o", D, D, True),
                  ("gate", FFN, D, False), ("up", FFN, D, True), ("down", D, FFN, True)]
        x_in = h
        for name, out, inn, chained in shapes:
            L = _random_stack_layer(out, inn, rng)
            y, bits = _check_layer(orc, L, x_in, rho, f"block {blk} {name}")
            realized.append(bits)
            L["layer"].close()
            if chained:  # the next layer reads silu(y) (pipeline.hpp:188-189)
                x_in = torch.nn.functional.silu(y.float()).to(torch.bfloat16)
        h = x_in
    assert len(realized) == 7 * BLOCKS
    # the model-level metric: mean over layers of the per-layer token means (pipeline.hpp:191-213)
    assert abs(float(np.mean(realized)) - target) <= 0.15, realized  # acceptance criterion 6
