"""GPU parity of the decode-size path (decode.cu, T <= 32): router GEMV + stream-K decode GEMM.

Checked three ways:
- against the CPU oracle on identical bf16 inputs, with the tolerances in gpu_helpers.py;
- against the bucketed tcgen05 path (debug impl 5 forces it at any T);
- for determinism: repeated calls, the PDL and non-PDL launches, and CUDA-graph replay must
  return identical bytes.
"""
import numpy as np
import pytest
import torch

from gpu_helpers import MASK_MARGIN, assert_y_close, gates_from_masks, make_layer, make_x, oracle_scores
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_20191_b200 import _lib
    _lib.lib()


def _impl(layer, n):
    layer.set_debug_impl(n)


DECODE = 10  # debug impl: the decode kernels for every batch they support (production: T <= 16)


def _masks(T, seed):
    rng = np.random.default_rng(seed)
    m = (rng.integers(0, 8, T) * 2 + 1).astype(np.uint8)
    m[: min(T, 4)] = [1, 15, 3, 9][: min(T, 4)]
    return m


DEC_SHAPES = [  # (out, in, gs, hidden, T)
    (4096, 4096, 128, 0, 1),
    (4096, 4096, 128, 0, 16),
    (1024, 4096, 128, 0, 32),
    (512, 1024, 128, 64, 2),
    (512, 1024, 128, 64, 8),
    (512, 1024, 128, 64, 9),
    (512, 1024, 128, 64, 17),
    (200, 192, 64, 16, 5),      # ragged rows, gs = 64
    (130, 200, 256, 50, 3),     # single group (gs > in), in not a multiple of 64
    (300, 136, 136, 24, 31),    # single group, in % 64 != 0, partial last row tile
    (14336 // 4, 4096, 128, 0, 4),  # more row tiles than SMs' worth of k-blocks per tile
    (4096, 4096, 128, 0, 8),    # slice-plane kernel at its 8-token limit
    (1024, 14336, 128, 0, 6),   # in = 14336 (down projection), planes kernel
    (14336, 4096, 128, 0, 1),   # gate/up: 448 row tiles, four per planes CTA
    (4768, 512, 128, 64, 3),    # 149 row tiles: two per CTA, the last CTA's second tile empty
    (9600, 256, 64, 16, 12),    # 300 row tiles, four per CTA, two token groups
    (20000, 128, 64, 16, 2),    # 625 row tiles, eight per CTA (two warps per tile)
]


@pytest.mark.parametrize("out,inn,gs,h,T", DEC_SHAPES)
def test_decode_masked_matches_oracle_and_bucketed(orc, out, inn, gs, h, T):
    L, layer = make_layer(out, inn, gs=gs, hidden=h, seed=out + T)
    xb, x64 = make_x(T, inn, seed=T + 7)
    masks = _masks(T, T)
    md = torch.from_numpy(masks).cuda()
    _impl(layer, DECODE)
    y = layer.forward_masked(xb, md)
    assert layer.last_plan()["gemm"] in ("decode_planes", "decode_merged")
    y_ref = orc.forward_elastic(x64, L["codes"], L["slice_bits"], L["scale"], L["zero"], gs,
                                gates_from_masks(masks, 3))
    assert_y_close(y, y_ref, f"decode {out}x{inn} T={T}")
    _impl(layer, 5)
    try:
        y_b = layer.forward_masked(xb, md)
    finally:
        _impl(layer, 0)
    assert_y_close(y_b, y_ref, f"bucketed {out}x{inn} T={T}")


@pytest.mark.parametrize("out,inn,gs,h,T", [(4096, 4096, 128, 0, 1), (512, 1024, 128, 64, 16),
                                            (300, 136, 136, 24, 32), (1024, 4096, 128, 0, 7),
                                            (1024, 14336, 128, 0, 1),     # 448 router CTAs: shallower ring, one wave
                                            (14336, 4096, 128, 0, 2)])    # gate/up: multi-tile planes CTAs
def test_decode_forward_routes_like_oracle(orc, out, inn, gs, h, T):
    L, layer = make_layer(out, inn, gs=gs, hidden=h, seed=out + 2 * T)
    _impl(layer, DECODE)
    xb, x64 = make_x(T, inn, seed=T + 9)
    s_ref = oracle_scores(orc, layer, x64)
    for rho in (0.0, 1 / 6, 1 / 3, 1.0):
        # delta from a large calibration pool so decode batches see a realistic mix
        delta = orc.calibrate_threshold(s_ref, rho) if T > 4 else float(np.median(s_ref))
        y, m = layer.forward(xb, delta, return_masks=True)
        m_gpu = m.cpu().numpy()
        m_ref = O.masks_from_gates(orc.gate_hard(s_ref, delta))
        near = np.any(np.abs(s_ref - delta) <= MASK_MARGIN, axis=1)
        assert np.array_equal(m_gpu[~near], m_ref[~near]), f"rho={rho}"
        y_ref = orc.forward_elastic(x64, L["codes"], L["slice_bits"], L["scale"], L["zero"], gs,
                                    gates_from_masks(m_gpu, 3))
        assert_y_close(y, y_ref, f"rho={rho}")
        # the host-buffer entry point returns the same bytes
        yh = layer.forward_host(xb.cpu(), delta)
        assert torch.equal(yh, y.cpu())


def test_decode_deterministic_repeat_pdl_and_graph():
    L, layer = make_layer(2048, 2048, gs=128, hidden=0, seed=4)
    delta = 0.0
    _impl(layer, DECODE)
    for T in (1, 6, 16, 29):
        xb, _ = make_x(T, 2048, seed=T)
        y0 = layer.forward(xb, delta).clone()
        for _ in range(4):  # arrival counters must be reset by every launch
            assert torch.equal(layer.forward(xb, delta), y0)
        _impl(layer, 6)  # same kernels without the programmatic (PDL) edge
        try:
            assert torch.equal(layer.forward(xb, delta), y0)
        finally:
            _impl(layer, DECODE)
        # CUDA-graph capture of the whole forward (router + decode GEMM), replayed on new inputs
        xg = xb.clone()
        yg = torch.empty_like(y0)
        layer.forward(xg, delta, y=yg)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                layer.forward(xg, delta, y=yg)
        torch.cuda.current_stream().wait_stream(s)
        x2, _ = make_x(T, 2048, seed=T + 100)
        xg.copy_(x2)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(yg, layer.forward(x2, delta))


def test_decode_path_skipped_when_unsupported(orc):
    """gs = 32 (not a multiple of the 64-wide k-block) stays on the bucketed path; still exact."""
    L, layer = make_layer(256, 256, gs=32, hidden=32, seed=12)
    xb, x64 = make_x(5, 256, seed=3)
    masks = _masks(5, 1)
    y = layer.forward_masked(xb, torch.from_numpy(masks).cuda())
    y_ref = orc.forward_elastic(x64, L["codes"], L["slice_bits"], L["scale"], L["zero"], 32,
                                gates_from_masks(masks, 3))
    assert_y_close(y, y_ref, "gs=32")


def test_production_prefers_prefill_path_above_16_tokens(orc):
    """Production kernel choice: decode kernels up to 16 tokens, the tcgen05 prefill path above (both
    within the stated tolerance of the oracle)."""
    L, layer = make_layer(1024, 1024, gs=128, hidden=0, seed=31)
    for T, kind in ((16, ("decode_planes", "decode_merged")), (17, ("gemm_pair",)), (32, ("gemm_pair",))):
        xb, x64 = make_x(T, 1024, seed=T)
        masks = _masks(T, T)
        y = layer.forward_masked(xb, torch.from_numpy(masks).cuda())
        assert layer.last_plan()["gemm"] in kind, (T, layer.last_plan())
        y_ref = orc.forward_elastic(x64, L["codes"], L["slice_bits"], L["scale"], L["zero"], 128,
                                    gates_from_masks(masks, 3))
        assert_y_close(y, y_ref, f"T={T}")


@pytest.mark.parametrize("out,inn,T", [(14336, 4096, 1), (20000, 128, 5)])
def test_tall_layers_stream_slice_planes(orc, out, inn, T):
    """Layers with more 32-row tiles than SMs (gate/up: 448) take the slice-plane GEMV with several
    tiles per CTA, so a decode step streams only its union's planes -- not the merged 8-bit codes."""
    L, layer = make_layer(out, inn, gs=64, hidden=16, seed=out + T)
    xb, x64 = make_x(T, inn, seed=T + 11)
    masks = _masks(T, T + 1)
    y = layer.forward_masked(xb, torch.from_numpy(masks).cuda())
    assert layer.last_plan()["gemm"] == "decode_planes", layer.last_plan()
    y_ref = orc.forward_elastic(x64, L["codes"], L["slice_bits"], L["scale"], L["zero"], 64,
                                gates_from_masks(masks, 3))
    assert_y_close(y, y_ref, f"{out}x{inn} T={T}")
