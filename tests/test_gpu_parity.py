"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical inputs.

Tolerances are stated in tests/gpu_helpers.py.  Every test here needs a B200.
"""
import numpy as np
import pytest
import torch

from conftest import GOLD
from gpu_helpers import (MASK_MARGIN, SCORE_ATOL, SCORE_RTOL, assert_y_close, gates_from_masks, make_layer,
                         make_x, oracle_scores)
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_20191_b200 import _lib
    _lib.lib()  # loud failure if the extension is missing


SHAPES = [  # (out, in, gs, hidden, T)
    (32, 32, 128, 8, 128),      # BASELINE config 1 geometry (toy: one partial group per row)
    (200, 96, 32, 16, 37),      # ragged rows, in not a multiple of 64
    (256, 384, 128, 0, 300),    # > one token tile, h = in/4
    (130, 200, 256, 50, 1),     # single token, gs > in
]


@pytest.mark.parametrize("out,inn,gs,h,T", SHAPES)
def test_unpack_codes_bit_exact(out, inn, gs, h, T):
    L, layer = make_layer(out, inn, gs=gs, hidden=h, seed=out)
    assert np.array_equal(layer.unpack_codes(), L["codes"])


def test_checkpoint_planes_ingest_bit_exact(orc):
    from paper_2602_20191_b200 import MobiLayer, checkpoint as ckpt
    ck = ckpt.load(GOLD / "toy_default_seed1.mobi")
    for rec in ck.layers:
        layer = MobiLayer.from_record(rec)
        assert np.array_equal(layer.unpack_codes(), orc.layer_stack(rec.planes, rec.cols, rec.slice_bits))


@pytest.mark.parametrize("out,inn,gs,h,T", SHAPES)
def test_router_scores_and_masks(orc, out, inn, gs, h, T):
    L, layer = make_layer(out, inn, gs=gs, hidden=h, seed=out + 1)
    xb, x64 = make_x(T, inn, seed=T)
    s_gpu = layer.score(xb).cpu().numpy().astype(np.float64)
    s_ref = oracle_scores(orc, layer, x64)
    err = np.abs(s_gpu - s_ref)
    assert np.all(err <= SCORE_ATOL + SCORE_RTOL * np.abs(s_ref)), f"max score err {err.max():.3e}"
    for rho in (0.0, 1 / 12, 1 / 6, 1 / 3, 1.0):
        delta = orc.calibrate_threshold(s_ref, rho)
        s, m, perm, inv, cnt = layer.route(xb, delta)
        g_ref = orc.gate_hard(s_ref, delta)
        m_ref = O.masks_from_gates(g_ref)
        near = np.any(np.abs(s_ref - delta) <= MASK_MARGIN, axis=1)
        m_gpu = m.cpu().numpy()
        assert np.array_equal(m_gpu[~near], m_ref[~near])
        # bucketing is exact for the GPU's own masks (bitplane.hpp:178-201)
        _, perm_ref, inv_ref, groups = orc.permute_by_slice(x64, m_gpu)
        assert np.array_equal(perm.cpu().numpy(), perm_ref)
        assert np.array_equal(inv.cpu().numpy(), inv_ref)
        c = cnt.cpu().numpy()
        assert [(mm, int(c[mm])) for mm in range(16) if c[mm]] == groups


@pytest.mark.parametrize("out,inn,gs,h,T", SHAPES)
def test_forward_masked_matches_oracle(orc, out, inn, gs, h, T):
    L, layer = make_layer(out, inn, gs=gs, hidden=h, seed=out + 2)
    xb, x64 = make_x(T, inn, seed=T + 3)
    rng = np.random.default_rng(T)
    masks = (rng.integers(0, 8, T) * 2 + 1).astype(np.uint8)
    masks[: min(T, 4)] = [1, 15, 3, 9][: min(T, 4)]
    y = layer.forward_masked(xb, torch.from_numpy(masks).cuda())
    g = gates_from_masks(masks, 3)
    y_ref = orc.forward_elastic(x64, L["codes"], L["slice_bits"], L["scale"], L["zero"], gs, g)
    assert_y_close(y, y_ref, f"{out}x{inn} T={T}")


@pytest.mark.parametrize("out,inn,gs,h,T", SHAPES)
def test_forward_full_matches_oracle(orc, out, inn, gs, h, T):
    L, layer = make_layer(out, inn, gs=gs, hidden=h, seed=out + 4)
    xb, x64 = make_x(T, inn, seed=T + 5)
    s_ref = oracle_scores(orc, layer, x64)
    delta = orc.calibrate_threshold(s_ref, 1 / 6)
    y, m = layer.forward(xb, delta, return_masks=True)
    m_gpu = m.cpu().numpy()
    g = gates_from_masks(m_gpu, 3)
    y_ref = orc.forward_elastic(x64, L["codes"], L["slice_bits"], L["scale"], L["zero"], gs, g)
    assert_y_close(y, y_ref, "forward")
    # end-to-end host call returns the same bytes
    yh = layer.forward_host(xb.cpu(), delta)
    assert torch.equal(yh, y.cpu())


def test_tcgen05_matches_cuda_core_reference_kernel():
    L, layer = make_layer(384, 512, gs=128, hidden=64, seed=9)
    xb, _ = make_x(700, 512, seed=2)
    masks = torch.from_numpy((np.arange(700) % 8 * 2 + 1).astype(np.uint8)).cuda()
    y_tc = layer.forward_masked(xb, masks)
    layer.set_debug_impl(1)
    try:
        y_ref = layer.forward_masked(xb, masks)
    finally:
        layer.set_debug_impl(0)
    d = (y_tc.float() - y_ref.float()).abs().max().item()
    assert d <= 2e-2 * y_ref.float().pow(2).mean().sqrt().item()


def test_toy_checkpoint_stream_matches_golden():
    """BASELINE config 1: the reference's toy_default checkpoint, layer by layer on calib batch 0."""
    from paper_2602_20191_b200 import MobiLayer, checkpoint as ckpt
    ck = ckpt.load(GOLD / "toy_default_seed1.mobi")
    z = np.load(GOLD / "toy_stream.npz")
    for t in (2, 3, 4):
        for li, rec in enumerate(ck.layers):
            k = f"t{t}_l{li}"
            layer = MobiLayer.from_record(rec)
            xb = torch.from_numpy(z[k + "_x"]).to(torch.bfloat16).cuda()
            m_ref = z[k + "_masks"]
            y = layer.forward_masked(xb, torch.from_numpy(m_ref).cuda())
            # oracle on the same bf16 inputs
            orc = O.restatement()
            y_ref = orc.forward_elastic(xb.double().cpu().numpy(), z[f"l{li}_codes"], rec.slice_bits,
                                        rec.base_scale, rec.base_zero, rec.group_size, z[k + "_g"])
            assert_y_close(y, y_ref, k)
            # routed masks agree with the golden masks outside the score margin
            s_gold = z[k + "_s"]
            delta = float(z[k + "_delta"])
            _, m = layer.forward(xb, delta, return_masks=True)
            near = np.any(np.abs(s_gold - delta) <= 0.05 * (1 + np.abs(s_gold).max()), axis=1)
            assert np.array_equal(m.cpu().numpy()[~near], m_ref[~near])


def test_empty_and_tile_boundaries(orc):
    L, layer = make_layer(128, 128, gs=128, hidden=32, seed=3)
    y = layer.forward(torch.empty((0, 128), dtype=torch.bfloat16, device="cuda"), 0.0)
    assert y.shape == (0, 128)
    for T in (255, 256, 257, 513):
        xb, x64 = make_x(T, 128, seed=T)
        masks = torch.full((T,), 7, dtype=torch.uint8, device="cuda")
        y = layer.forward_masked(xb, masks)
        y_ref = orc.forward_elastic(x64, L["codes"], L["slice_bits"], L["scale"], L["zero"], 128,
                                    gates_from_masks(np.full(T, 7), 3))
        assert_y_close(y, y_ref, f"T={T}")


def test_invalid_arguments_raise_like_reference():
    from paper_2602_20191_b200 import MobiInvalidArgument, MobiLayer
    L = O.synthetic_layer(64, 64, seed=1, group_size=64, hidden=16)
    bad = L["codes"].copy()
    bad[1, 3, 5] = 4
    with pytest.raises(MobiInvalidArgument, match="out of"):
        MobiLayer.from_stack(bad, [2] * 4, L["scale"], L["zero"], 64, L["w1"], L["b1"], L["w2"], L["b2"])
    sc = L["scale"].copy()
    sc[3] = 0.0
    with pytest.raises(MobiInvalidArgument, match="non-positive scale at group 3"):
        MobiLayer.from_stack(L["codes"], [2] * 4, sc, L["zero"], 64, L["w1"], L["b1"], L["w2"], L["b2"])
    layer = MobiLayer.from_stack(L["codes"], [2] * 4, L["scale"], L["zero"], 64, L["w1"], L["b1"], L["w2"], L["b2"])
    with pytest.raises(ValueError, match="token dim"):
        layer.forward(torch.zeros((2, 63), dtype=torch.bfloat16, device="cuda"), 0.0)
    with pytest.raises(ValueError, match="hard gate not binary"):
        layer.forward_gates(torch.zeros((2, 64), dtype=torch.bfloat16, device="cuda"), np.full((2, 3), 0.5))


def test_gpu_decompose_bit_exact(orc):
    from paper_2602_20191_b200 import decompose
    rng = O.Rng(5)
    for out, inn, gs in ((64, 256, 128), (33, 70, 32), (16, 16, 16)):
        w = rng.normal(out * inn, 0.02).reshape(out, inn)
        codes, scale, zero, cc = decompose(torch.from_numpy(w).cuda(), gs, [2, 2, 2, 2], 4.0)
        s_ref, z_ref = orc.params_from_clip(w, gs, 2, 4.0)
        c_ref, _, cc_ref = orc.decompose(w, gs, s_ref, z_ref, [2, 2, 2, 2])
        assert np.array_equal(scale.cpu().numpy(), s_ref)
        assert np.array_equal(zero.cpu().numpy(), z_ref)
        assert np.array_equal(codes.cpu().numpy(), c_ref)
        assert np.array_equal(cc, cc_ref)


def test_permute_by_slice_generic_keys(orc):
    from paper_2602_20191_b200 import permute_by_slice
    rng = np.random.default_rng(0)
    for T in (1, 50, 1023, 1024, 1025, 5000):
        m = rng.integers(0, 16, T).astype(np.uint8)  # test_bitplane.cpp:264-281 uses uniform_index(16)
        perm, inv, groups = permute_by_slice(torch.from_numpy(m).cuda())
        _, p_ref, i_ref, g_ref = orc.permute_by_slice(np.zeros((T, 1)), m)
        assert np.array_equal(perm.cpu().numpy(), p_ref)
        assert np.array_equal(inv.cpu().numpy(), i_ref)
        assert groups == g_ref


def test_calibrate_threshold_matches_reference_on_device_scores(orc):
    """router.hpp:167-174 on the device (radix select, select.cu): bit-identical to the oracle's sort,
    on 1.5e6 pooled scores (the toy calibration pool is 49152), with ties and negative zeros."""
    from paper_2602_20191_b200 import calibrate_threshold
    g = torch.Generator(device="cuda").manual_seed(3)
    pools = [torch.randn(4096 * 3, device="cuda", generator=g),
             14.0 * torch.randn(500_000 * 3, device="cuda", generator=g),
             torch.round(torch.randn(300_000, device="cuda", generator=g) * 4) / 4,  # heavy ties
             torch.tensor([0.0, -0.0, 1.0, -1.0, 0.0, 2.5, -0.0], device="cuda")]
    for s in pools:
        s64 = s.double().cpu().numpy()
        for rho in (0.0, 1e-6, 0.1, 1 / 6, 1 / 3, 0.5, 0.9, 1.0 - 1e-7, 1.0):
            assert calibrate_threshold(s, rho) == orc.calibrate_threshold(s64, rho), (s.numel(), rho)


@pytest.mark.parametrize("out,inn,T", [(4096, 4096, 16), (1024, 4096, 4)])
def test_llama_shapes(orc, out, inn, T):
    """configs[1] geometry (q/o 4096x4096, k/v 1024x4096) at h = in/4 against the oracle."""
    L, layer = make_layer(out, inn, gs=128, seed=7)
    xb, x64 = make_x(T, inn, seed=11)
    s_ref = oracle_scores(orc, layer, x64)
    delta = orc.calibrate_threshold(s_ref, 1 / 6)
    y, m = layer.forward(xb, delta, return_masks=True)
    s_gpu = layer.score(xb).cpu().numpy()
    assert np.all(np.abs(s_gpu - s_ref) <= SCORE_ATOL + SCORE_RTOL * np.abs(s_ref))
    y_ref = orc.forward_elastic(x64, L["codes"], L["slice_bits"], L["scale"], L["zero"], 128,
                                gates_from_masks(m.cpu().numpy(), 3))
    assert_y_close(y, y_ref, f"{out}x{inn}")


@pytest.mark.parametrize("inn,h,T", [(512, 128, 300), (4096, 1024, 130), (96, 16, 1)])
def test_router_tcgen05_matches_cuda_core_router(orc, inn, h, T):
    L, layer = make_layer(64, inn, gs=32 if inn < 128 else 128, hidden=h, seed=inn)
    xb, x64 = make_x(T, inn, seed=T)
    s_tc = layer.score(xb).cpu().numpy()
    layer.set_debug_impl(1)
    try:
        s_cc = layer.score(xb).cpu().numpy()
    finally:
        layer.set_debug_impl(0)
    s_ref = oracle_scores(orc, layer, x64)
    for s in (s_tc, s_cc):
        assert np.all(np.abs(s - s_ref) <= SCORE_ATOL + SCORE_RTOL * np.abs(s_ref))


@pytest.mark.parametrize("T", [1100, 2100])
def test_forward_host_chunked_pipeline_equals_device_forward(T):
    """mobi_forward_host splits large batches into token chunks pipelined over copy/compute streams;
    tokens are independent, so outputs and masks must equal the single device-side call exactly."""
    from paper_2602_20191_b200 import calibrate_threshold
    L, layer = make_layer(512, 384, gs=128, seed=T)
    xb, _ = make_x(T, 384, seed=T + 1)
    delta = calibrate_threshold(layer.score(xb), 1 / 6)
    y, m = layer.forward(xb, delta, return_masks=True)
    xh = xb.cpu().pin_memory()
    yh = torch.empty((T, 512), dtype=torch.bfloat16).pin_memory()
    mh = torch.empty(T, dtype=torch.uint8).pin_memory()
    layer.forward_host(xh, delta, y_host=yh, masks_host=mh)
    assert torch.equal(yh, y.cpu()) and torch.equal(mh, m.cpu())
    y2 = layer.forward_host(xb.cpu(), delta)  # pageable buffers take the staging path
    assert torch.equal(y2, y.cpu())


# router kernel variants (router_tc.cu): CTA-pair tiles with N = 128 and N = 256 hidden units, and the
# 1-CTA tiles with K split over a cluster of 3 (DSMEM reduction into rank 0); shapes chosen so each
# variant's selection rule fires on a 148-SM B200 (launch_router_tc)
@pytest.mark.parametrize("out,inn,h,T", [(256, 512, 2048, 1024),   # pair, N = 128
                                         (256, 256, 4096, 1280),   # pair, N = 256
                                         (256, 1024, 256, 512),    # 1-CTA, cluster K-split x3
                                         (256, 4096, 1024, 300),   # 1-CTA, cluster K-split x3, ragged T
                                         (256, 512, 2048, 1300),   # pair, ragged: the last pair's peer is empty
                                         (256, 1024, 200, 400)])   # cluster K-split, partial hidden tile
def test_router_variants_match_oracle(orc, out, inn, h, T):
    L, layer = make_layer(out, inn, gs=128, hidden=h, seed=h + T)
    xb, x64 = make_x(T, inn, seed=T + 5)
    s_gpu = layer.score(xb).cpu().numpy().astype(np.float64)
    s_ref = oracle_scores(orc, layer, x64)
    err = np.abs(s_gpu - s_ref)
    assert np.all(err <= SCORE_ATOL + SCORE_RTOL * np.abs(s_ref)), f"max score err {err.max():.3e}"
    delta = orc.calibrate_threshold(s_ref, 1 / 6)
    y, m = layer.forward(xb, delta, return_masks=True)
    near = np.any(np.abs(s_ref - delta) <= MASK_MARGIN, axis=1)
    m_ref = O.masks_from_gates(orc.gate_hard(s_ref, delta))
    assert np.array_equal(m.cpu().numpy()[~near], m_ref[~near])
    y_ref = orc.forward_elastic(x64, L["codes"], L["slice_bits"], L["scale"], L["zero"], 128,
                                gates_from_masks(m.cpu().numpy(), 3))
    assert_y_close(y, y_ref)


@pytest.mark.parametrize("T", [1, 8, 300, 2048])
def test_chained_layers_under_pdl_equal_synchronized(orc, T):
    """Layer 2 consumes layer 1's output directly (no op in between), so its PDL-launched router may
    be scheduled while layer 1's GEMM drains; it must still read the finished output.  Compared
    bit-for-bit with the same two forwards separated by a device synchronisation."""
    from paper_2602_20191_b200 import calibrate_threshold
    _, l1 = make_layer(1024, 512, gs=128, seed=21)
    _, l2 = make_layer(512, 1024, gs=128, seed=22)
    xb, _ = make_x(T, 512, seed=T + 2)
    d1 = calibrate_threshold(l1.score(xb), 1 / 6)
    y1 = l1.forward(xb, d1)
    d2 = calibrate_threshold(l2.score(y1), 1 / 6)
    torch.cuda.synchronize()
    ref2 = l2.forward(y1.clone(), d2)
    torch.cuda.synchronize()
    for _ in range(3):
        a = l1.forward(xb, d1)
        b = l2.forward(a, d2)  # back to back on one stream
    torch.cuda.synchronize()
    assert torch.equal(a, y1) and torch.equal(b, ref2)


@pytest.mark.parametrize("T", [40, 64, 300])
def test_one_cta_splitk_gemm_matches_oracle(orc, T):
    """The 1-CTA split-K tcgen05 GEMM (gemm_tc.cu, debug impl 5: a comparison path since the CTA-pair
    kernel took over 33..64 tokens) still computes forward_elastic within the stated tolerance."""
    L, layer = make_layer(512, 384, gs=128, seed=T + 77)
    xb, x64 = make_x(T, 384, seed=T + 78)
    rng = np.random.default_rng(T)
    masks = (rng.integers(0, 8, T) * 2 + 1).astype(np.uint8)
    layer.set_debug_impl(5)
    try:
        y = layer.forward_masked(xb, torch.from_numpy(masks).cuda())
    finally:
        layer.set_debug_impl(0)
    y_ref = orc.forward_elastic(x64, L["codes"], L["slice_bits"], L["scale"], L["zero"], 128, gates_from_masks(masks, 3))
    assert_y_close(y, y_ref, f"1-CTA split-K T={T}")
    y_pair = layer.forward_masked(xb, torch.from_numpy(masks).cuda())
    assert layer.last_plan()["gemm"] == "gemm_pair"
    assert_y_close(y_pair, y_ref, f"CTA-pair T={T}")
