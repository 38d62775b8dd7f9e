"""Pin the CPU oracle (C restatement) before trusting it.

(1) known-answer tests lifted from the reference's own unit tests
    (test_router.cpp, test_bitplane.cpp, test_slicer.cpp);
(2) bit-exact agreement with the reference itself (oracle/_ref) on seeded inputs;
(3) bit-exact agreement with the golden fixtures minted from the reference
    (tests/golden/make_golden.py).
"""
import hashlib
import math

import numpy as np
import pytest

from conftest import GOLD
from oracle import oracle as O


def sig(x):
    return 1.0 / (1.0 + math.exp(-x)) if x >= 0 else math.exp(x) / (1.0 + math.exp(x))


# ---------------- (1) reference known answers ----------------
def test_score_hand_example(orc):  # test_router.cpp:42-60
    w1 = np.array([[0.5], [-1.0]])
    s = orc.score(np.array([[1.0, 0.5]]), w1, [0.25], np.array([[2.0]]), [-0.125])
    assert s[0, 0] == 0.25 * sig(0.25) * 2.0 - 0.125


def test_score_rejects_dim_mismatch(orc):  # test_router.cpp:77-82
    with pytest.raises(ValueError):
        orc.score(np.zeros((2, 7)), np.zeros((8, 2)), np.zeros(2), np.zeros((2, 3)), np.zeros(3))


def test_gate_hard_strict_at_delta(orc):  # router.hpp:95 strict '>'
    g = orc.gate_hard(np.array([[1.0, 2.0, 3.0]]), 2.0)
    assert g.tolist() == [[0.0, 0.0, 1.0]]


def test_ratio_and_avg_bits_known(orc):  # test_router.cpp:293-321
    bits = [2, 2, 2, 2]
    assert abs(orc.ratio_from_target_bits(4.0, bits) - 1 / 3) < 1e-15
    assert orc.ratio_from_target_bits(2.0, bits) == 0.0
    assert orc.ratio_from_target_bits(8.0, bits) == 1.0
    with pytest.raises(ValueError):
        orc.ratio_from_target_bits(1.5, bits)
    assert orc.avg_bits(np.ones((10, 3)), bits) == 8.0
    assert orc.avg_bits(np.zeros((10, 3)), bits) == 2.0
    half = np.zeros((10, 3))
    half[:5, 0] = 1.0
    assert orc.avg_bits(half, bits) == 3.0


def test_calibrate_threshold_known(orc):  # test_router.cpp:323-372
    sc = [0.5, -1.0, 2.0, 0.0, 1.5]
    assert orc.calibrate_threshold(sc, 1.0) < -1.0
    assert orc.calibrate_threshold(sc, 0.0) >= 2.0
    d = orc.calibrate_threshold(np.arange(1, 101, dtype=float), 0.25)
    assert 24 <= int(np.sum(np.arange(1, 101) - d > 0)) <= 26
    rng = O.Rng(14)
    s = rng.normal(4096)
    for rho in (0.1, 0.3333, 0.5, 0.9):
        d = orc.calibrate_threshold(s, rho)
        assert abs(np.sum(s - d > 0) / 4096 - rho) <= 1 / 4096 + 1e-12
    with pytest.raises(ValueError):
        orc.calibrate_threshold([], 0.5)
    with pytest.raises(ValueError):
        orc.calibrate_threshold([1.0], 1.1)


def test_pack_known(orc):  # test_bitplane.cpp:68-105
    p = orc.pack_bit_major(np.array([[3]], np.uint8), 2)
    assert p.shape == (2, 1, 1) and p[0, 0, 0] & 1 and p[1, 0, 0] & 1
    rng = O.Rng(1)
    c = np.array([rng.uniform_index(256) for _ in range(16 * 70)], np.uint8).reshape(16, 70)
    p = orc.pack_bit_major(c, 8)
    for b in range(8):
        bits = (p[7 - b][:, :, None] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)
        assert np.array_equal(bits.reshape(16, -1)[:, :70].astype(np.uint8), (c >> b) & 1)
    with pytest.raises(ValueError):
        orc.pack_bit_major(np.array([[4]], np.uint8), 2)


def test_merge_and_split_known(orc):  # test_slicer.cpp:216-230 merge (2,3) -> 11
    codes = np.array([[[2]], [[3]]], np.uint8)
    assert orc.merge_codes(codes, [2, 2])[0, 0] == 11


def test_permute_known(orc):  # test_bitplane.cpp:244-262
    toks = np.arange(4, dtype=float).reshape(4, 1)
    permuted, perm, inv, groups = orc.permute_by_slice(toks, np.array([1, 3, 1, 3], np.uint8))
    assert groups == [(1, 2), (3, 2)]
    assert permuted[:, 0].tolist() == [0.0, 2.0, 1.0, 3.0]
    assert perm.tolist() == [0, 2, 1, 3] and inv.tolist() == [0, 2, 1, 3]


def test_forward_elastic_properties(orc):  # test_router.cpp:188-253
    rng = O.Rng(8)
    n = 8
    w = rng.normal(n * n).reshape(n, n)
    scale, zero = orc.params_from_clip(w, n, 2, 40.0)
    codes, _, _ = orc.decompose(w, n, scale, zero, [2, 2, 2, 2])
    x = rng.normal(5 * n).reshape(5, n)
    on = orc.forward_elastic(x, codes, [2] * 4, scale, zero, n, np.ones((5, 3)))
    full = x @ orc.reconstruct(codes, [2] * 4, scale, zero, n, 4).T
    assert np.allclose(on, full, rtol=1e-12, atol=1e-12)
    off = orc.forward_elastic(x, codes, [2] * 4, scale, zero, n, np.zeros((5, 3)))
    w1 = orc.reconstruct(codes, [2] * 4, scale, zero, n, 1)
    exp = np.array([[sum(x[i, k] * w1[j, k] for k in range(n)) for j in range(n)] for i in range(5)])
    assert np.array_equal(off, exp)  # EXPECT_EQ in test_router.cpp:202-212
    with pytest.raises(ValueError):
        orc.forward_elastic(x, codes, [2] * 4, scale, zero, n, np.full((5, 3), 0.5), hard=True)
    soft = orc.forward_elastic(x, codes, [2] * 4, scale, zero, n, np.ones((5, 3)), hard=False)
    assert np.array_equal(soft, on)


def test_bitplane_matmul_merged_equals_reconstruction(orc):  # test_bitplane.cpp:199-217
    rng = O.Rng(30)
    w = 0.4 * rng.normal(256).reshape(16, 16)
    scale, zero = orc.params_from_clip(w, 16, 2, 4.0)
    codes, _, _ = orc.decompose(w, 16, scale, zero, [2, 2, 2, 2])
    merged = orc.merge_codes(codes, [2] * 4)
    planes = orc.pack_bit_major(merged, 8)
    mscale, mzero = scale / 64.0, zero * 64.0  # slicer.hpp:166-175 merged_params
    x = rng.normal(80).reshape(5, 16)
    y = orc.bitplane_matmul(x, planes, 16, 16, mscale, mzero, list(range(8)))
    assert np.allclose(y, x @ orc.reconstruct(codes, [2] * 4, scale, zero, 16, 4).T, rtol=1e-12, atol=1e-12)


# ---------------- (2) bit-exact vs the reference itself ----------------
@pytest.mark.parametrize("out,inn,gs,h,T", [(48, 96, 32, 16, 9), (32, 32, 128, 8, 17), (40, 70, 64, 0, 5)])
def test_restatement_matches_reference(orc, ref, out, inn, gs, h, T):
    L = O.synthetic_layer(out, inn, seed=out + inn, group_size=gs, hidden=h)
    L2 = O.synthetic_layer(out, inn, seed=out + inn, group_size=gs, hidden=h, backend=ref)
    for k in ("scale", "zero", "codes", "clamp_counts"):
        assert np.array_equal(L[k], L2[k]), k
    x, _ = O.gen_calibset(1, T, inn, 0.05, 8.0, 5)
    x = x[0]
    s = orc.score(x, L["w1"], L["b1"], L["w2"], L["b2"])
    assert np.array_equal(s, ref.score(x, L["w1"], L["b1"], L["w2"], L["b2"]))
    for rho in (0.0, 1 / 12, 1 / 6, 1 / 3, 1.0):
        d = orc.calibrate_threshold(s, rho)
        assert d == ref.calibrate_threshold(s, rho)
        g = orc.gate_hard(s, d)
        assert np.array_equal(g, ref.gate_hard(s, d))
        y = orc.forward_elastic(x, L["codes"], L["slice_bits"], L["scale"], L["zero"], gs, g)
        assert np.array_equal(y, ref.forward_elastic(x, L["codes"], L["slice_bits"], L["scale"], L["zero"], gs, g))
        assert orc.avg_bits(g, L["slice_bits"]) == ref.avg_bits(g, L["slice_bits"])
        m = O.masks_from_gates(g)
        a, b = orc.permute_by_slice(x, m), ref.permute_by_slice(x, m)
        for u, v in zip(a[:3], b[:3]):
            assert np.array_equal(u, v)
        assert a[3] == b[3]
    merged = orc.merge_codes(L["codes"], L["slice_bits"])
    assert np.array_equal(merged, ref.merge_codes(L["codes"], L["slice_bits"]))
    planes = orc.pack_bit_major(merged, 8)
    assert np.array_equal(planes, ref.pack_bit_major(merged, 8))
    assert np.array_equal(orc.layer_stack(planes, inn, L["slice_bits"]), ref.layer_stack(planes, inn, L["slice_bits"]))
    assert np.array_equal(orc.layer_stack(planes, inn, L["slice_bits"]), L["codes"])
    act = [0, 3, 5, 7]
    xi = np.round(4 * x)
    assert np.array_equal(orc.bitplane_matmul(xi, planes, inn, gs, L["scale"] / 64, L["zero"] * 64, act),
                          ref.bitplane_matmul(xi, planes, inn, gs, L["scale"] / 64, L["zero"] * 64, act))


def test_restatement_matches_reference_errors(orc, ref):
    for be in (orc, ref):
        with pytest.raises(ValueError, match="hard gate not binary"):
            be.forward_elastic(np.zeros((1, 4)), np.zeros((4, 4, 4), np.uint8), [2] * 4, np.ones(4),
                               np.zeros(4), 4, np.full((1, 3), 0.5))
        with pytest.raises(ValueError, match="outside"):
            be.ratio_from_target_bits(9.0, [2, 2, 2, 2])


# ---------------- (3) golden fixtures minted from the reference ----------------
def test_golden_toy_stream(orc):
    from paper_2602_20191_b200 import checkpoint as ckpt
    ck = ckpt.load(GOLD / "toy_default_seed1.mobi")
    z = np.load(GOLD / "toy_stream.npz")
    for li, L in enumerate(ck.layers):
        codes = orc.layer_stack(L.planes, L.cols, L.slice_bits)
        assert np.array_equal(codes, z[f"l{li}_codes"])
        assert np.array_equal(L.stack(), codes)  # product-side ingest == oracle split
    for t in (2, 3, 4):
        rho = orc.ratio_from_target_bits(float(t), [2, 2, 2, 2])
        for li, L in enumerate(ck.layers):
            k = f"t{t}_l{li}"
            x = z[k + "_x"]
            s = orc.score(x, L.w1, L.b1, L.w2, L.b2)
            assert np.array_equal(s, z[k + "_s"])
            d = orc.calibrate_threshold(s, rho)
            assert d == float(z[k + "_delta"])
            g = orc.gate_hard(s, d)
            assert np.array_equal(g, z[k + "_g"])
            y = orc.forward_elastic(x, z[f"l{li}_codes"], L.slice_bits, L.base_scale, L.base_zero, L.group_size, g)
            assert np.array_equal(y, z[k + "_y"])
            m = O.masks_from_gates(g)
            assert np.array_equal(m, z[k + "_masks"])
            assert np.array_equal(orc.permute_by_slice(x, m)[1], z[k + "_perm"])
            assert orc.avg_bits(g, L.slice_bits) == float(z[k + "_avg_bits"])


def test_golden_checkpoint_roundtrip():
    from paper_2602_20191_b200 import checkpoint as ckpt
    raw = (GOLD / "toy_default_seed1.mobi").read_bytes()
    ck = ckpt.loads(raw)
    assert len(ck.layers) == 3 and ck.layers[0].rows == 32 and ck.layers[0].w1.shape == (32, 8)
    assert ckpt.dumps(ck) == raw  # bit-identical round trip (test_bench.cpp:163-185)
    with pytest.raises(ckpt.CheckpointError, match="bad magic"):
        ckpt.loads(b"XOBI" + raw[4:])
    with pytest.raises(ckpt.CheckpointError, match="version mismatch"):
        ckpt.loads(raw[:4] + b"\x02" + raw[5:])


def test_golden_small_cases(orc):
    z = np.load(GOLD / "small_cases.npz")
    for tag, n in (("n8", 8), ("n6", 6)):
        scale, zero = orc.params_from_clip(z[f"{tag}_w"], n, 2, 40.0)
        assert np.array_equal(scale, z[f"{tag}_scale"]) and np.array_equal(zero, z[f"{tag}_zero"])
        codes, _, _ = orc.decompose(z[f"{tag}_w"], n, scale, zero, [2, 2, 2, 2])
        assert np.array_equal(codes, z[f"{tag}_codes"])
        for name in ("on", "off", "mixed"):
            y = orc.forward_elastic(z[f"{tag}_x"], codes, [2] * 4, scale, zero, n, z[f"{tag}_{name}_g"])
            assert np.array_equal(y, z[f"{tag}_{name}_y"])
    assert z["perm_1313"].tolist() == [0, 2, 1, 3]


@pytest.mark.slow
def test_golden_qo_T4(orc):
    z = np.load(GOLD / "qo_T4.npz")
    L = O.synthetic_layer(4096, 4096, seed=7)
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    assert sha(L["codes"]) == str(z["codes_sha"]) and sha(L["scale"]) == str(z["scale_sha"])
    assert sha(L["w1"]) == str(z["w1_sha"])
    s = orc.score(z["x"], L["w1"], L["b1"], L["w2"], L["b2"])
    assert np.array_equal(s, z["s"])
    g = orc.gate_hard(s, float(z["delta"]))
    assert np.array_equal(g, z["g"])
    y = orc.forward_elastic(z["x"], L["codes"], L["slice_bits"], L["scale"], L["zero"], 128, g)
    assert np.array_equal(y, z["y"])


# ---- stage-2 calibration step (trainer.hpp:203-263, 341-396) ----

def joint_case(out=48, inn=160, T=24, h=16, gs=64, slice_bits=(2, 2, 2, 2), seed=5):
    """Small calibration-step inputs: partial groups (160 = 2.5 x 64), one constant group (the
    epsilon-floored scale branch, trainer.hpp:323-337), random clip gammas and a non-zero w2."""
    rng = np.random.default_rng(seed)
    w = rng.normal(0, 0.02, (out, inn))
    w[3, 64:128] = 0.01  # constant group -> floored scale
    G = (inn + gs - 1) // gs
    glo = rng.uniform(1.0, 5.0, out * G)
    ghi = rng.uniform(1.0, 5.0, out * G)
    nr = len(slice_bits) - 1
    w1 = rng.normal(0, 1 / np.sqrt(inn), (inn, h))
    b1 = rng.normal(0, 0.1, h)
    w2 = rng.normal(0, 0.5, (h, nr))
    b2 = rng.normal(0, 0.1, nr)
    x = rng.normal(0, 1.0, (T, inn))
    y_fp = x @ w.T
    return dict(w=w, group_size=gs, slice_bits=slice_bits, gamma_lo=glo, gamma_hi=ghi, w1=w1, b1=b1, w2=w2,
                b2=b2, x=x, y_fp=y_fp)


JOINT_KEYS = ("y_hat", "d_gamma_lo", "d_gamma_hi", "d_w1", "d_b1", "d_w2", "d_b2")


def assert_joint_close(a, b, rtol=1e-9):
    for k in ("data_term", "reg_term", "avg_bits", "sched_b", "loss", "tau"):
        assert abs(a[k] - b[k]) <= rtol * max(1.0, abs(b[k])), (k, a[k], b[k])
    for k in JOINT_KEYS:
        if k not in b:
            continue
        scale = max(np.abs(b[k]).max(), 1e-300)
        err = np.abs(np.asarray(a[k]) - b[k]).max() / scale
        assert err <= rtol, (k, err)


@pytest.mark.skipif(not O.LIB_REF.exists(), reason="reference library not built")
@pytest.mark.parametrize("sched,t,force", [((8.0, 3.0, 10, 0, 1e-3), 4, False),   # soft gates, log schedule
                                          ((8.0, 3.0, 10, 0, 1e-3), 10, False),  # t = L: indicator gates
                                          ((6.0, 2.5, 7, 2, 1e-2), 3, False),    # cosine schedule
                                          ((6.0, 2.5, 7, 3, 1e-2), 5, False),    # exponential
                                          ((8.0, 3.0, 10, 1, 1e-3), 2, True)])   # force_gates_on ablation
def test_joint_step_restatement_matches_reference(sched, t, force):
    c = joint_case()
    ref = O.reference().joint_step(**c, sched=sched, t=t, force_gates_on=force)
    port = O.joint_step_np(**c, sched=sched, t=t, force_gates_on=force)
    assert_joint_close(port, ref)
    assert np.abs(ref["d_gamma_lo"]).max() > 0 and (force or t == 10 or np.abs(ref["d_w1"]).max() > 0)


@pytest.mark.skipif(not O.LIB_REF.exists(), reason="reference library not built")
def test_joint_step_non_uniform_slices():
    c = joint_case(slice_bits=(4, 2, 2), seed=9)
    sched = (8.0, 3.0, 12, 1, 1e-3)
    assert_joint_close(O.joint_step_np(**c, sched=sched, t=5), O.reference().joint_step(**c, sched=sched, t=5))


@pytest.mark.skipif(not O.LIB_REF.exists(), reason="reference library not built")
@pytest.mark.parametrize("bits", [(2, 2, 2, 2), (4, 2, 2), (3, 5)])
def test_msb_step_restatement_matches_reference(bits):
    """trainer.hpp:404-426 (stage 1): slice 1 alone, with the epsilon-floored group of joint_case."""
    c = joint_case(slice_bits=bits, seed=13)
    args = dict(w=c["w"], group_size=c["group_size"], slice_bits=bits, gamma_lo=c["gamma_lo"],
                gamma_hi=c["gamma_hi"], x=c["x"], y_fp=c["y_fp"])
    ref = O.reference().msb_step(**args)
    port = O.msb_step_np(**args)
    assert abs(port["loss"] - ref["loss"]) <= 1e-9 * ref["loss"]
    for k in ("y_msb", "d_gamma_lo", "d_gamma_hi"):
        assert np.abs(port[k] - ref[k]).max() <= 1e-9 * np.abs(ref[k]).max(), k
