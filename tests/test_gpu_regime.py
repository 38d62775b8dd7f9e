"""GPU parity in the regime the bench runs (production kernels, no debug override), at the BASELINE
performance configs, against the CPU oracle on identical inputs.

  * q/o 4096x4096 and k/v 1024x4096 at T = 2048 (configs[1]); gate/up 14336x4096 and down 4096x14336
    at T = 8192 (configs[3], one GPU's share is the same kernels) -- router h = in/4, delta for 3 bits;
  * the CTA-pair GEMM runs several units per pair (asserted from mobi_layer_last_plan), so the
    unit ring, the accumulator hand-over and the stage-ring phases across units are exercised;
  * the oracle (fp64, router.hpp:63-132) sees a token subset covering every bucket and a row subset
    covering every 128-row weight tile, which keeps it to seconds;
  * per-slice isolation: with slice 1 exactly zero (c1 = 0, z = 1/2) a mask {1, e} returns X.W_e^T
    alone, so a wrong scale or offset of any one slice is visible at full relative precision;
  * avg_bits (router.hpp:135-150), batch-size invariance of routing outside the margin
    (test_router.cpp:62-75), chunked host entry == one device call at the production shape, and
    concurrent forwards on distinct streams (re-entrancy).

Tolerances: tests/gpu_helpers.py.
"""
import math
import threading

import numpy as np
import pytest
import torch

from gpu_helpers import (MASK_MARGIN, SCORE_ATOL, SCORE_RTOL, Y_MAX_ABS, Y_REL_L2, assert_y_close, gates_from_masks,
                         make_x)
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_20191_b200 import _lib
    _lib.lib()


def random_layer(out, inn, *, seed, gs=128, hidden=0, c1_zero=False):
    """Random-init slices (BASELINE config 5 recipe: uniform 2-bit codes, group scales of an N(0, 0.02)
    weight) and a RouterState-style router with w2 = 0.3 N(0,1), b2 = 0.1 N(0,1) (mobi.cpp:211-212)."""
    from paper_2602_20191_b200 import MobiLayer
    rng = np.random.default_rng(seed)
    h = hidden or max(1, inn // 4)
    G = math.ceil(inn / gs)
    codes = rng.integers(0, 4, (4, out, inn), dtype=np.uint8)
    scale = rng.uniform(0.006, 0.014, out * G)
    zero = rng.uniform(1.0, 3.0, out * G)
    if c1_zero:  # W_1 = s*((c1 + 1/2) - z) = 0 exactly
        codes[0] = 0
        zero[:] = 0.5
    w1 = rng.standard_normal((inn, h)) / math.sqrt(inn)
    b1 = np.zeros(h)
    w2 = 0.3 * rng.standard_normal((h, 3))
    b2 = 0.1 * rng.standard_normal(3)
    L = dict(codes=codes, slice_bits=[2, 2, 2, 2], scale=scale, zero=zero, gs=gs, G=G, w1=w1, b1=b1, w2=w2, b2=b2)
    layer = MobiLayer.from_stack(codes, [2, 2, 2, 2], scale, zero, gs, w1, b1, w2, b2, device=0)
    return L, layer


def row_subset(out, n=512):
    """Rows covering every 128-row tile (both CTAs of every pair): a stride plus per-tile edges."""
    rows = set(range(0, out, max(1, out // n)))
    for t in range(0, out, 128):
        rows.update({t, min(out - 1, t + 127)})
    return np.array(sorted(rows))


def oracle_rows(orc, L, x64, gates, rows):
    """forward_elastic restricted to weight rows `rows` (a row's output needs only its codes/groups)."""
    G = L["G"]
    sc = L["scale"].reshape(-1, G)[rows].ravel()
    ze = L["zero"].reshape(-1, G)[rows].ravel()
    return orc.forward_elastic(x64, np.ascontiguousarray(L["codes"][:, rows, :]), L["slice_bits"], sc, ze, L["gs"],
                               gates)


def token_subset(masks, per_bucket=8, extra=16, seed=0):
    rng = np.random.default_rng(seed)
    toks = []
    for m in np.unique(masks):
        idx = np.flatnonzero(masks == m)
        toks.extend(rng.choice(idx, min(per_bucket, idx.size), replace=False).tolist())
    toks.extend(rng.choice(masks.size, min(extra, masks.size), replace=False).tolist())
    return np.array(sorted(set(toks)))


REGIME = [  # (name, out, in, T, min units per CTA pair)
    ("q/o", 4096, 4096, 2048, 2),
    ("k/v", 1024, 4096, 2048, 0),
    ("gate/up", 14336, 4096, 8192, 2),
    ("down", 4096, 14336, 8192, 2),
]


@pytest.mark.parametrize("name,out,inn,T,min_units", REGIME, ids=[r[0] for r in REGIME])
def test_bench_regime_matches_oracle(orc, name, out, inn, T, min_units):
    from paper_2602_20191_b200 import avg_bits_from_masks, calibrate_threshold
    L, layer = random_layer(out, inn, seed=out + inn)
    xb, x64 = make_x(T, inn, seed=T + 1)
    s_gpu = layer.score(xb)
    delta = calibrate_threshold(s_gpu, 1 / 6)  # 3.0 bits, pooled over the batch (pipeline.hpp:146-160)
    y, m = layer.forward(xb, delta, return_masks=True)
    plan = layer.last_plan()
    torch.cuda.synchronize()
    assert plan["gemm"] == "gemm_pair", plan
    pairs = plan["gemm_ctas"] // 2
    assert plan["units"] >= max(1, min_units * pairs), plan  # several units per CTA pair
    m_gpu = m.cpu().numpy()
    assert np.count_nonzero(np.bincount(m_gpu, minlength=16)) == 8, "all 8 buckets populated"
    # router: scores of a strided token subset against the oracle, masks outside the margin
    ts = np.arange(0, T, max(1, T // (128 if inn > 8192 else 256)))
    w1, b1, w2, b2 = (a.astype(np.float64) for a in layer.export_router())
    s_ref = orc.score(x64[ts], w1, b1, w2, b2)
    s_sub = s_gpu.cpu().numpy().astype(np.float64)[ts]
    err = np.abs(s_sub - s_ref)
    assert np.all(err <= SCORE_ATOL + SCORE_RTOL * np.abs(s_ref)), f"max score err {err.max():.3e}"
    near = np.any(np.abs(s_ref - delta) <= MASK_MARGIN, axis=1)
    m_ref = O.masks_from_gates(orc.gate_hard(s_ref, delta))
    assert np.array_equal(m_gpu[ts][~near], m_ref[~near])
    # realized bits (router.hpp:135-150) == the oracle's avg_bits of the same gates
    g_all = gates_from_masks(m_gpu, 3)
    assert avg_bits_from_masks(m, [2, 2, 2, 2]) == orc.avg_bits(g_all, [2, 2, 2, 2])
    # nested residual GEMM: tokens of every bucket x rows of every weight tile
    toks = token_subset(m_gpu, seed=T)
    rows = row_subset(out)
    y_ref = oracle_rows(orc, L, x64[toks], g_all[toks], rows)
    yg = y[torch.from_numpy(toks).cuda()][:, torch.from_numpy(rows).cuda()]
    assert_y_close(yg, y_ref, f"{name} T={T}")


@pytest.mark.parametrize("T", [1, 16, 300, 2048])
def test_per_slice_isolation(orc, T):
    """Slice 1 set to exactly zero: mask {1, e} gives X.W_e^T alone (W_e = s 4^-(e-1) (c_e - 3/2),
    slicer.hpp:51-61), so each residual slice is checked at full relative precision; mask 1 gives 0."""
    out, inn = 512, 1024
    L, layer = random_layer(out, inn, seed=T + 5, c1_zero=True)
    xb, x64 = make_x(T, inn, seed=T + 2)
    y0 = layer.forward_masked(xb, torch.ones(T, dtype=torch.uint8, device="cuda")).float()
    rows = np.arange(out)
    for e in (2, 3, 4):
        masks = np.full(T, 1 | (1 << (e - 1)), np.uint8)
        y = layer.forward_masked(xb, torch.from_numpy(masks).cuda())
        y_ref = oracle_rows(orc, L, x64, gates_from_masks(masks, 3), rows)
        assert_y_close(y, y_ref, f"slice {e} alone, T={T}")
        if e == 2:
            # slice 1 alone is zero (the decode GEMVs cancel their code offset with activation sums,
            # which leaves a rounding residue ~1e-3 of the largest residual slice's output)
            assert y0.abs().max().item() <= 2e-3 * float(np.sqrt(np.mean(y_ref ** 2)))
    # all residual slices at once, mixed per token
    rng = np.random.default_rng(T)
    masks = (rng.integers(0, 8, T) * 2 + 1).astype(np.uint8)
    y = layer.forward_masked(xb, torch.from_numpy(masks).cuda())
    y_ref = oracle_rows(orc, L, x64, gates_from_masks(masks, 3), rows)
    keep = masks != 1  # mask-1 rows are ~zero (checked above); relative error needs a signal
    if keep.any():
        assert_y_close(y[torch.from_numpy(np.flatnonzero(keep)).cuda()], y_ref[keep], f"mixed residual, T={T}")


def test_routing_is_batch_size_invariant_outside_margin(orc):
    """The same tokens routed inside batches of 1, 8, 16, 40, 64, 300 and 2048 (decode GEMV router up to
    16 tokens / 1-CTA cluster K-split / CTA-pair router), through score() and through forward()'s masks,
    get the oracle's masks except within the stated margin (test_router.cpp:62-75 pins batch ==
    row-wise for the fp64 reference)."""
    L, layer = random_layer(4096, 4096, seed=3)
    xb, x64 = make_x(2048, 4096, seed=4)
    n = 16
    s_ref = orc.score(x64[:n], *(a.astype(np.float64) for a in layer.export_router()))
    delta = float(np.quantile(s_ref, 0.8))
    near = np.any(np.abs(s_ref - delta) <= MASK_MARGIN, axis=1)
    m_ref = O.masks_from_gates(orc.gate_hard(s_ref, delta))
    for T in (1, 8, 16, 40, 64, 300, 2048):
        k = min(n, T)
        s = layer.score(xb[:T].contiguous()).cpu().numpy()[:k].astype(np.float64)
        assert np.all(np.abs(s - s_ref[:k]) <= SCORE_ATOL + SCORE_RTOL * np.abs(s_ref[:k])), f"T={T}"
        _, m = layer.forward(xb[:T].contiguous(), delta, return_masks=True)
        assert np.array_equal(m.cpu().numpy()[:k][~near[:k]], m_ref[:k][~near[:k]]), f"T={T}"


@pytest.mark.parametrize("T", [2048, 2305, 2340])
def test_forward_host_chunks_match_device_call_at_production_shape(T):
    """mobi_forward_host pipelines token chunks; the kernels are chosen for the whole batch and no
    chunk is shorter than 256 tokens, so its output equals one device-side forward bit for bit
    (2305 = 3 x 768 + 1 and 2340 leave the tails the chunker folds)."""
    from paper_2602_20191_b200 import calibrate_threshold
    L, layer = random_layer(4096, 4096, seed=T)
    xb, _ = make_x(T, 4096, seed=T + 3)
    delta = calibrate_threshold(layer.score(xb), 1 / 6)
    y, m = layer.forward(xb, delta, return_masks=True)
    xh = xb.cpu().pin_memory()
    yh = torch.empty((T, 4096), dtype=torch.bfloat16).pin_memory()
    mh = torch.empty(T, dtype=torch.uint8).pin_memory()
    layer.forward_host(xh, delta, y_host=yh, masks_host=mh)
    assert torch.equal(mh, m.cpu())
    assert torch.equal(yh, y.cpu())


def test_concurrent_forwards_on_distinct_streams():
    """A handle serves every stream with its own workspace: forwards interleaved on two streams from
    two host threads give the serial results bit for bit (the hot path is re-entrant)."""
    from paper_2602_20191_b200 import calibrate_threshold
    L, layer = random_layer(1024, 1024, seed=8)
    xs = [make_x(T, 1024, seed=T)[0] for T in (1, 37, 700, 1500)]
    delta = calibrate_threshold(layer.score(xs[-1]), 1 / 6)
    ref = [layer.forward(x, delta).clone() for x in xs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [[None] * len(xs) for _ in range(2)]
    errs = []

    def work(k):
        try:
            with torch.cuda.stream(streams[k]):
                for rep in range(6):
                    for i in range(len(xs)):
                        j = (i + k + rep) % len(xs)
                        outs[k][j] = layer.forward(xs[j], delta, stream=streams[k])
            streams[k].synchronize()
        except Exception as ex:  # surfaced below
            errs.append(ex)

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errs, errs
    for k in range(2):
        for j in range(len(xs)):
            assert torch.equal(outs[k][j], ref[j]), (k, j)


def test_tolerances_are_tight():
    """Stated tolerances (tests/gpu_helpers.py): a 5% error in one slice's scale must fail them."""
    assert Y_REL_L2 <= 4e-3 and Y_MAX_ABS <= 3e-2


def test_shared_activation_buffer_bit_identical_and_smaller():
    """mobi_layers_share_activations: serial layers on one stream share one permuted-activation buffer;
    outputs are bit-identical to private buffers and the device frees the others."""
    import torch
    from gpu_helpers import make_layer, make_x
    from paper_2602_20191_b200 import calibrate_threshold, share_activations
    dims = [(256, 512), (512, 2048), (256, 1024)]
    layers = [make_layer(o, i, seed=k + 1)[1] for k, (o, i) in enumerate(dims)]
    T = 1536
    xs = [make_x(T, i, seed=5 + k)[0] for k, (_, i) in enumerate(dims)]
    deltas = [calibrate_threshold(ly.score(x), 1 / 6) for ly, x in zip(layers, xs)]
    for ly in layers:
        ly.reserve(T)
    ref = [ly.forward(x, d).clone() for ly, x, d in zip(layers, xs, deltas)]
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    share_activations(layers)
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    for _ in range(2):  # interleaved: each layer overwrites the shared buffer the previous one used
        for ly, x, d, r in zip(layers, xs, deltas, ref):
            assert torch.equal(ly.forward(x, d), r)
    assert free1 > free0, (free0, free1)
