"""Partitioned layer on one B200: the row shards of a column-parallel layer, each run through the C-ABI
path, concatenate to exactly the unsharded layer's output (bit-for-bit for the same kernel config,
SURVEY 8(e) scaling test), and the NCCL all-gather wrapper reproduces it at world size 1.  Token
shards likewise equal the corresponding rows of the full batch."""
import os
import socket

import numpy as np
import pytest
import torch

from gpu_helpers import make_x
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _layers(out, inn, world, align=128, seed=3):
    from paper_2602_20191_b200 import MobiLayer
    from paper_2602_20191_b200.sharding import balanced_ranges, shard_stack_rows
    L = O.synthetic_layer(out, inn, seed=seed, group_size=128)
    full = MobiLayer.from_stack(L["codes"], L["slice_bits"], L["scale"], L["zero"], 128, L["w1"], L["b1"], L["w2"],
                                L["b2"])
    ranges, per = balanced_ranges(out, world, align)
    shards = []
    for r0, r1 in ranges:
        c, s, z = shard_stack_rows(L["codes"], L["scale"], L["zero"], 128, r0, r1)
        shards.append(MobiLayer.from_stack(c, L["slice_bits"], s, z, 128, L["w1"], L["b1"], L["w2"], L["b2"]))
    return L, full, shards, ranges


@pytest.mark.parametrize("T", [512, 8])
@pytest.mark.parametrize("world", [2, 4])
def test_column_shards_concat_equals_full(T, world):
    out, inn = 1024, 512
    L, full, shards, ranges = _layers(out, inn, world)
    xb, x64 = make_x(T, inn, seed=T + world)
    s = full.score(xb)
    from paper_2602_20191_b200 import calibrate_threshold
    delta = calibrate_threshold(s, 1 / 6)
    y_full, m_full = full.forward(xb, delta, return_masks=True)
    kernels = {full.last_plan()["gemm"]}
    parts = []
    for sh in shards:
        y, m = sh.forward(xb, delta, return_masks=True)
        kernels.add(sh.last_plan()["gemm"])
        assert torch.equal(m, m_full), "replicated router must decide identical masks on every shard"
        parts.append(y)
    y_cat = torch.cat(parts, dim=1)
    # prefill kernels and the slice-plane decode GEMV (one CTA per 32-row tile, K split by a fixed
    # warp partition) do the same per-row work whatever the row split -> bit-identical;
    # the stream-K merged-code GEMV splits K by the grid, i.e. by the row count
    if T > 32 or kernels == {"decode_planes"}:
        assert torch.equal(y_cat, y_full), kernels
    else:  # stream-K decode: equal up to fp32 summation order
        d = (y_cat.float() - y_full.float()).abs().max().item()
        assert d <= 2e-2 * y_full.float().abs().max().item()


def test_create_rows_equals_sliced_stack():
    from paper_2602_20191_b200 import MobiInvalidArgument, MobiLayer, calibrate_threshold
    from paper_2602_20191_b200.sharding import shard_stack_rows
    L = O.synthetic_layer(600, 320, seed=12, group_size=64)
    args = (L["slice_bits"], L["scale"], L["zero"], 64, L["w1"], L["b1"], L["w2"], L["b2"])
    r0, r1 = 128, 472
    a = MobiLayer.from_stack_rows(L["codes"], *args, r0, r1)
    c, s, z = shard_stack_rows(L["codes"], L["scale"], L["zero"], 64, r0, r1)
    b = MobiLayer.from_stack(c, L["slice_bits"], s, z, 64, L["w1"], L["b1"], L["w2"], L["b2"])
    assert a.out == r1 - r0 and np.array_equal(a.unpack_codes(), b.unpack_codes())
    xb, _ = make_x(200, 320, seed=3)
    delta = calibrate_threshold(a.score(xb), 1 / 6)
    assert torch.equal(a.forward(xb, delta), b.forward(xb, delta))
    with pytest.raises(MobiInvalidArgument):
        MobiLayer.from_stack_rows(L["codes"], *args, 500, 700)


def test_column_parallel_layer_nccl_world1():
    import torch.distributed as dist
    from paper_2602_20191_b200 import calibrate_threshold
    from paper_2602_20191_b200.sharding import ColumnParallelMobiLayer
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        L, full, _, _ = _layers(640, 256, 1)
        cp = ColumnParallelMobiLayer(L["codes"], L["slice_bits"], L["scale"], L["zero"], 128, L["w1"], L["b1"],
                                     L["w2"], L["b2"], device=0, rank=0, world=1)
        xb, _ = make_x(300, 256, seed=9)
        delta = calibrate_threshold(full.score(xb), 1 / 6)
        assert torch.equal(cp.forward(xb, delta), full.forward(xb, delta))
    finally:
        dist.destroy_process_group()


def test_token_shards_equal_full_rows():
    from paper_2602_20191_b200 import calibrate_threshold
    from paper_2602_20191_b200.sharding import token_range
    L, full, _, _ = _layers(512, 512, 1)
    T = 700
    xb, _ = make_x(T, 512, seed=4)
    delta = calibrate_threshold(full.score(xb), 1 / 6)
    y_full = full.forward(xb, delta)
    for rank in range(3):
        t0, t1 = token_range(T, rank, 3)
        y = full.forward(xb[t0:t1].contiguous(), delta)
        assert torch.equal(y, y_full[t0:t1])


@pytest.mark.parametrize("T", [8, 64, 700])
def test_output_descriptor_places_every_shard_into_every_destination(T):
    """The fused all-gather primitive (mobi_forward_out): each of P row shards writes its columns into
    all P full [T, out] buffers (local stand-ins for the ranks' peer-mapped buffers).  Every buffer must
    equal the unsharded layer's output -- bit for bit on the prefill kernels (epilogue multi-store) and
    on the staged small-T paths (scatter copy of the shard's own output)."""
    from paper_2602_20191_b200 import calibrate_threshold
    out, inn, world = 1000, 512, 3
    L, full, shards, ranges = _layers(out, inn, world)
    xb, _ = make_x(T, inn, seed=T)
    delta = calibrate_threshold(full.score(xb), 1 / 6)
    bufs = [torch.full((T, out), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    parts = []
    for sh, (r0, r1) in zip(shards, ranges):
        sh.forward_out(xb, delta, [b.data_ptr() for b in bufs], ldy=out, col0=r0)
        parts.append(sh.forward(xb, delta))
    torch.cuda.synchronize()
    y_cat = torch.cat(parts, dim=1)
    for b in bufs:
        assert torch.equal(b, y_cat)
    if T > 32:
        assert torch.equal(y_cat, full.forward(xb, delta))


def _peer_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2602_20191_b200 import calibrate_threshold
        from paper_2602_20191_b200.sharding import ColumnParallelMobiLayer
        L, full, _, _ = _layers(1024, 512, 1)
        cp = ColumnParallelMobiLayer(L["codes"], L["slice_bits"], L["scale"], L["zero"], 128, L["w1"], L["b1"],
                                     L["w2"], L["b2"], device=0, rank=rank, world=world, collective="peer")
        ok = True
        for T in (600, 16):
            xb, _ = make_x(T, 512, seed=T)
            delta = calibrate_threshold(full.score(xb), 1 / 6)
            ref = full.forward(xb, delta)
            for _ in range(3):  # double-buffered outputs, stores into the other process's buffers
                y = cp.forward(xb, delta)
                torch.cuda.synchronize()
                if T > 32:
                    ok = ok and torch.equal(y, ref)
                else:
                    ok = ok and (y.float() - ref.float()).abs().max().item() <= 2e-2 * ref.float().abs().max().item()
        q.put((rank, cp.collective, bool(ok)))
        del cp
    except Exception as ex:  # reported to the parent
        q.put((rank, "error", repr(ex)))
    finally:
        dist.destroy_process_group()


def test_column_parallel_peer_stores_two_processes_one_gpu():
    """The fused column-parallel path end to end with real CUDA IPC: two processes (two "ranks") on the
    one GPU map each other's output buffers; every GEMM epilogue stores its columns into both, and a
    collective orders the reads.  Both ranks see the unsharded layer's output."""
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_peer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(r[1] == "peer" and r[2] is True for r in res), res
