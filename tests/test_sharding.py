"""Multi-GPU partitioning host logic on CPU with gloo, world_size 2.

Each rank takes its row shard of a synthetic SliceStack, computes its [T, rows_p] outputs with the
oracle (the CUDA per-rank forward is the single-GPU path, tested in test_gpu_parity.py), and the
same all-gather + re-interleave the ColumnParallelMobiLayer uses must reproduce the full layer's
output exactly.  Token sharding must cover every token once.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_20191_b200.sharding import (all_gather_columns, balanced_ranges, interleave_columns,
                                            shard_stack_rows, token_range)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dim, in_dim, T, align, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        orc = O.restatement()
        L = O.synthetic_layer(out_dim, in_dim, seed=5, group_size=64)
        x, _ = O.gen_calibset(1, T, in_dim, 0.05, 8.0, 3)
        x = x[0]
        s = orc.score(x, L["w1"], L["b1"], L["w2"], L["b2"])
        delta = orc.calibrate_threshold(s, 1 / 6)
        g = (s - delta > 0).astype(np.float64)
        ranges, per = balanced_ranges(out_dim, world, align)
        r0, r1 = ranges[rank]
        c, sc, ze = shard_stack_rows(L["codes"], L["scale"], L["zero"], 64, r0, r1)
        y_loc = orc.forward_elastic(x, c, L["slice_bits"], sc, ze, 64, g)  # this rank's rows
        y = all_gather_columns(torch.from_numpy(y_loc), per, out_dim)
        y_full = orc.forward_elastic(x, L["codes"], L["slice_bits"], L["scale"], L["zero"], 64, g)
        t0, t1 = token_range(T, rank, world)
        toks = torch.zeros(T, dtype=torch.int64)
        toks[t0:t1] = 1
        dist.all_reduce(toks)
        q.put((rank, bool(np.array_equal(y.numpy(), y_full)), bool((toks == 1).all())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("out_dim,align", [(96, 16), (100, 1), (64, 32)])
def test_column_parallel_gloo_world2(out_dim, align):
    world, T, in_dim = 2, 24, 128
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out_dim, in_dim, T, align, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, covered in res:
        assert same, f"rank {rank}: gathered column shards differ from the full layer output"
        assert covered, f"rank {rank}: token ranges do not cover every token exactly once"


def test_balanced_ranges_and_shard_rows():
    ranges, per = balanced_ranges(14336, 8, 128)
    assert per == 1792 and ranges[-1] == (12544, 14336)
    ranges, per = balanced_ranges(100, 3, 16)
    assert per == 48 and ranges == [(0, 48), (48, 96), (96, 100)]
    codes = np.arange(2 * 6 * 8, dtype=np.uint8).reshape(2, 6, 8)
    scale = np.arange(6 * 2, dtype=np.float64)  # gs = 4 -> 2 groups per row
    c, s, z = shard_stack_rows(codes, scale, -scale, 4, 2, 5)
    assert c.shape == (2, 3, 8) and np.array_equal(c, codes[:, 2:5])
    assert np.array_equal(s, scale[4:10]) and np.array_equal(z, -scale[4:10])
    with pytest.raises(ValueError):
        shard_stack_rows(codes, scale, scale, 4, 4, 7)


def test_interleave_columns_layout():
    world, T, per, out = 3, 2, 4, 10
    # rank p's block holds values 100*p + 10*t + j for its column j
    g = torch.stack([torch.tensor([[100 * p + 10 * t + j for j in range(per)] for t in range(T)])
                     for p in range(world)]).reshape(world * T, per)
    y = interleave_columns(g, world, T, per, out)
    assert y.shape == (T, out)
    for t in range(T):
        for c in range(out):
            p, j = divmod(c, per)
            assert y[t, c] == 100 * p + 10 * t + j
