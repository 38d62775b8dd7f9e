"""BASELINE config 5: the full LLaMA3-8B layer stack (32 blocks x 7 MoBi linears, random-init slices),
token-adaptive routing sweep of average bits.  For every target budget the per-layer thresholds are
calibrated on the batch (pipeline.hpp:146-160), the realized bits are measured (acceptance criterion 6:
within +-0.15 of the target, acceptance.cpp:334-353), and the whole-stack forward is timed as one CUDA
graph replay.

  python tools/stack_sweep.py [--blocks 32 --tokens 2048 --steps 10]
  python -m torch.distributed.run --nproc-per-node N tools/stack_sweep.py ...   (replicas, token-sharded)

Prints one JSON line per target budget (rank 0; tokens/s is the whole job, time = max over ranks).
"""
import argparse
import functools
import json
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=32)
    ap.add_argument("--tokens", type=int, default=2048, help="tokens per GPU per forward")
    ap.add_argument("--targets", type=float, nargs="+", default=[2.0, 2.5, 3.0, 3.5, 4.0])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--concurrent", action="store_true",
                    help="run q/k/v and gate/up as parallel graph branches (side streams)")
    ap.add_argument("--calib-tokens", type=int, default=0,
                    help="calibrate the thresholds on a separate batch of this many tokens (decode runs: "
                         "--tokens 1 --calib-tokens 2048); 0 = calibrate on the timed batch itself")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    from paper_2602_20191_b200.stack import MobiStack
    t0 = time.time()
    stack = MobiStack(blocks=args.blocks, device=local, seed=args.seed,
                      max_tokens=max(args.tokens, args.calib_tokens), concurrent=args.concurrent)
    build_s = time.time() - t0
    g = torch.Generator(device="cuda").manual_seed(args.seed * 7919 + rank)
    pool = max(args.tokens, args.calib_tokens)
    x = torch.randn((pool, stack.d), generator=g, device="cuda")
    ch = torch.randperm(stack.d, generator=g, device="cuda")[: round(0.05 * stack.d)]
    x[:, ch] *= 8.0
    x = x.to(torch.bfloat16)
    xcal, x = x, x[: args.tokens].contiguous()
    from paper_2602_20191_b200.layer import avg_bits_from_masks
    for target in args.targets:
        res = stack.sweep_point(xcal, target)
        deltas = {id(layer): d for layer, d in zip(stack.layers, res.per_layer_delta)}
        masks: list = []
        stack.forward(x, deltas, masks)  # the timed batch's own masks
        timed_bits = [avg_bits_from_masks(m, [2, 2, 2, 2]) for m in masks]
        # slice-code bytes the timed batch's masks select (union over its tokens, per layer): the decode
        # kernels read exactly the planes some token needs, so at T=1 this is the weight traffic
        union_bytes = 0
        for layer, m in zip(stack.layers, masks):
            u = functools.reduce(lambda a, b: a | b, torch.unique(m).tolist(), 0)
            union_bytes += layer.out * layer.inn * 2 * bin(u).count("1") // 8
        graph, _ = stack.capture(x, deltas)
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        if world > 1:
            t = torch.tensor([ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        del graph
        if rank == 0:
            print(json.dumps({
                "config": "llama3-8b MoBi stack", "blocks": args.blocks, "linears": 7 * args.blocks,
                "tokens_per_gpu": args.tokens, "n_gpus": world, "parallelism": f"replicas, token-sharded x{world}",
                "target_bits": target, "realized_avg_bits": round(res.realized_bits, 4),
                "criterion6_within_0.15": abs(res.realized_bits - target) <= 0.15,
                "per_layer_bits_min": round(min(res.per_layer_bits), 4),
                "per_layer_bits_max": round(max(res.per_layer_bits), 4),
                "calib_tokens": args.calib_tokens or args.tokens,
                "branches": "q/k/v and gate/up as parallel graph branches" if args.concurrent else "serial",
                "timed_batch_avg_bits": round(float(sum(timed_bits) / len(timed_bits)), 4),
                "slice_code_bytes_selected": union_bytes,
                "slice_code_GBps": round(union_bytes / (ms / 1e3) / 1e9, 1),
                "ms_per_forward": round(ms, 3), "tokens_per_s": round(args.tokens * world / (ms / 1e3), 1),
                "device_gib": round(stack.device_bytes() / 2**30, 2), "build_s": round(build_s, 1),
                "data": "random-init slices (uniform 2-bit codes, unit-gain group scales), calibset-style X"}),
                flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
