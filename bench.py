#!/usr/bin/env python
"""MoBi-linear benchmark (BASELINE.json metric: tokens/s at LLaMA3-8B shapes vs avg bits,
% of tensor/HBM roofline).

  python bench.py [--gpus N --steps K --warmup W] [--out --in --tokens --target-bits --hidden]
  python bench.py --gpus N ...            (N > 1 without torchrun: re-launches itself under torchrun)
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
  python bench.py --impl reference ...    (the reference's own CPU implementation, oracle/_ref)

Workloads (synthetic data; random-init slices of LLaMA3-8B shapes):
  * N = 1 (configs[1]): q_proj 4096x4096, T = 2048 tokens per step, 3.0 average bits (rho = 1/6 of
    the pooled routed scores above delta), router h = in/4, group 128, slices 2+2+2+2.
  * N > 1 (configs[3]): MLP gate/up 14336x4096, T = 8192 tokens per step, column-parallel: every rank
    owns out/N weight rows (router replicated), one all-gather of the [T, out/N] outputs (strong
    scaling: total work fixed).  ``--parallel token`` instead runs token-sharded replicas (weak).
Synthetic data: W ~ N(0, 0.02^2) sliced by the GPU decompose (bit-exact with the reference), router
per RouterState::init with w2 = 0.3 N(0,1), b2 = 0.1 N(0,1) (tools/mobi.cpp:211), X per gen_calibset
(N(0,1), 5% channels x8).  delta comes from the batch's own pooled scores (eval_at_ratio,
pipeline.hpp:146-160); decode-size batches (T <= 32) take it from a 4096-token calibration pool.

A step = one full layer forward (route -> bucket -> gather -> tcgen05 GEMM + un-permute) over one
batch.  L2 hygiene: the step cycles through a ring of R independent (layer, X, Y) triples whose
combined footprint exceeds 2x the 126 MB L2, so no step finds its inputs in L2.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

L2_BYTES = 126 * 1024 * 1024
DECODE_MAX_T = 32  # the C-ABI's decode path
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
METRIC = "MoBi-linear tokens/s at LLaMA3-8B shapes vs avg bits; % of TC/HBM roofline"
SLICE_BITS = [2, 2, 2, 2]


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="mobi", choices=["mobi", "reference"])
    p.add_argument("--out", type=int, default=None)
    p.add_argument("--in", dest="inn", type=int, default=None)
    p.add_argument("--tokens", type=int, default=None)
    p.add_argument("--target-bits", type=float, default=3.0)
    p.add_argument("--hidden", type=int, default=0, help="router hidden width (0 = in/4, the reference default)")
    p.add_argument("--group-size", type=int, default=128)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--cpu-threads", type=int, default=0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--ring", type=int, default=0)
    p.add_argument("--parallel", default=None, choices=["token", "column"],
                   help="N>1: column-parallel rows + all-gather (default, configs[3]) or token-sharded replicas")
    p.add_argument("--graph", action="store_true",
                   help="replay each ring slot's forward from a captured CUDA graph (default for decode-size T)")
    args = p.parse_args(argv)
    return args


def workload(args, world):
    """Fill the shape defaults: configs[1] at N = 1, configs[3] (column-parallel MLP prefill) at N > 1."""
    if args.parallel is None:
        args.parallel = "column" if world > 1 else "token"
    mlp = world > 1 and args.parallel == "column"
    if args.out is None:
        args.out = 14336 if mlp else 4096
    if args.inn is None:
        args.inn = 4096
    if args.tokens is None:
        args.tokens = 8192 if mlp else 2048
    h = args.hidden if args.hidden else max(1, args.inn // 4)
    names = {(4096, 4096): "q/o proj", (1024, 4096): "k/v proj", (14336, 4096): "MLP gate/up",
             (4096, 14336): "MLP down"}
    name = names.get((args.out, args.inn), "linear")
    column = args.parallel == "column" and world > 1
    return {"workload": f"llama3-8b {name} {args.out}x{args.inn}, MoBi 2+2+2+2 slices, T={args.tokens} tokens "
                        f"{'per step (all ranks)' if column else 'per GPU per step'}, target {args.target_bits} avg "
                        f"bits, router h={h}",
            "out": args.out, "in": args.inn, "tokens_per_step": args.tokens * (1 if column else world),
            "tokens_per_gpu": args.tokens, "target_bits": args.target_bits, "group_size": args.group_size,
            "router_hidden": h,
            "parallelism": (f"column-parallel x{world} (weight rows split, router replicated, all-gather of Y)"
                            if column else f"token-sharded x{world} (replicas, no collective)" if world > 1
                            else "single GPU")}


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        return json.loads(f.read_text()), "measured"
    return dict(FALLBACK_PEAKS), "fallback"


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


# ------------------------------------------------------------------------------------------
# multi-GPU launch: re-exec under torchrun when --gpus N > 1 is given without a process group
# ------------------------------------------------------------------------------------------
def spawn_if_needed(args, argv):
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if args.impl == "mobi":
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {n} CUDA device(s) visible")
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + list(argv)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------------------------------------
# clocks sampler (NVML polled on the host while the timed region runs; nvidia-smi fallback)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.nvml = None
        self.samples = []

    def _nvml_sample(self):
        nv, h = self.nvml
        try:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            self.samples.append((sm, smax, fn(h)))
        except Exception:
            pass

    def poll_until(self, event):
        if not self.nvml:
            return
        self._nvml_sample()
        while not event.query():
            self._nvml_sample()
            time.sleep(0.0005)

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml = (nv, nv.nvmlDeviceGetHandleByIndex(self.dev))
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.nvml:
            nv = self.nvml[0]
            bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4}
            reasons = sorted({n for _, _, r in self.samples for n, b in bits.items() if r & b})
            if not self.samples:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": reasons, "samples": 0, "source": "nvml"}
            return {"sm_mhz": statistics.median([a for a, _, _ in self.samples]),
                    "sm_max_mhz": max(b for _, b, _ in self.samples), "reasons": reasons,
                    "samples": len(self.samples), "source": "nvml, polled while the timed region ran"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# GPU workload
# ------------------------------------------------------------------------------------------
def make_stack(args, dev, seed):
    import torch
    from paper_2602_20191_b200 import decompose
    g = torch.Generator(device=dev).manual_seed(seed)
    out, inn, gs = args.out, args.inn, args.group_size
    h = args.hidden if args.hidden else max(1, inn // 4)
    w = torch.randn((out, inn), generator=g, device=dev, dtype=torch.float64) * 0.02
    codes, scale, zero, _ = decompose(w, gs, SLICE_BITS, 4.0)
    del w
    w1 = torch.randn((inn, h), generator=g, device=dev, dtype=torch.float64) / math.sqrt(inn)
    w2 = torch.randn((h, 3), generator=g, device=dev, dtype=torch.float64) * 0.3
    b2 = torch.randn(3, generator=g, device=dev, dtype=torch.float64) * 0.1
    return dict(codes=codes, scale=scale.cpu().numpy(), zero=zero.cpu().numpy(), w1=w1.cpu().numpy(),
                b1=np.zeros(h), w2=w2.cpu().numpy(), b2=b2.cpu().numpy())


def make_layer(args, dev, seed):
    from paper_2602_20191_b200 import MobiLayer
    st = make_stack(args, dev, seed)
    layer = MobiLayer.from_device_stack(st["codes"], SLICE_BITS, st["scale"], st["zero"], args.group_size, st["w1"],
                                        st["b1"], st["w2"], st["b2"])
    return layer, st


def make_x(args, dev, seed, T=None):
    import torch
    T = T or args.tokens
    g = torch.Generator(device=dev).manual_seed(seed)
    x = torch.randn((T, args.inn), generator=g, device=dev)
    n_out = max(1, round(0.05 * args.inn))
    ch = torch.randperm(args.inn, generator=g, device=dev)[:n_out]
    x[:, ch] *= 8.0
    return x.to(torch.bfloat16)


def gemm_flops(args, T):
    # the kernel folds a bucket's active slices into one effective weight (one MMA per k-step),
    # so its algorithmic work is the dense contraction 2*T*in*out
    return 2.0 * T * args.inn * args.out


def router_flops(args, T):
    h = args.hidden if args.hidden else max(1, args.inn // 4)
    return 2.0 * T * (args.inn * h + 3 * h)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    rc = spawn_if_needed(args, argv)
    if rc is not None:
        return rc
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.gpus != world:
        raise SystemExit(f"bench.py --gpus {args.gpus} launched with WORLD_SIZE={world}")
    config = workload(args, world)
    if args.impl == "reference":
        return main_reference(args, rank, world, config)
    return main_mobi(args, rank, world, local, config)


def main_mobi(args, rank, world, local, config):
    import torch
    from paper_2602_20191_b200 import avg_bits_from_masks, calibrate_threshold, ratio_from_target_bits
    dist = world > 1
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if dist:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=dev)
    column = dist and args.parallel == "column"
    T = args.tokens
    rho = ratio_from_target_bits(args.target_bits, SLICE_BITS)
    per_step_bytes = args.out * args.inn + 2 * T * args.inn * 2 + T * args.out * 2
    R = args.ring or max(1, math.ceil(2 * L2_BYTES / per_step_bytes))
    R = min(R, 16 if args.out * args.inn <= 2 ** 24 else 6)
    ring = []
    for i in range(R):
        seed = args.seed * 1000 + i  # identical layers on every rank (replicas / shards of one layer)
        st = make_stack(args, dev, seed)
        # column-parallel: every rank sees the same tokens; token-sharded: every rank its own
        x = make_x(args, dev, args.seed * 7919 + (0 if column else 104729 * rank) + i)
        if column:
            from paper_2602_20191_b200.sharding import ColumnParallelMobiLayer
            layer = ColumnParallelMobiLayer(st["codes"].cpu().numpy(), SLICE_BITS, st["scale"], st["zero"],
                                            args.group_size, st["w1"], st["b1"], st["w2"], st["b2"], device=local,
                                            rank=rank, world=world)
        else:
            from paper_2602_20191_b200 import MobiLayer
            layer = MobiLayer.from_device_stack(st["codes"], SLICE_BITS, st["scale"], st["zero"], args.group_size,
                                                st["w1"], st["b1"], st["w2"], st["b2"])
        # delta pooled over the batch's own scores (eval_at_ratio); decode sizes: a 4096-token pool
        xcal = x if T > DECODE_MAX_T else make_x(args, dev, args.seed * 31 + i, T=4096)
        delta = calibrate_threshold(layer.score(xcal), rho)
        layer.reserve(T)
        y = torch.empty((T, args.out), dtype=torch.bfloat16, device=dev)
        ring.append(dict(layer=layer, host=st if i == 0 else None, x=x, y=y, delta=delta))
        del st
    config["l2"] = f"ring of {R} independent layer/X/Y sets ({R * per_step_bytes / 2**20:.0f} MiB > 2x L2)"
    config["delta"] = ("batch's own pooled scores" if T > DECODE_MAX_T else
                       "4096-token calibration pool per layer (decode batches are too small to pool)")

    def step(i, masks=False):
        r = ring[i % R]
        return r["layer"].forward(r["x"], r["delta"], y=r["y"], return_masks=masks)

    for i in range(max(3, args.warmup)):
        step(i)
    torch.cuda.synchronize()
    graphs = None
    if (args.graph or T <= 64) and not column:  # decode sizes: host launch overhead would dominate
        graphs = []
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            for r in ring:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cs):
                    r["layer"].forward(r["x"], r["delta"], y=r["y"])
                graphs.append(g)
            ring_graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(ring_graph, stream=cs):
                for r in ring:
                    r["layer"].forward(r["x"], r["delta"], y=r["y"])
        torch.cuda.current_stream().wait_stream(cs)
        for i in range(max(3, args.warmup)):
            graphs[i % R].replay()
        ring_graph.replay()
        torch.cuda.synchronize()
        config["launch"] = (f"CUDA graphs: the ring's {R} forwards captured as one graph (replayed steps//{R} "
                            f"times) + per-slot graphs for the remainder")
    clk = ClockSampler(local)
    clk.start()
    if not clk.nvml:
        time.sleep(0.05)
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    per_step_launches = [r["layer"].last_launches() for r in ring]
    e0.record(stream)
    if graphs is not None:
        for _ in range(args.steps // R):
            ring_graph.replay()
        for i in range(args.steps - args.steps % R, args.steps):
            graphs[i % R].replay()
        launches = sum(per_step_launches[i % R] for i in range(args.steps))
    else:
        for i in range(args.steps):
            step(i)
            launches += ring[i % R]["layer"].last_launches()
    e1.record(stream)
    clk.poll_until(e1)
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    tokens_total = T * args.steps * (1 if column else world)
    value = tokens_total / (ms / 1e3)

    # which kernels the step ran (mobi_layer_last_plan) and the realized bits over every ring entry's
    # tokens (decode batches of 1..32 tokens realize 2/4/6/8 bits each: the budget shows over the ring)
    ms_all = []
    for i in range(R):
        _, m = step(i, masks=True)
        ms_all.append(m)
    plan = ring[0]["layer"].last_plan() if hasattr(ring[0]["layer"], "last_plan") else \
        ring[0]["layer"].local.last_plan()
    m = torch.cat(ms_all)
    realized = avg_bits_from_masks(m, SLICE_BITS)
    counts = torch.bincount(m.to(torch.int64), minlength=16).cpu().tolist()
    config["realized_avg_bits"] = round(realized, 4)
    config["realized_over_tokens"] = int(m.numel())
    config["buckets"] = {str(i): c for i, c in enumerate(counts) if c}
    config["kernels"] = {k: plan[k] for k in ("router", "gemm", "gemm_ctas", "token_tiles", "units")}

    # per-kernel device times: an eager pass after the timed region with CUDA events around every
    # launch, queued behind a device spin (device time only; PDL overlap disabled in this pass)
    for r in ring:
        r["layer"].profile(True)
    torch.cuda._sleep(int(2e7))
    for i in range(min(args.steps, 50)):
        step(i)
    torch.cuda.synchronize()
    config["kernel_times"] = ("eager profiled pass after the timed region, launches queued behind a device spin "
                              "(no host gaps, no PDL overlap)")
    kern = {k: [0.0, 0] for k in ("router", "bucket", "gather", "gemm")}
    for r in ring:
        for k, (t_ms, n) in r["layer"].profile_read().items():
            kern[k][0] += t_ms
            kern[k][1] += n
        r["layer"].profile(False)

    pk, pk_src = peaks()
    peak_tf = pk.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"])
    hbm = pk.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"])
    rows = args.out // world if column else args.out  # this rank's weight rows
    gemm_ms = kern["gemm"][0] / max(1, kern["gemm"][1])
    router_ms = kern["router"][0] / max(1, kern["router"][1])
    G = math.ceil(args.inn / args.group_size)
    h_s = args.hidden or args.inn // 4
    step_ms = ms / args.steps
    if plan["gemm"] in ("decode_planes", "decode_merged"):
        # decode sizes are HBM-bound: algorithmic bytes = the union of the batch's active
        # slices (2 bits each per weight) + group constants (s, s*z) + activations in/out
        union = 0
        for v in (int(k) for k in config["buckets"]):
            union |= v
        n_sl = bin(union).count("1")
        alg = rows * args.inn * 2 * n_sl / 8 + rows * G * 8 + T * (args.inn + rows) * 2
        streamed = alg if plan["gemm"] == "decode_planes" else rows * args.inn + rows * G * 8 + T * (args.inn + rows) * 2
        gb = alg / (gemm_ms * 1e-3) / 1e9
        step_bytes = alg + args.inn * h_s * 2  # + the router's w1 (bf16), read once per step
        roofline = {"bound": "hbm", "achieved": round(gb, 1), "peak": hbm, "unit": "GB/s", "frac": round(gb / hbm, 4),
                    "traffic": None, "kernel": plan["gemm"],
                    "bytes_per_launch": alg,
                    "bytes_basis": f"union of active slices ({n_sl} of 4) x 2 bit/weight + group constants 8 B/group "
                                   f"+ bf16 X and Y; the kernel streams {streamed:.0f} B/launch; kernel time from the "
                                   "eager profiled pass (no router overlap)",
                    "step": {"bytes": step_bytes, "ms": round(step_ms, 5),
                             "gbs": round(step_bytes / (step_ms * 1e-3) / 1e9, 1),
                             "frac": round(step_bytes / (step_ms * 1e-3) / 1e9 / hbm, 4),
                             "basis": "whole decode step (router w1 + the GEMV's algorithmic bytes) over the timed "
                                      "per-step time: the kernels overlap under PDL"},
                    "peak_source": f"{pk_src} HBM copy bandwidth (MEASURED_PEAKS.json hbm_gbs)"}
    else:
        f_gemm = 2.0 * T * args.inn * rows
        achieved = f_gemm / (gemm_ms * 1e-3) / 1e12
        traffic = None
        tf = ROOT / "profiles" / "gemm_traffic.json"
        if tf.exists():
            d = json.loads(tf.read_text())
            if d.get("out") == rows and d.get("in") == args.inn and d.get("tokens") == T:
                traffic = d.get("dram_bytes_per_launch")
        roofline = {"bound": "tensor", "achieved": round(achieved, 2), "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": round(achieved / peak_tf, 4), "traffic": traffic, "kernel": plan["gemm"],
                    "flops_per_launch": f_gemm,
                    "flops_basis": "dense 2*T*in*rows (bucket slices folded into one effective weight per MMA)",
                    "peak_source": f"{pk_src} burst bf16 (MEASURED_PEAKS.json bf16_tflops)"}
        # whole step: router + GEMM flops and the step's bytes against both roofs;
        # time_lb = max(F / P_tc, B / P_hbm), achieved = time_lb / measured step time
        f_step = f_gemm + router_flops(args, T)
        b_step = rows * args.inn * 2 * 4 / 8 + rows * G * 8 + args.inn * h_s * 2 + T * (args.inn + rows) * 2
        t_tc = f_step / (peak_tf * 1e12) * 1e3
        t_hbm = b_step / (hbm * 1e9) * 1e3
        roofline["step"] = {"flops": f_step, "bytes": b_step, "ms": round(step_ms, 5),
                            "tflops": round(f_step / (step_ms * 1e-3) / 1e12, 1),
                            "time_lb_ms": round(max(t_tc, t_hbm), 5), "binds": "tensor" if t_tc >= t_hbm else "hbm",
                            "achieved": round(max(t_tc, t_hbm) / step_ms, 4),
                            "basis": "router 2*T*(in*h+3h) + dense GEMM 2*T*in*rows flops; bytes = all 4 slices' "
                                     "codes (2 bit each) + group constants + router w1 + X/Y"
                                     + ("; the step includes the all-gather" if column else "")}
    router_bytes = args.inn * h_s * 2 + T * args.inn * 2
    kernels = {k: {"ms_per_launch": round(v[0] / max(1, v[1]), 5), "launches": v[1],
                   "share": round(v[0] / max(1e-9, sum(x[0] for x in kern.values())), 4)} for k, v in kern.items()}
    if router_ms:
        kernels["router"]["kernel"] = plan["router"]
        kernels["router"]["tflops"] = round(router_flops(args, T) / (router_ms * 1e-3) / 1e12, 2)
        kernels["router"]["frac_tensor"] = round(kernels["router"]["tflops"] / peak_tf, 4)
        kernels["router"]["gbs"] = round(router_bytes / (router_ms * 1e-3) / 1e9, 1)
        kernels["router"]["frac_hbm"] = round(kernels["router"]["gbs"] / hbm, 4)
    if kern["gather"][1]:
        kernels["gather"]["gbs"] = round(2 * T * args.inn * 2 / (kernels["gather"]["ms_per_launch"] * 1e-3) / 1e9, 1)
    if dist:  # per-rank roofline fractions, gathered so rank 0 reports them all
        mine = torch.tensor([roofline["frac"], roofline.get("step", {}).get("achieved", 0.0)], device=dev,
                            dtype=torch.float64)
        allr = [torch.zeros_like(mine) for _ in range(world)]
        tdist.all_gather(allr, mine)
        roofline["per_rank_frac"] = [round(float(a[0]), 4) for a in allr]

    # ---------------- e2e through the public host-buffer API ----------------
    e2e = None
    if not args.no_e2e:
        r = ring[0]
        xh = r["x"].cpu().pin_memory()
        yh = torch.empty((T, args.out), dtype=torch.bfloat16).pin_memory()
        mh = torch.empty(T, dtype=torch.uint8).pin_memory()
        for _ in range(10):
            r["layer"].forward_host(xh, r["delta"], y_host=yh, masks_host=mh)
        if dist:
            tdist.barrier()
        torch.cuda.synchronize()
        # five back-to-back windows; the median window is reported (the calls are synchronous, copies
        # included), which keeps a transient host or PCIe hiccup in one window from setting the number
        k2 = 5 * max(1, min(args.steps, 50) // 5)
        windows = []
        for _w in range(5):
            t0 = time.perf_counter()
            for _ in range(k2 // 5):
                r["layer"].forward_host(xh, r["delta"], y_host=yh, masks_host=mh)
            torch.cuda.synchronize()
            windows.append(time.perf_counter() - t0)
        wall = sorted(windows)[2] * 5
        if dist:
            t = torch.tensor([wall], device=dev, dtype=torch.float64)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            wall = float(t.item())
        e2e = {"value": round(T * k2 * (1 if column else world) / wall, 1), "unit": "tokens/s",
               "h2d_bytes_per_step": T * args.inn * 2,
               "d2h_bytes_per_step": T * args.out * 2 + T,
               "steps": k2, "windows_ms_per_step": [round(w / (k2 // 5) * 1e3, 4) for w in windows],
               "api": "mobi_forward_host (pinned host bf16 in/out, synchronous); median of 5 windows"}

    # ---------------- CPU baseline (rank 0, N=1): the reference itself ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            h0 = ring[0]["host"]
            host = dict(codes=h0["codes"].cpu().numpy(), scale=h0["scale"], zero=h0["zero"], w1=h0["w1"], b1=h0["b1"],
                        w2=h0["w2"], b2=h0["b2"])
            cpu = reference_sample(args, host, ring[0]["x"][:64].double().cpu().numpy(), ring[0]["delta"], steps=1)
        except Exception as ex:  # the baseline is reported, never a reason to fail the bench
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference", "sample": f"failed: {ex}"}

    line = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(step_ms, 5), "higher_is_better": True,
            "scaling": "strong" if column else "weak", "vs_baseline": None,
            "dtype": "fp16 operands (bf16 X rescaled per token by a power of two), fp32 accumulate, bf16 out",
            "data": "synthetic (W~N(0,0.02^2) GPU-decomposed, random-init router, calibset-style X)",
            "config": config, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks, "kernels": kernels, "hbm_peak_gbs": hbm}
    if column:
        line["collective"] = ring[0]["layer"].collective
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        tdist.barrier()
        tdist.destroy_process_group()
    return 0


# ------------------------------------------------------------------------------------------
# the reference's own CPU implementation (oracle/_ref: the unmodified reference headers compiled)
# ------------------------------------------------------------------------------------------
def ref_threads(args):
    return args.cpu_threads or max(1, min(os.cpu_count() or 1, 64))


def reference_forward(ref, host, x, delta, args, threads):
    """The reference's score -> gate_hard(delta) -> forward_elastic (router.hpp:63-132) over the tokens x,
    token-sharded for the router and row-sharded for forward_elastic across `threads` host threads."""
    f = ref.lib.ref_layer_forward_rowsharded
    P = lambda a: a.ctypes.data_as(C.c_void_p)
    x = np.ascontiguousarray(x, np.float64)
    T = x.shape[0]
    codes = np.ascontiguousarray(host["codes"], np.uint8)
    sb = np.array(SLICE_BITS, np.int32)
    arrs = {k: np.ascontiguousarray(host[k], np.float64) for k in ("scale", "zero", "w1", "b1", "w2", "b2")}
    h = arrs["w1"].shape[1]
    y = np.zeros((T, args.out))
    g = np.zeros((T, 3))
    t0 = time.perf_counter()
    rc = f(P(x), C.c_int64(T), C.c_int64(args.inn), P(codes), C.c_int32(4), P(sb), P(arrs["scale"]), P(arrs["zero"]),
           C.c_int64(args.out), C.c_int64(args.group_size), C.c_int64(h), P(arrs["w1"]), P(arrs["b1"]), P(arrs["w2"]),
           P(arrs["b2"]), C.c_double(delta), C.c_int(threads), P(g), P(y))
    dt = time.perf_counter() - t0
    if rc != 0:
        raise RuntimeError(ref.lib.ref_last_error().decode())
    return dt, y, g


def reference_sample(args, host, x, delta, steps):
    """Fixed cost (the per-call reconstruction of all slices, router.hpp:117-120) and per-token slope of
    the reference path, measured at two sample sizes; the reported rate is tokens/s at the larger one."""
    from oracle import oracle as O
    ref = O.reference()
    thr = ref_threads(args)
    t_big = min(x.shape[0], max(16, 2 * thr))
    t1, _, _ = reference_forward(ref, host, x[:1], delta, args, thr)
    times = [reference_forward(ref, host, x[:t_big], delta, args, thr)[0] for _ in range(steps)]
    tb = min(times)
    slope = max(0.0, (tb - t1) / max(1, t_big - 1))
    return {"value": round(t_big / tb, 3), "unit": "tokens/s", "cores": thr, "kind": "reference",
            "cpu_model": cpu_model(), "fixed_cost_s": round(t1, 4), "per_token_s": round(slope, 5),
            "sample": f"{t_big} tokens of the same layer/X/delta per call: reference score -> gate_hard -> "
                      f"forward_elastic (oracle/_ref, -O3, {thr} threads: router token-sharded, forward_elastic "
                      f"row-sharded); best of {steps}; fixed cost from a 1-token call"}


def main_reference(args, rank, world, config):
    """--impl reference: the reference's own CPU implementation on the box's host cores.  Builds its layer,
    scores and delta through the reference itself (oracle/_ref); never imports the product package."""
    if rank != 0:
        return 0
    from oracle import oracle as O
    ref = O.reference()
    thr = ref_threads(args)
    h = args.hidden if args.hidden else max(1, args.inn // 4)
    L = O.synthetic_layer(args.out, args.inn, seed=args.seed, group_size=args.group_size, hidden=h, backend=ref)
    host = {k: L[k] for k in ("codes", "scale", "zero", "w1", "b1", "w2", "b2")}
    xs, _ = O.gen_calibset(1, 256, args.inn, 0.05, 8.0, args.seed)
    xs = xs[0]
    # delta: calibrate_threshold over the pooled scores of a calibration sample (router.hpp:167-174)
    rho = ref.ratio_from_target_bits(args.target_bits, SLICE_BITS)
    t0 = time.perf_counter()
    s = ref.score(xs, L["w1"], L["b1"], L["w2"], L["b2"])
    t_score = time.perf_counter() - t0
    t0 = time.perf_counter()
    delta = ref.calibrate_threshold(s, rho)
    t_cal = time.perf_counter() - t0
    # each step: a bounded token sample sized so the whole run stays within ~3 minutes
    t1, _, _ = reference_forward(ref, host, xs[:1], delta, args, thr)
    budget = 150.0 / max(1, args.steps + args.warmup)
    per_tok_guess = 0.13 * (args.out * args.inn) / 4096 ** 2 / max(1, thr) * 4
    ts = int(max(1, min(256, (budget - t1) / max(1e-4, per_tok_guess))))
    for _ in range(args.warmup):
        reference_forward(ref, host, xs[:ts], delta, args, thr)
    times = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        times.append(reference_forward(ref, host, xs[:ts], delta, args, thr)[0])
    wall = time.perf_counter() - t_all
    value = ts * args.steps / wall
    slope = max(0.0, (min(times) - t1) / max(1, ts - 1))
    sample = (f"{ts} tokens per step of the same workload ({args.out}x{args.inn}, delta for {args.target_bits} bits "
              f"from {xs.shape[0]} calibration tokens); reference score -> gate_hard -> forward_elastic (oracle/_ref, "
              f"-O3), {thr} threads")
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "tokens/s",
                      "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                      "ms_per_step": round(wall / args.steps * 1e3, 3), "higher_is_better": True,
                      "scaling": "strong" if (world > 1 and args.parallel == "column") else "weak",
                      "vs_baseline": None, "dtype": "f64",
                      "data": "synthetic (same recipe as the GPU arm, generated on the host)", "config": config,
                      "cpu_baseline": {"value": round(value, 3), "unit": "tokens/s", "cores": thr, "kind": "reference",
                                       "cpu_model": cpu_model(), "sample": sample,
                                       "fixed_cost_s": round(t1, 4), "per_token_s": round(slope, 5),
                                       "calibrate_threshold_s": round(t_cal, 5),
                                       "score_s_per_token": round(t_score / xs.shape[0], 6)},
                      "e2e": {"value": round(value, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                              "d2h_bytes_per_step": 0}}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
