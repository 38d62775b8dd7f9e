"""Model-level driver: a LLaMA3-8B-shaped stack of MoBi linear layers (BASELINE config 5).

The reference's model-level loop is ``bench::eval_at_ratio`` (pipeline.hpp:125-218): for every layer it
pools the router scores of the calibration tokens, sets the layer's threshold with
``calibrate_threshold(pooled, rho)`` (router.hpp:167-174), gates, runs ``forward_elastic`` and feeds
``silu(y)`` to the next layer; the realized bits are averaged over tokens, then over layers
(router.hpp:135-150, pipeline.hpp:191-213).  Here the same loop runs over the seven linears of each of
LLaMA3-8B's 32 blocks (q/o 4096x4096, k/v 1024x4096, gate/up 14336x4096, down 4096x14336), every one a
device-resident MobiLayer, chained as a synthetic pre-norm block without attention (n = RMSNorm
without a learned gain, as LLaMA's pre-attention / pre-MLP norms):

    a = n(h);  q, k, v = Lq(a), Lk(a), Lv(a);  h = h + Lo(silu(q));
    b = n(h);  h = h + Ld(silu(Lg(b)) * Lu(b))

(k and v are computed -- their bytes and flops are part of the block -- but only q feeds forward).
Weights are random-init slices: i.i.d. uniform 2-bit codes with group scales sized for unit gain,
routers per ``RouterState::init`` with ``w2 = 0.3 N(0,1)``, ``b2 = 0.1 N(0,1)`` (tools/mobi.cpp:211).
Forwards replay as one CUDA graph per (budget, batch) so the 224 x 3 launches cost one host call.
With ``concurrent=True`` the linears that share an input (q/k/v on ``a``, gate/up on ``b``) run on side
streams, so the graph holds them as parallel branches.  Measured on the 32-block stack at T = 1
(tools/stack_sweep.py, three alternating runs): 5.31 vs 5.06 ms at 2 bits and 5.48-5.78 vs 5.59-5.61 ms
at 3 bits -- the decode pairs rely on the router and plane GEMV being co-resident on each SM, which
concurrent layers break -- so the default is serial.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np
import torch

LLAMA3_8B = dict(d=4096, kv=1024, ffn=14336, blocks=32)
LINEARS = ("q", "k", "v", "o", "gate", "up", "down")


def rmsnorm(h: torch.Tensor, eps: float = 1e-5) -> torch.Tensor:
    f = h.float()
    return (f * torch.rsqrt(f.pow(2).mean(dim=-1, keepdim=True) + eps)).to(h.dtype)


def linear_shapes(cfg=LLAMA3_8B) -> Dict[str, tuple]:
    d, kv, f = cfg["d"], cfg["kv"], cfg["ffn"]
    return {"q": (d, d), "k": (kv, d), "v": (kv, d), "o": (d, d), "gate": (f, d), "up": (f, d), "down": (d, f)}


def random_layer(out: int, inn: int, *, gs: int = 128, hidden: int = 0, gen: torch.Generator, device: int):
    """One random-init MoBi layer (2+2+2+2 slices) built on the device."""
    from .layer import MobiLayer
    dev = torch.device("cuda", device)
    codes = torch.randint(0, 4, (4, out, inn), generator=gen, device=dev, dtype=torch.uint8)
    G = -(-inn // gs)
    # W = s * (F - z) with F roughly uniform on [0, 4): unit gain needs std(W) ~ 1/sqrt(in)
    s0 = 1.0 / (math.sqrt(inn) * 4.0 / math.sqrt(12.0))
    scale = (s0 * (0.8 + 0.4 * torch.rand(out * G, generator=gen, device=dev, dtype=torch.float64))).cpu().numpy()
    zero = (2.0 + 0.1 * torch.randn(out * G, generator=gen, device=dev, dtype=torch.float64)).cpu().numpy()
    h = hidden or max(1, inn // 4)
    w1 = (torch.randn((inn, h), generator=gen, device=dev) / math.sqrt(inn)).double().cpu().numpy()
    w2 = (0.3 * torch.randn((h, 3), generator=gen, device=dev)).double().cpu().numpy()
    b2 = (0.1 * torch.randn(3, generator=gen, device=dev)).double().cpu().numpy()
    layer = MobiLayer.from_device_stack(codes, [2, 2, 2, 2], scale, zero, gs, w1, np.zeros(h), w2, b2)
    del codes
    return layer


@dataclass
class StackResult:
    target_bits: float
    realized_bits: float
    per_layer_bits: List[float] = field(default_factory=list)
    per_layer_delta: List[float] = field(default_factory=list)


class MobiStack:
    """LLaMA3-8B-shaped stack of MobiLayers on one GPU (replicated per rank for token-sharded runs)."""

    def __init__(self, blocks: int = LLAMA3_8B["blocks"], device: int = 0, seed: int = 1, cfg=LLAMA3_8B,
                 max_tokens: int = 2048, concurrent: bool = False):
        self.device = device
        self.concurrent = concurrent
        self._side = [torch.cuda.Stream(device=device) for _ in range(2)]
        self.shapes = linear_shapes(cfg)
        self.d = cfg["d"]
        gen = torch.Generator(device=torch.device("cuda", device)).manual_seed(seed)
        self.blocks: List[Dict[str, object]] = []
        for _ in range(blocks):
            blk = {n: random_layer(*self.shapes[n], gen=gen, device=device) for n in LINEARS}
            for layer in blk.values():
                layer.reserve(max_tokens)
            self.blocks.append(blk)
        self.layers = [blk[n] for blk in self.blocks for n in LINEARS]
        if not concurrent:  # serial layers: one permuted-activation buffer for the whole stack
            from .layer import share_activations
            share_activations(self.layers)

    def device_bytes(self) -> int:
        return sum(layer.device_bytes() for layer in self.layers)

    # ---------------- the block ----------------
    def _block(self, blk, h, deltas, masks: Optional[list]):
        res: Dict[str, tuple] = {}

        def lin(name, x):
            res[name] = blk[name].forward(x, deltas[id(blk[name])], return_masks=True)
            return res[name][0]

        def branches(names, x):
            """names[0] on the current stream, the others on side streams (joined before returning)."""
            if not self.concurrent:
                for n in names:
                    lin(n, x)
                return
            cur = torch.cuda.current_stream()
            for s in self._side[: len(names) - 1]:
                s.wait_stream(cur)
            for n, s in zip(names[1:], self._side):
                with torch.cuda.stream(s):
                    lin(n, x)
            lin(names[0], x)
            for n, s in zip(names[1:], self._side):
                cur.wait_stream(s)
                res[n][0].record_stream(cur)
                res[n][1].record_stream(cur)

        a = rmsnorm(h)
        branches(("q", "k", "v"), a)
        h = h + lin("o", torch.nn.functional.silu(res["q"][0]))
        b = rmsnorm(h)
        branches(("gate", "up"), b)
        h = h + lin("down", torch.nn.functional.silu(res["gate"][0]) * res["up"][0])
        if masks is not None:
            masks.extend(res[n][1] for n in LINEARS)
        return h

    def forward(self, x: torch.Tensor, deltas: Dict[int, float], masks: Optional[list] = None) -> torch.Tensor:
        h = x
        for blk in self.blocks:
            h = self._block(blk, h, deltas, masks)
        return h

    # ---------------- calibration (pipeline.hpp:146-160) ----------------
    def calibrate(self, x: torch.Tensor, target_bits: float) -> Dict[int, float]:
        """Per-layer delta = calibrate_threshold(pooled scores of the layer's own input, rho(target)),
        filled in as the stack runs (each layer's input depends on the thresholds before it)."""
        from .layer import calibrate_threshold, ratio_from_target_bits
        rho = ratio_from_target_bits(target_bits, [2, 2, 2, 2])
        deltas: Dict[int, float] = {}

        h = x
        for blk in self.blocks:
            def lin(name, inp, blk=blk):
                layer = blk[name]
                deltas[id(layer)] = calibrate_threshold(layer.score(inp), rho)
                return layer.forward(inp, deltas[id(layer)])
            a = rmsnorm(h)
            q = lin("q", a)
            lin("k", a)
            lin("v", a)
            h = h + lin("o", torch.nn.functional.silu(q))
            b = rmsnorm(h)
            g = lin("gate", b)
            u = lin("up", b)
            h = h + lin("down", torch.nn.functional.silu(g) * u)
        return deltas

    def realized_bits(self, x: torch.Tensor, deltas: Dict[int, float]) -> List[float]:
        """Per-layer realized bits (router.hpp:135-150) on x."""
        from .layer import avg_bits_from_masks
        masks: list = []
        self.forward(x, deltas, masks)
        return [avg_bits_from_masks(m, [2, 2, 2, 2]) for m in masks]

    def sweep_point(self, x: torch.Tensor, target_bits: float) -> StackResult:
        deltas = self.calibrate(x, target_bits)
        bits = self.realized_bits(x, deltas)
        return StackResult(target_bits, float(np.mean(bits)), bits, [deltas[id(layer)] for layer in self.layers])

    def capture(self, x: torch.Tensor, deltas: Dict[int, float]):
        """One CUDA graph of the whole stack forward on the static input x; returns (graph, output)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.forward(x, deltas)  # warm the workspaces outside capture
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                out = self.forward(x, deltas)
        torch.cuda.current_stream().wait_stream(s)
        return g, out
