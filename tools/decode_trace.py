"""Development tool: per-CTA globaltimer marks of the decode router + decode GEMM (debug impl 9)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2602_20191_b200 import _lib, calibrate_threshold  # noqa: E402


def main():
    args = bench.parse()
    bench.workload(args, 1)
    dev = torch.device("cuda", 0)
    layer, _ = bench.make_layer(args, dev, 1)
    x = bench.make_x(args, dev, 2)
    delta = calibrate_threshold(layer.score(x), (args.target_bits - 2) / 6)
    for _ in range(5):
        layer.forward(x, delta)
    layer.set_debug_impl(9)
    # replay from a CUDA graph, as bench.py does at decode sizes: the PDL edge only overlaps the two
    # kernels when the dependent launch is already queued on the device
    y = torch.empty((x.shape[0], layer.out), dtype=torch.bfloat16, device=dev)
    layer.forward(x, delta, y=y)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            layer.forward(x, delta, y=y)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    layer.set_debug_impl(0)
    full = np.zeros(32 * 1024, np.uint64)
    lib = _lib.lib()
    lib.mobi_debug_read_trace.argtypes = [C.c_void_p, C.c_int]
    _lib.check(lib.mobi_debug_read_trace(full.ctypes.data, 1))
    t = full.astype(np.int64).reshape(-1, 8)
    r, g = t[:2048], t[2048:4096]
    r = r[r[:, 0] > 0]
    g = g[g[:, 0] > 0]
    t0 = min(r[:, 0].min() if len(r) else 1 << 62, g[:, 0].min())
    def show(name, a, cols):
        for i, c in enumerate(cols):
            v = a[:, i]
            v = v[v > 0] - t0
            if len(v):
                print(f"{name:7s} {c:28s} n={len(v):4d}  min {v.min():8d}  med {int(np.median(v)):8d}  max {v.max():8d} ns")
    show("router", r, ["start", "loads done", "split arrived", "tile epilogue done", "final masks"])
    if len(g):
        cyc = (g[:, 5] - g[:, 7]).astype(np.float64)
        ns = (g[:, 6] - g[:, 0]).astype(np.float64)
        ok = (g[:, 5] > 0) & (ns > 0)
        if ok.any():
            print("gemm SM clock (GHz, median over CTAs):", float(np.median(cyc[ok] / ns[ok])))
    if False: show("gemm", g, ["start", "x prep done", "grid dep resolved", "main loop done", "end"])
    show("planes", g, ["start", "x prep done", "slice 1 done", "grid dep resolved", "union slices done", "end",
                       "x token 0 loaded", "x last token loaded"])
    it = full.astype(np.int64)[24576:24576 + 16 * 32 * 4].reshape(16, 32, 4)
    for w in (0, 5, 15):
        print(f"planes CTA0 warp {w} per item (ns rel. kernel start: pre-wait, data, mma done, issued):")
        for ci in range(32):
            if it[w, ci, 0]:
                print("   ", ci, [int(v - t0) for v in it[w, ci]])
    return
    ft = full.astype(np.int64)[24576:24576 + 4 * 64].reshape(4, 64)
    for c in range(2):
        print(f"cta {c} warp7 full-wait start:", [int(v - t0) if v else -1 for v in ft[c, :16]])
        print(f"cta {c} warp7 full-wait done:", [int(v - t0) if v else -1 for v in ft[c, 32:48]])
        rf = full.astype(np.int64)[24576 + 256 + c * 64: 24576 + 256 + c * 64 + 16]
        print(f"cta {c} refill issue (it):  ", [int(v - t0) if v else -1 for v in rf])


if __name__ == "__main__":
    main()
