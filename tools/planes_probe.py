"""Development tool: the decode-planes GEMV alone (forward_masked, no router), timed with events and
traced (debug impl 9), for a few masks."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2602_20191_b200 import _lib, set_debug_impl  # noqa: E402


def main():
    args = bench.parse()
    dev = torch.device("cuda", 0)
    layer, _ = bench.make_layer(args, dev, 1)
    x = bench.make_x(args, dev, 2)
    for mval in (1, 3, 15):
        m = torch.full((args.tokens,), mval, dtype=torch.uint8, device=dev)
        for _ in range(5):
            layer.forward_masked(x, m)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            layer.forward_masked(x, m)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 50 * 1e3
        nsl = bin(mval).count("1")
        mb = args.out * args.inn * 2 * nsl / 8 / 1e6
        print(f"mask {mval:2d}: {us:7.2f} us/launch (eager, back to back)  {mb:5.1f} MB slices -> {mb / us * 1e-3:6.2f} TB/s")
        set_debug_impl(9)
        layer.forward_masked(x, m)
        torch.cuda.synchronize()
        set_debug_impl(0)
        full = np.zeros(32 * 1024, np.uint64)
        lib = _lib.lib()
        lib.mobi_debug_read_trace.argtypes = [C.c_void_p, C.c_int]
        _lib.check(lib.mobi_debug_read_trace(full.ctypes.data, 1))
        g = full.astype(np.int64).reshape(-1, 8)[2048:4096]
        g = g[g[:, 0] > 0]
        t0 = g[:, 0].min()
        names = ["start", "x prep", "slice1", "griddep", "union", "end"]
        print("   ", "  ".join(f"{n} {int(np.median(g[:, i] - t0))}" for i, n in enumerate(names)))


if __name__ == "__main__":
    main()
