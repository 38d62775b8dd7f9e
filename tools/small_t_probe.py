"""Development tool: forward() step time at 33..128 tokens with the 1-CTA split-K GEMM (debug impl 5)
vs the CTA-pair GEMM (debug impl 3), q/o 4096x4096, 3 bits (CUDA events over 50 calls)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2602_20191_b200 import calibrate_threshold  # noqa: E402


def main():
    args = bench.parse()
    bench.workload(args, 1)
    dev = torch.device("cuda", 0)
    layer, _ = bench.make_layer(args, dev, 1)
    args.tokens = 4096
    xcal = bench.make_x(args, dev, 5)
    delta = calibrate_threshold(layer.score(xcal), 1 / 6)
    for T in (33, 48, 64, 96, 128):
        x = xcal[:T].contiguous()
        res = {}
        for impl in (5, 3, 0):
            layer.set_debug_impl(impl)
            for _ in range(5):
                layer.forward(x, delta)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(50):
                layer.forward(x, delta)
            e1.record()
            torch.cuda.synchronize()
            res[impl] = e0.elapsed_time(e1) / 50 * 1e3
        layer.set_debug_impl(0)
        print(f"T={T:4d}: split-K 1-CTA {res[5]:6.1f} us, CTA-pair {res[3]:6.1f} us, production {res[0]:6.1f} us")


if __name__ == "__main__":
    main()
