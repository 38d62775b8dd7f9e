"""Development tool: forward() step time at small batches with the production kernel choice (debug impl 0),
the 1-CTA split-K GEMM (impl 5), the CTA-pair GEMM path (impl 3: router + gather + pair GEMM, never the
decode kernels) and the decode kernels (impl 10), 3 bits, CUDA events over 50 calls (not graph-replayed).
Shape from bench.py's --out/--in; MOBI_PROBE_T="16,24,32" picks the token counts, MOBI_PROBE_IMPLS the
variants."""
import os
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
    Ts = [int(t) for t in os.environ.get("MOBI_PROBE_T", "33,48,64,96,128").split(",")]
    IMPLS = [int(i) for i in os.environ.get("MOBI_PROBE_IMPLS", "5,3,0").split(",")]
    for T in Ts:
        x = xcal[:T].contiguous()
        res = {}
        for impl in IMPLS:
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
        layer.forward(x, delta)
        names = {5: "split-K 1-CTA", 3: "CTA-pair path", 10: "decode kernels", 0: "production"}
        print(f"{layer.out}x{layer.inn} T={T:4d}: " + ", ".join(f"{names.get(i, i)} {res[i]:6.1f} us" for i in IMPLS)
              + f" ({layer.last_plan()['gemm']})", flush=True)


if __name__ == "__main__":
    main()
