"""Development tool: time the GEMM kernel alone (forward_masked, per-kernel CUDA events) for
controlled bucket distributions, to separate full-tile efficiency from small-bucket cost."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def run(layer, x, masks, reps=20):
    for _ in range(3):
        layer.forward_masked(x, masks)
    layer.profile(True)
    for _ in range(reps):
        layer.forward_masked(x, masks)
    prof = layer.profile_read()
    layer.profile(False)
    return prof["gemm"][0] / prof["gemm"][1], prof["gather"][0] / prof["gather"][1], prof["bucket"][0] / prof["bucket"][1]


def main():
    args = bench.parse()
    bench.workload(args, 1)
    import os
    dev = torch.device("cuda", 0)
    layer, _ = bench.make_layer(args, dev, 1)
    layer.set_debug_impl(int(os.environ.get("MOBI_IMPL", "0")))
    quick = os.environ.get('GB_QUICK')
    for T in ((2048, 8192) if quick else (256, 2048, 8192)):
        args.tokens = T
        x = bench.make_x(args, dev, 2)
        flops = 2.0 * T * args.inn * args.out
        rng = np.random.default_rng(0)
        dists = {
            "all mask 15 (one bucket)": np.full(T, 15),
            "all mask 1": np.full(T, 1),
            "8 equal buckets": (np.arange(T) % 8) * 2 + 1,
            "realistic 3-bit mix": rng.choice([1, 3, 5, 7, 9, 11, 13, 15], T,
                                              p=np.array([1181, 234, 151, 36, 334, 72, 31, 9]) / 2048),
        }
        for name, m in dists.items():
            if quick and name not in ('all mask 1', 'realistic 3-bit mix'):
                continue
            masks = torch.from_numpy(m.astype(np.uint8)).to(dev)
            g, ga, bk = run(layer, x, masks)
            print(f"T={T:5d} {name:28s} gemm {g * 1e3:8.1f} us  {flops / (g * 1e-3) / 1e12:7.1f} TFLOP/s   "
                  f"gather {ga * 1e3:6.1f} us  bucket {bk * 1e3:6.1f} us")


if __name__ == "__main__":
    main()
