"""Development tool: one CTA-pair GEMM unit per pair (q/o 4096x4096, T=256, one bucket) -- the
epilogue (TMEM drain + un-permute scatter) of the only unit is fully exposed; for ncu source views."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    tok = int(sys.argv.pop(1)) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 256
    args = bench.parse()
    bench.workload(args, 1)
    dev = torch.device("cuda", 0)
    layer, _ = bench.make_layer(args, dev, 1)
    args.tokens = tok
    x = bench.make_x(args, dev, 2)
    m = torch.ones(args.tokens, dtype=torch.uint8, device=dev)
    for _ in range(6):
        layer.forward_masked(x, m)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
