"""Development tool: the cost_model sanity law (bitplane.hpp:203-251; tests/test_bitplane.cpp:283-330)
measured with ncu: the decode GEMV's DRAM bytes must grow with the union of active slices
(out*in*2/8 bytes per slice) plus constants.

  ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:decode_planes --csv \
      --log-file gpurun_out/cost_law.csv python tools/cost_law.py [out in]

For each union size |U| = 1..4 it runs forward_masked at T=1 with the token's mask = slices 1..|U|
(REPS launches per size, in order), after a 256 MiB L2 flush so every launch reads from HBM.
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from gpu_helpers import make_layer, make_x  # noqa: E402

REPS = 3


def main():
    out = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    inn = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    _, layer = make_layer(out, inn, gs=128, hidden=inn // 4, seed=5)
    xb, _ = make_x(1, inn, seed=9)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for u in range(1, 5):
        mask = torch.tensor([(1 << u) - 1], dtype=torch.uint8, device="cuda")  # slices 1..u
        for _ in range(REPS):
            flush.fill_(u)
            layer.forward_masked(xb, mask)
    torch.cuda.synchronize()
    print("plan", layer.last_plan())


if __name__ == "__main__":
    main()
