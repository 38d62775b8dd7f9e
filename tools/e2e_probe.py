"""Development tool: PCIe copy rates (pinned, alone and concurrent) and the end-to-end host-buffer
forward (mobi_forward_host) at the bench shape; the chunk count comes from MOBI_E2E_CHUNKS."""
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2602_20191_b200 import calibrate_threshold  # noqa: E402


def rate(fn, nbytes, reps=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t0) / 1e9


def main():
    args = bench.parse()
    bench.workload(args, 1)
    dev = torch.device("cuda", 0)
    T, inn, out = args.tokens, args.inn, args.out
    if os.environ.get("E2E_PCIE", "1") == "1":
        hx = torch.empty((T, inn), dtype=torch.bfloat16, pin_memory=True)
        hy = torch.empty((T, out), dtype=torch.bfloat16, pin_memory=True)
        dx = torch.empty((T, inn), dtype=torch.bfloat16, device=dev)
        dy = torch.empty((T, out), dtype=torch.bfloat16, device=dev)
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        h2d = rate(lambda: dx.copy_(hx, non_blocking=True), hx.numel() * 2)
        d2h = rate(lambda: hy.copy_(dy, non_blocking=True), hy.numel() * 2)

        def both():
            with torch.cuda.stream(s1):
                dx.copy_(hx, non_blocking=True)
            with torch.cuda.stream(s2):
                hy.copy_(dy, non_blocking=True)
        bi = rate(both, hx.numel() * 2 + hy.numel() * 2)
        print(f"PCIe pinned {hx.numel() * 2 / 2**20:.0f} MiB: H2D {h2d:.1f} GB/s, D2H {d2h:.1f} GB/s, "
              f"both directions {bi:.1f} GB/s total")
    layer, _ = bench.make_layer(args, dev, 1)
    x = bench.make_x(args, dev, 2)
    delta = calibrate_threshold(layer.score(x), (args.target_bits - 2) / 6)
    xh = x.cpu().pin_memory()
    yh = torch.empty((T, out), dtype=torch.bfloat16, pin_memory=True)
    for _ in range(3):
        layer.forward_host(xh, delta, y_host=yh)
    reps = 30
    t0 = time.perf_counter()
    for _ in range(reps):
        layer.forward_host(xh, delta, y_host=yh)
    dt = (time.perf_counter() - t0) / reps
    print(f"e2e chunks={os.environ.get('MOBI_E2E_CHUNKS', 'default')}: {dt * 1e3:.3f} ms/step, "
          f"{T / dt / 1e6:.2f} M tokens/s")


if __name__ == "__main__":
    main()
