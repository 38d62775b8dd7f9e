"""Development tool: device timeline of a chunked host-buffer forward, rebuilt with torch streams
(H2D chunks on one stream, the layer on another, D2H on a third; timed events on each) to see where
mobi_forward_host's pipeline serialises.  Prints per-chunk start/end (us) of each phase."""
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
    T, inn, out = args.tokens, args.inn, args.out
    layer, _ = bench.make_layer(args, dev, 1)
    x = bench.make_x(args, dev, 2)
    delta = calibrate_threshold(layer.score(x), (args.target_bits - 2) / 6)
    xh = x.cpu().pin_memory()
    yh = torch.empty((T, out), dtype=torch.bfloat16, pin_memory=True)
    dx = torch.empty_like(x)
    dy = torch.empty((T, out), dtype=torch.bfloat16, device=dev)
    sh, sc, sd = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    for nch in (1, 2, 4, 8):
        n = T // nch
        for rep in range(3):
            ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
            t0 = ev()
            marks = []
            torch.cuda.synchronize()
            t0.record(sh)
            for c in range(nch):
                a, b, e0, e1, f0, f1 = ev(), ev(), ev(), ev(), ev(), ev()
                with torch.cuda.stream(sh):
                    a.record(sh)
                    dx[c * n:(c + 1) * n].copy_(xh[c * n:(c + 1) * n], non_blocking=True)
                    b.record(sh)
                sc.wait_event(b)
                with torch.cuda.stream(sc):
                    e0.record(sc)
                    layer.forward(dx[c * n:(c + 1) * n], delta, y=dy[c * n:(c + 1) * n], stream=sc)
                    e1.record(sc)
                sd.wait_event(e1)
                with torch.cuda.stream(sd):
                    f0.record(sd)
                    yh[c * n:(c + 1) * n].copy_(dy[c * n:(c + 1) * n], non_blocking=True)
                    f1.record(sd)
                marks.append((a, b, e0, e1, f0, f1))
            torch.cuda.synchronize()
            if rep < 2:
                continue
            rows = [[round(t0.elapsed_time(m) * 1e3) for m in mk] for mk in marks]
            total = rows[-1][5]
            print(f"chunks {nch}: total {total} us; per chunk (h2d start,end | compute start,end | d2h start,end):")
            for r in rows:
                print("   ", r)
    # copies alone vs concurrently, 4.2 MB pieces
    n = T // 4
    for label, both in (("h2d alone", False), ("h2d+d2h concurrent", True)):
        torch.cuda.synchronize()
        a, b, c_, d = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        a.record(sh)
        with torch.cuda.stream(sh):
            for c in range(4):
                dx[c * n:(c + 1) * n].copy_(xh[c * n:(c + 1) * n], non_blocking=True)
        b.record(sh)
        if both:
            c_.record(sd)
            with torch.cuda.stream(sd):
                for c in range(4):
                    yh[c * n:(c + 1) * n].copy_(dy[c * n:(c + 1) * n], non_blocking=True)
            d.record(sd)
        torch.cuda.synchronize()
        print(label, f"h2d {a.elapsed_time(b) * 1e3:.0f} us", f"d2h {c_.elapsed_time(d) * 1e3:.0f} us" if both else "")


if __name__ == "__main__":
    main()
