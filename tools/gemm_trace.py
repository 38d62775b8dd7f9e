"""Development tool: run the traced tcgen05 GEMM (debug impl 2) on the bench workload and print
where each warp role spends its cycles (barrier waits vs. work)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2602_20191_b200 import _lib, calibrate_threshold  # noqa: E402


def main():
    a = bench.parse.__wrapped__() if hasattr(bench.parse, "__wrapped__") else None
    sys.argv = [sys.argv[0]] + sys.argv[1:]
    args = bench.parse()
    bench.workload(args, 1)
    dev = torch.device("cuda", 0)
    layer, _ = bench.make_layer(args, dev, 1)
    x = bench.make_x(args, dev, 2)
    delta = calibrate_threshold(layer.score(x), (args.target_bits - 2) / 6)
    for _ in range(3):
        layer.forward(x, delta)
    import os
    impl = int(os.environ.get("MOBI_TRACE_IMPL", "2"))
    layer.set_debug_impl(impl)
    if os.environ.get("MOBI_TRACE_MASK1"):  # one bucket (every token slice 1 only): forward_masked
        layer.forward_masked(x, torch.ones(x.shape[0], dtype=torch.uint8, device=dev))
    else:
        layer.forward(x, delta)
    torch.cuda.synchronize()
    layer.set_debug_impl(0)
    n = torch.cuda.get_device_properties(0).multi_processor_count
    full = np.zeros(32 * 1024, np.uint64)
    buf = full[: 16 * 1024].reshape(1024, 16)[:n]
    lib = _lib.lib()
    lib.mobi_debug_read_trace.argtypes = [C.c_void_p, C.c_int]
    _lib.check(lib.mobi_debug_read_trace(full.ctypes.data, n))
    names = ["tma wait empty", "mma wait acc_empty", "mma wait full_b", "mma wait full_a", "mma loop total",
             "dq wait empty", "dq loop total", "epi wait acc_full", "epi loop total", "tiles", "dq compute next",
             "dq wait::st", "dq st16 issue", "dq fetch issue", "dq next_tile"]
    for i, nm in enumerate(names):
        col = buf[:, i].astype(np.float64)
        print(f"{nm:22s} mean {col.mean():12.0f}  min {col.min():12.0f}  max {col.max():12.0f}")
    timeline(full)
    if impl == 4:
        ev = full[20480 + 512:20480 + 512 + 4 * 64].reshape(4, 64).astype(np.int64)
        e0 = full[20480:20480 + 64].astype(np.int64)
        t0 = e0[e0 > 0].min()
        print("leader MMA thread: elected / desc done / 4 MMAs issued / committed")
        for kb in range(24):
            print(f"{kb:2d} " + " ".join(f"{(ev[e][kb] - t0) if ev[e][kb] else -1:10d}" for e in range(4)))
    units(full)
    ch = full[28672:28672 + 64].astype(np.int64)
    if ch[0]:
        print("epilogue warp 0 drain (cycles from first chunk): before wait / after wait")
        print(" ".join(f"{int(ch[2*i]-ch[0])}/{int(ch[2*i+1]-ch[0])}" for i in range(8) if ch[2*i]))
    per = full[16 * 1024:20480].reshape(-1, 2)
    per = per[per[:, 0] > 0]
    for N in sorted(set(per[:, 0].tolist())):
        c = per[per[:, 0] == N][:, 1].astype(np.float64)
        print(f"tile N={N:4d}: {len(c):4d} tiles  cycles mean {c.mean():9.0f} min {c.min():9.0f} max {c.max():9.0f}"
              f"   ideal MMA {64 * 4 * 137.5 * N / 256:9.0f}")


def units(full):
    ev = full[24576:24576 + 2 * 8 * 16].reshape(2, 8, 16).astype(np.int64)
    t0 = ev[ev > 0].min() if (ev > 0).any() else 0
    names = ["mma:acc_empty ok", "mma:last kb", "epi:acc_full", "epi:released", "epi:scatter done", "epi:drain start"]
    print("unit events (ns from first): leader / peer")
    print("u   " + " ".join(f"{n:>17s}" for n in names))
    print("unit N:", full[24576 + 6 * 16:24576 + 7 * 16].tolist())
    for u in range(16):
        for r in range(2):
            print(f"{u:2d}{'LP'[r]} " + " ".join(f"{(ev[r][e][u] - t0) if ev[r][e][u] else -1:17d}" for e in range(6)))


def timeline(full, base=20480):
    timeline1(full, base)
    print("peer CTA (clock of the peer SM, offset unknown):")
    timeline1(full, base + 8 * 64)


def timeline1(full, base):
    ev = full[base:base + 8 * 64].reshape(8, 64).astype(np.int64)
    t0 = ev[0][ev[0] > 0].min() if (ev[0] > 0).any() else 0
    names = ["tma:empty ok", "mma:full_b ok", "dq3:arrive", "mma:issued", "dq:empty ok", "dq:arrive-ready", "cw:c_empty ok",
             "mma:full_a ok"]
    print("kb  " + " ".join(f"{n:>14s}" for n in names))
    for kb in range(0, 24):
        print(f"{kb:2d}  " + " ".join(f"{(ev[e][kb] - t0) if ev[e][kb] else -1:14d}" for e in range(8)))


if __name__ == "__main__":
    main()
