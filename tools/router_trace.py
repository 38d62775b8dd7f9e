"""Development tool: timeline of the tcgen05 router kernel on CTA 0 (debug impl 7)."""
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
    for _ in range(3):
        layer.score(x)
    set_debug_impl(7)
    layer.score(x)
    torch.cuda.synchronize()
    set_debug_impl(0)
    full = np.zeros(32 * 1024, np.uint64)
    lib = _lib.lib()
    lib.mobi_debug_read_trace.argtypes = [C.c_void_p, C.c_int]
    _lib.check(lib.mobi_debug_read_trace(full.ctypes.data, 1))
    t = full.astype(np.int64)
    print("kb  tma:empty-ok  mma:full-ok")
    for kb in range(64):
        print(f"{kb:3d} {t[128 + kb]:10d} {t[kb]:10d}")
    g = t[4096:4096 + 4 * 148].reshape(-1, 4)
    g = g[g[:, 1] > 0]
    t0 = g[:, 0].min()
    print(f"CTAs {len(g)}: start spread {(g[:, 0].max() - t0) / 1e3:.2f} us, end min/med/max "
          f"{(g[:, 1].min() - t0) / 1e3:.2f}/{(np.median(g[:, 1]) - t0) / 1e3:.2f}/{(g[:, 1].max() - t0) / 1e3:.2f} us, "
          f"cycles min/max {g[:, 3].min()}/{g[:, 3].max()}, clock {np.median(g[:, 3] / ((g[:, 1] - g[:, 0]) + 1)):.3f} GHz")
    print("cluster: rank0 recv_full", t[212], " rank1 acc_full", t[1024 + 200], "staged", t[1024 + 210],
          "peer_go", t[1024 + 211], "rank1 mma end", t[1024 + 203], "tma end", t[1024 + 204])
    print("epi acc_full", t[200], "epi drained", t[201], "end epi/mma/tma", t[202], t[203], t[204], "exit", t[205])


if __name__ == "__main__":
    main()
