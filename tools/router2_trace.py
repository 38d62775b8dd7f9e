"""Development tool: per-CTA timing of the CTA-pair prefill router (debug impl 7) at the bench shape."""
import ctypes as C, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, '/root/repo')
import bench
from paper_2602_20191_b200 import _lib
args = bench.parse()
bench.workload(args, 1)
dev = torch.device("cuda", 0)
layer, _ = bench.make_layer(args, dev, 1)
x = bench.make_x(args, dev, 2)
for _ in range(5): layer.score(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): layer.score(x)
e1.record(); torch.cuda.synchronize()
print("score() avg us", e0.elapsed_time(e1) / 20 * 1e3)
import os
if os.environ.get("MOBI_COLD"):  # evict X and w1 from L2 first (the bench ring's condition)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush.fill_(1)
    torch.cuda.synchronize()
    e0.record(); layer.score(x); e1.record(); torch.cuda.synchronize()
    print("cold score() us", e0.elapsed_time(e1) * 1e3)
    flush.fill_(2)
    torch.cuda.synchronize()
layer.set_debug_impl(7)
layer.score(x)
torch.cuda.synchronize()
layer.set_debug_impl(0)
full = np.zeros(32 * 1024, np.uint64)
lib = _lib.lib(); lib.mobi_debug_read_trace.argtypes = [C.c_void_p, C.c_int]
_lib.check(lib.mobi_debug_read_trace(full.ctypes.data, 1))
t = full.astype(np.int64)[4096:4096 + 8 * 148].reshape(148, 8)
t = t[t[:, 5] > 0]
g0 = t[:, 4].min()
print("CTAs", len(t), "start spread us", (t[:, 4].max() - g0) / 1e3, "end min/med/max us", (t[:, 5].min() - g0) / 1e3, np.median(t[:, 5] - g0) / 1e3, (t[:, 5].max() - g0) / 1e3)
print("cycles: prologue med", np.median(t[:, 1]), "acc_full med", np.median(t[:, 2]), "epi done med", np.median(t[:, 3]), "total med/max", np.median(t[:, 6]), t[:, 6].max())
print("clock GHz", np.median(t[:, 6] / (t[:, 5] - t[:, 4])))
kbt = full.astype(np.int64)[8192:8192 + 64]
print("CTA0 tile0 per-k-block full-ok cycles:", kbt[:24].tolist())
print("cadence (median diff)", np.median(np.diff(kbt[kbt > 0])))
