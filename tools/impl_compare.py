"""Development tool: forward time of the prefill GEMM variants (debug impls 0 / 3 = pair / 5 = 1-CTA) at small T."""
import sys, torch
sys.path.insert(0, '/root/repo')
import bench
from paper_2602_20191_b200 import calibrate_threshold, set_debug_impl
for T in (40, 64, 96):
    sys.argv = ['x', '--tokens', str(T)]
    args = bench.parse()
    dev = torch.device('cuda', 0)
    layer, _ = bench.make_layer(args, dev, 1)
    x = bench.make_x(args, dev, 2)
    d = calibrate_threshold(layer.score(x), 1 / 6)
    for impl in (0, 3, 5):
        set_debug_impl(impl)
        for _ in range(5): layer.forward(x, d)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): layer.forward(x, d)
        e1.record(); torch.cuda.synchronize()
        print(T, impl, round(e0.elapsed_time(e1) / 50 * 1e3, 1), 'us')
    set_debug_impl(0)
