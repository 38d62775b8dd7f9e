python - <<'PY'
import torch, numpy as np, sys
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
from gpu_helpers import make_layer, make_x, assert_y_close, gates_from_masks
from oracle import oracle as O
from paper_2602_20191_b200 import set_debug_impl, calibrate_threshold
orc = O.restatement()
for (out, inn, T) in [(256, 384, 300), (512, 512, 1000), (1024, 1024, 2048)]:
    L, layer = make_layer(out, inn, seed=out)
    xb, x64 = make_x(T, inn, seed=T)
    d = calibrate_threshold(layer.score(xb), 1/6)
    y0, m = layer.forward(xb, d, return_masks=True)
    set_debug_impl(3)
    y3 = layer.forward(xb, d)
    set_debug_impl(0)
    torch.cuda.synchronize()
    g = gates_from_masks(m.cpu().numpy(), 3)
    y_ref = orc.forward_elastic(x64, L["codes"], L["slice_bits"], L["scale"], L["zero"], 128, g)
    print(out, inn, T, "tc vs tc2 bit-equal:", torch.equal(y0, y3), "tc2 vs oracle:", assert_y_close(y3, y_ref, "tc2"))
PY
