import sys, torch, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from gpu_helpers import make_layer, make_x
L, layer = make_layer(256, 512, gs=128, hidden=128, seed=3)
xb, _ = make_x(64, 512)
try:
    s = layer.score(xb); torch.cuda.synchronize(); print("score ok", s.shape)
except Exception as e:
    print("ERR", e)
