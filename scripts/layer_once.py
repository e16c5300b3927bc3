"""One GILR-LSTM layer forward (+ optional backward) at the C3 shape, for ncu
captures: python scripts/layer_once.py [tf32|fp32] [fwd|both] [T]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1709_04057_b200 import layers as L

prec = sys.argv[1] if len(sys.argv) > 1 else "tf32"
what = sys.argv[2] if len(sys.argv) > 2 else "fwd"
T = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
b, m, n = 4, 512, 512
gen = torch.Generator().manual_seed(7)
p = L.gilr_lstm_init(gen, m, n, 1.0, "cuda")
x = torch.rand(T, b, m, device="cuda") * 2 - 1
dh = torch.rand(T, b, n, device="cuda") * 2 - 1
z = torch.zeros(b, n, device="cuda")
cache = L.GilrLstmCache()
grads = L.GilrLstmGrads.zeros_like(p)
for _ in range(2):
    L.gilr_lstm_forward(p, x, z, z, precision=prec, cache=cache)
    if what == "both":
        L.gilr_lstm_backward(p, x, z, z, cache, dh, grads, precision=prec)
torch.cuda.synchronize()
print("done")
