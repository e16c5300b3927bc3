"""Tiny scans through the device path (dev probe): python scripts/dev/tiny_scan.py T W [f32|f64]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from paper_1709_04057_b200 import torch_ops  # noqa: E402

T, W = int(sys.argv[1]), int(sys.argv[2])
dt = torch.float64 if (len(sys.argv) > 3 and sys.argv[3] == "f64") else torch.float32
g = torch.Generator().manual_seed(0)
lam = torch.empty(T, W, dtype=torch.float64).uniform_(0.05, 0.95, generator=g)
x = torch.empty(T, W, dtype=torch.float64).uniform_(-1, 1, generator=g)
dh = torch.empty(T, W, dtype=torch.float64).uniform_(-1, 1, generator=g)
h_ref = torch.empty_like(x)
c = torch.zeros(W, dtype=torch.float64)
for t in range(T):
    c = lam[t] * c + x[t]
    h_ref[t] = c
d = torch.device("cuda")
L, X, DH = (t.view(T, 1, W).to(d, dt) for t in (lam, x, dh))
h = torch_ops.scan(L, X, torch.zeros(1, W, dtype=dt, device=d))
torch.cuda.synchronize()
err = ((h.double().cpu().view(T, W) - h_ref).abs().max() / h_ref.abs().max()).item()
dl, dx, dh0 = torch_ops.scan_backward(L, torch.zeros(1, W, dtype=dt, device=d), h, DH)
torch.cuda.synchronize()
print(f"T={T} W={W} {dt}: fwd err {err:.2e}, bwd ok")
