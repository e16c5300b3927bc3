"""Developer probe for compute-sanitizer (round 2): the CTA-local scans
(T <= 4096, vector and scalar paths, fp32/fp64), the split scans with their
fix-ups at slow decays (deep walks, one-round backward fix-up), and a
channel-sharded host scan over 2 column blocks."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np
import torch
from paper_1709_04057_b200 import sharded, torch_ops as ops

for T, W, dt in ((4096, 256, torch.float32), (300, 6, torch.float32), (1000, 64, torch.float64),
                 (20000, 16, torch.float32)):
    for lo in (0.05, 0.99):
        lam = (torch.rand(T, 1, W, device="cuda", dtype=dt) * (1 - lo) + lo)
        x = torch.rand_like(lam) - 0.5
        dh = torch.rand_like(lam) - 0.5
        h0 = torch.rand(1, W, device="cuda", dtype=dt)
        h = ops.scan(lam, x, h0)
        hs = ops.scan(lam, x, h0, mode="serial")
        g = ops.scan_backward(lam, h0, hs, dh)
        gs = ops.scan_backward(lam, h0, hs, dh, mode="serial")
        torch.cuda.synchronize()
        print(T, W, dt, lo, ((h - hs).abs().max() / hs.abs().max()).item(),
              max(((a - b).abs().max() / b.abs().max()).item() for a, b in zip(g, gs)), flush=True)
lam = np.random.rand(500, 2, 40).astype(np.float32) * 0.9
x = np.random.rand(500, 2, 40).astype(np.float32) - 0.5
h = sharded.channel_sharded_scan(lam, x, None, devices=[0, 0])
print("channel-sharded ok", h.shape)
# decay-adaptive stitch: deep (lam ~ U(0.99, 1)) and shallow decays on split scans
for lo in (0.05, 0.995):
    T, W = 300000, 128
    lam = torch.rand(T, 1, W, device="cuda") * (1 - lo) + lo
    x = torch.rand_like(lam) - 0.5
    dh = torch.rand_like(lam) - 0.5
    h0 = torch.rand(1, W, device="cuda")
    h = ops.scan(lam, x, h0)
    hs = ops.scan(lam, x, h0, mode="serial")
    g = ops.scan_backward(lam, h0, hs, dh)
    gs = ops.scan_backward(lam, h0, hs, dh, mode="serial")
    torch.cuda.synchronize()
    print("adaptive", lo, ((h - hs).abs().max() / hs.abs().max()).item(),
          max(((a - b).abs().max() / b.abs().max()).item() for a, b in zip(g, gs)), flush=True)
