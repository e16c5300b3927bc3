"""Developer probe for compute-sanitizer: small chained scans fwd + bwd
(run with LINREC_CHAINS=1 for deep single-chain look-backs)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
from paper_1709_04057_b200 import capi, torch_ops as ops
for T, W in ((6144, 128), (3000, 32), (200000, 16)):
    lam = torch.rand(T, 1, W, device="cuda") * 0.5 + 0.5
    x = torch.rand_like(lam) - 0.5
    dh = torch.rand_like(lam) - 0.5
    h0 = torch.rand(1, W, device="cuda")
    h = ops.scan(lam, x, h0); hs = ops.scan(lam, x, h0, mode="serial")
    g = ops.scan_backward(lam, h0, hs, dh)
    torch.cuda.synchronize()
    print(T, W, ((h - hs).abs().max() / hs.abs().max()).item())
