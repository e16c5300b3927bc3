"""Developer probe for compute-sanitizer: the cluster scans (fp32, forward and
backward, 8- and 16-CTA clusters, full and ragged columns, the segment
backward's carry-in) and the fp64 layers (GILR-LSTM and QRNN forward +
backward, split-K weight gradients)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch  # noqa: E402

from paper_1709_04057_b200 import capi, layers as L, torch_ops as ops  # noqa: E402

for T, W in ((4096, 256), (1000, 36), (600, 4), (2049, 64)):
    print(T, W, capi.scan_kernel_name(T, W), flush=True)
    lam = torch.rand(T, 1, W, device="cuda") * 0.9 + 0.05
    x = torch.rand_like(lam) - 0.5
    dh = torch.rand_like(lam) - 0.5
    h0 = torch.rand(1, W, device="cuda")
    h = ops.scan(lam, x, h0)
    hs = ops.scan(lam, x, h0, mode="serial")
    g = ops.scan_backward(lam, h0, hs, dh)
    gs = ops.scan_backward(lam, h0, hs, dh, mode="serial")
    torch.cuda.synchronize()
    print("  err", ((h - hs).abs().max() / hs.abs().max()).item(),
          max(((a - b).abs().max() / b.abs().max()).item() for a, b in zip(g, gs)), flush=True)
    Lr, DH, H = lam.view(T, W), dh.view(T, W), hs.view(T, W)
    ln, gn = torch.rand(W, device="cuda"), torch.rand(W, device="cuda")
    DL, DX, D0 = torch.empty_like(Lr), torch.empty_like(Lr), torch.empty(W, device="cuda")
    capi.scan_backward_segment(Lr.data_ptr(), None, H.data_ptr(), DH.data_ptr(), ln.data_ptr(), gn.data_ptr(),
                               DL.data_ptr(), DX.data_ptr(), D0.data_ptr(), T, W)
    torch.cuda.synchronize()
gen = torch.Generator().manual_seed(0)
T, b, m, n = 70, 3, 12, 10
p = L.gilr_lstm_init(gen, m, n, dtype=torch.float64)
x = torch.rand(T, b, m, device="cuda", dtype=torch.float64) - 0.5
cache = L.GilrLstmCache()
h = L.gilr_lstm_forward(p, x, cache=cache)
grads = L.GilrLstmGrads.zeros_like(p)
L.gilr_lstm_backward(p, x, None, None, cache, torch.rand_like(h), grads)
q = L.qrnn_init(gen, m, n, 3, dtype=torch.float64)
qc = L.QrnnCache()
hq = L.qrnn_forward(q, x, cache=qc)
L.qrnn_backward(q, x, None, qc, torch.rand_like(hq), L.QrnnGrads.zeros_like(q))
torch.cuda.synchronize()
print("fp64 layers ok", flush=True)
