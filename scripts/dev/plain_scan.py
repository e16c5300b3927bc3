"""Dev probe: plain single-GPU scan fwd+bwd at a given (T, W), a few reps (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1709_04057_b200 import capi
T, W = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
lam = torch.empty(T, W, device=dev).uniform_(0.05, 0.95, generator=g)
x = torch.empty(T, W, device=dev).uniform_(-1, 1, generator=g)
dh = torch.empty(T, W, device=dev).uniform_(-1, 1, generator=g)
h0 = torch.zeros(W, device=dev)
h, dl, dx, dh0 = torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(h0)
st = torch.cuda.current_stream().cuda_stream
for r in range(4):
    capi.scan(lam.data_ptr(), x.data_ptr(), h0.data_ptr(), h.data_ptr(), T, W, capi.PARALLEL, 4, None, st)
    capi.scan_backward(lam.data_ptr(), h0.data_ptr(), h.data_ptr(), dh.data_ptr(), dl.data_ptr(), dx.data_ptr(),
                       dh0.data_ptr(), T, W, capi.PARALLEL, 4, None, st)
torch.cuda.synchronize()
