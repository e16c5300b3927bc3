"""Dev probe: C4 scan fwd + bwd with slow decays lam ~ U(0.99, 1) (the fix-up's worst case), a few reps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1709_04057_b200 import capi
T, W = 1 << 20, 128
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
lam = torch.empty(T, W, device=dev).uniform_(0.99, 1.0, generator=g)
x = torch.empty(T, W, device=dev).uniform_(-1, 1, generator=g)
dh = torch.empty(T, W, device=dev).uniform_(-1, 1, generator=g)
h0 = torch.zeros(W, device=dev)
h, dl, dx, dh0 = torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(h0)
st = torch.cuda.current_stream().cuda_stream
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for r in range(reps):
    ev[0].record()
    capi.scan(lam.data_ptr(), x.data_ptr(), h0.data_ptr(), h.data_ptr(), T, W, capi.PARALLEL, 4, None, st)
    ev[1].record()
    capi.scan_backward(lam.data_ptr(), h0.data_ptr(), h.data_ptr(), dh.data_ptr(), dl.data_ptr(), dx.data_ptr(),
                       dh0.data_ptr(), T, W, capi.PARALLEL, 4, None, st)
    ev[2].record()
    torch.cuda.synchronize()
    print(f"fwd {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us  bwd {ev[1].elapsed_time(ev[2]) * 1e3:.1f} us", flush=True)
