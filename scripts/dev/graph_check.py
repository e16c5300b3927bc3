"""Dev probe: eager vs CUDA-graph-replayed scan (fwd + bwd) on one shape."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1709_04057_b200 import capi
T, W = int(sys.argv[1]), int(sys.argv[2])
lo = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
st = s.cuda_stream
ws = capi.Workspace(0)
g = torch.Generator(device=dev).manual_seed(0)
with torch.cuda.stream(s):
    lam = torch.empty(T, W, device=dev).uniform_(lo, 0.95 if lo < 0.9 else 1.0, generator=g)
    x = torch.empty(T, W, device=dev).uniform_(-1, 1, generator=g)
    h0 = torch.zeros(W, device=dev)
    dh = torch.empty(T, W, device=dev).uniform_(-1, 1, generator=g)
    h, dl, dx, dh0 = (torch.empty_like(lam) for _ in range(3)) + (torch.empty_like(h0),) if False else (torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(h0))
def fwd():
    capi.scan(lam.data_ptr(), x.data_ptr(), h0.data_ptr(), h.data_ptr(), T, W, capi.PARALLEL, 4, ws.handle, st)
def bwd():
    capi.scan_backward(lam.data_ptr(), h0.data_ptr(), h.data_ptr(), dh.data_ptr(), dl.data_ptr(), dx.data_ptr(), dh0.data_ptr(), T, W, capi.PARALLEL, 4, ws.handle, st)
fwd(); bwd(); s.synchronize()
ref = [t.clone() for t in (h, dl, dx, dh0)]
gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
with torch.cuda.graph(gf, stream=s):
    fwd()
with torch.cuda.graph(gb, stream=s):
    bwd()
for t in (h, dl, dx, dh0):
    t.zero_()
torch.cuda.synchronize()
for _ in range(3):
    gf.replay(); gb.replay()
torch.cuda.synchronize()
errs = [((a - b).abs().max() / b.abs().max()).item() for a, b in zip((h, dl, dx, dh0), ref)]
print(f"T={T} W={W} lam>={lo}: graph vs eager max rel diff h {errs[0]:.2e} dlam {errs[1]:.2e} dx {errs[2]:.2e} dh0 {errs[3]:.2e}")
