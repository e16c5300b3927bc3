"""Developer probe: the explicit-plan (three-phase) scan vs the chained scan
at small shapes (C1), CUDA-event timed around the C calls."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
from paper_1709_04057_b200 import capi
T, W = int(sys.argv[1]), int(sys.argv[2])
lam = torch.rand(T, W, device="cuda") * 0.9 + 0.05
x = torch.rand(T, W, device="cuda") * 2 - 1
dh = torch.rand(T, W, device="cuda") * 2 - 1
h0 = torch.zeros(W, device="cuda")
h, dl, dx = (torch.empty_like(lam) for _ in range(3)); d0 = torch.empty_like(h0)
st = torch.cuda.current_stream().cuda_stream
p = lambda t: t.data_ptr()
def tm(fn, n=50):
    for _ in range(5): fn()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    ts.sort(); return ts[len(ts) // 2]
ws = capi.Workspace(0)
print("chained fwd %.1f bwd %.1f" % (
    tm(lambda: capi.scan(p(lam), p(x), p(h0), p(h), T, W, capi.PARALLEL, 4, ws.handle, st)),
    tm(lambda: capi.scan_backward(p(lam), p(h0), p(h), p(dh), p(dl), p(dx), p(d0), T, W, capi.PARALLEL, 4, ws.handle, st))))
for chunk in (16, 32, 64, 128, 256):
    pc = T // chunk
    plan = [(i * chunk + 1, (i + 1) * chunk) for i in range(pc)]
    print("plan chunk %d (p=%d) fwd %.1f bwd %.1f" % (chunk, pc,
        tm(lambda: capi.scan_plan(p(lam), p(x), p(h0), p(h), T, W, plan, stream=st)),
        tm(lambda: capi.scan_backward_plan(p(lam), p(h0), p(h), p(dh), p(dl), p(dx), p(d0), T, W, plan, stream=st))))
