"""Developer probe: forward / backward scan time (CUDA events, graph-free,
median of reps) at one shape; run under several LINREC_CHAINS values.
Usage: split_sweep.py T W"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch  # noqa: E402

from paper_1709_04057_b200 import capi  # noqa: E402

T, W = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda").manual_seed(0)
lam = torch.empty(T, W, device="cuda").uniform_(0.05, 0.95, generator=g)
x = torch.empty(T, W, device="cuda").uniform_(-1, 1, generator=g)
dh = torch.empty(T, W, device="cuda").uniform_(-1, 1, generator=g)
h0 = torch.zeros(W, device="cuda")
h, dl, dx = (torch.empty_like(lam) for _ in range(3))
d0 = torch.empty_like(h0)
ws = capi.Workspace(0)
st = torch.cuda.current_stream().cuda_stream
p = lambda t: t.data_ptr()  # noqa: E731
f = lambda: capi.scan(p(lam), p(x), p(h0), p(h), T, W, capi.PARALLEL, 4, ws.handle, st)  # noqa: E731
b = lambda: capi.scan_backward(p(lam), p(h0), p(h), p(dh), p(dl), p(dx), p(d0), T, W, capi.PARALLEL, 4,  # noqa
                               ws.handle, st)
res = []
for fn in (f, b):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    res.append(ts[len(ts) // 2])
print(f"T={T} W={W} chains={os.environ.get('LINREC_CHAINS', 'default')} fwd {res[0]:.1f} us bwd {res[1]:.1f} us "
      f"launches fwd {capi.scan_kernel_count(T, W, False)} bwd {capi.scan_kernel_count(T, W, True)}")
