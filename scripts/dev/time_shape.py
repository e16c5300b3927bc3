"""Time one fwd+bwd scan step at (T, W) for decays U(lo, hi): the step as one
CUDA graph, replayed; prints us per step and el/s.  Usage: time_shape.py T W lo hi"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1709_04057_b200 import capi  # noqa: E402

T, W, lo, hi = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), float(sys.argv[4])
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
lam = torch.empty(T, W, device=dev).uniform_(lo, hi, generator=g)
x = torch.empty(T, W, device=dev).uniform_(-1, 1, generator=g)
dh = torch.empty(T, W, device=dev).uniform_(-1, 1, generator=g)
h0 = torch.zeros(W, device=dev)
h, dl, dx, d0 = torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(h0)
s = torch.cuda.Stream()
ws = capi.Workspace(0)
p = lambda t: t.data_ptr()  # noqa: E731


def step():
    capi.scan(p(lam), p(x), p(h0), p(h), T, W, capi.PARALLEL, 4, ws.handle, s.cuda_stream)
    capi.scan_backward(p(lam), p(h0), p(h), p(dh), p(dl), p(dx), p(d0), T, W, capi.PARALLEL, 4, ws.handle,
                       s.cuda_stream)


with torch.cuda.stream(s):
    step()
    s.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        step()
    for _ in range(3):
        gr.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    a.record(s)
    for _ in range(n):
        gr.replay()
    b.record(s)
    b.synchronize()
us = a.elapsed_time(b) / n * 1e3
print(f"T={T} W={W} lam~U({lo},{hi}): {us:.1f} us per fwd+bwd step, {T * W / (us * 1e-6):.3e} el/s "
      f"[{capi.scan_kernel_count(T, W)} + {capi.scan_kernel_count(T, W, True)} kernels]", flush=True)
