"""Diagnostic: how many chain positions per virtual segment carry a non-zero
entering product (the fix-up's work) at the C4 shape, forward and backward.
Usage: fixup_diag.py [T] [W]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1709_04057_b200 import capi  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
W = int(sys.argv[2]) if len(sys.argv) > 2 else 128
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
lam = torch.empty(T, W, device=dev).uniform_(0.05, 0.95, generator=g)
x = torch.empty(T, W, device=dev).uniform_(-1, 1, generator=g)
dh = torch.empty(T, W, device=dev).uniform_(-1, 1, generator=g)
h, dlam, dx = torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(lam)
dh0, hprev, ones = torch.empty(W, device=dev), torch.zeros(W, device=dev), torch.ones(W, device=dev)
agg = torch.empty(2, W, device=dev)
ws = capi.Workspace(0)
st = torch.cuda.current_stream().cuda_stream
p = lambda t: t.data_ptr()  # noqa: E731
for back in (False, True):
    n = capi.segment_prod_rows(T, W, back)
    rows = capi.segment_tile_rows(T, W, back)
    sp = torch.empty(n, W, device=dev)
    if back:
        capi.segment_scan_backward(p(lam), p(hprev), p(h), p(dh), p(ones), p(dlam), p(dx), p(dh0), p(sp), p(agg),
                                   T, W, 4, ws.handle, st)
    else:
        capi.segment_scan(p(lam), p(x), None, p(h), p(sp), p(agg), T, W, 4, ws.handle, st)
    torch.cuda.synchronize()
    # n = nseg*ntt + nseg ; ntt*rows ~ tseg
    cands = [k for k in range(1, n + 1) if n % k == 0 and n // k > 1
             and k * (n // k - 1) * rows >= T and (k - 1) * (n // k - 1) * rows < T]
    nseg = cands[-1]  # the finest split consistent with the row count
    ntt = n // nseg - 1
    pos = sp[: nseg * ntt].view(nseg, ntt, W)
    nzpos = (pos != 0).any(dim=2)  # [nseg][ntt]
    counts = nzpos.sum(dim=1)
    prefix = torch.stack([(~r).int().argmax() if (~r).any() else torch.tensor(ntt, device=dev) for r in nzpos])
    print(f"{'bwd' if back else 'fwd'}: nseg={nseg} ntt={ntt} rows={rows}  nz positions per segment: "
          f"min {int(counts.min())} mean {float(counts.float().mean()):.2f} max {int(counts.max())}; "
          f"nz prefix max {int(prefix.max())}")

# GPU time of the forward rank fix-up alone, from CUDA graphs (no host
# gaps): warm (replayed on the same data), and after a 256 MB write
# (difference of [write; fix-up] and [write])
n = capi.segment_prod_rows(T, W, False)
rows = capi.segment_tile_rows(T, W, False)
sp = torch.empty(n, W, device=dev)
capi.segment_scan(p(lam), p(x), None, p(h), p(sp), p(agg), T, W, 4, ws.handle, st)
c_in = torch.empty(W, device=dev).uniform_(-1, 1, generator=g)
big = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s2 = torch.cuda.Stream()
graphs = {}
with torch.cuda.stream(s2):
    sid = s2.cuda_stream
    for name, parts in (("fix", ("fix",)), ("fill+fix", ("fill", "fix")), ("fill", ("fill",)),
                        ("scan+fix", ("scan", "fix")), ("scan", ("scan",))):
        def body(parts=parts):
            for q in parts:
                if q == "fill":
                    big.fill_(1)
                elif q == "scan":
                    capi.segment_scan(p(lam), p(x), None, p(h), p(sp), p(agg), T, W, 4, ws.handle, sid)
                else:
                    capi.segment_fixup(p(lam), p(h), p(sp), p(c_in), T, W, rows, 4, sid)
        body()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s2):
            body()
        graphs[name] = gr
torch.cuda.synchronize()
res = {}
for name, gr in graphs.items():
    for _ in range(3):
        gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / 20 * 1000
print(f"rank fix-up: warm {res['fix']:.1f} us; after a 256 MB write {res['fill+fix'] - res['fill']:.1f} us; "
      f"after the segment scan {res['scan+fix'] - res['scan']:.1f} us (scan {res['scan']:.1f} us)")
