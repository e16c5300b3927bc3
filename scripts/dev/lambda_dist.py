"""Scan time vs. the λ distribution (the fix-up walk is decay-bounded, so its
length depends on the data).  Times fwd and bwd of the chained scan at the C2
and C4 shapes for the bench distribution, the reference's stress sets
(verify.hpp:59-67: λ~U(-1,1), λ≡1, λ~U(0.99,1)) and λ≡0, and checks each
forward against the serial kernel.  Usage: python scripts/dev/lambda_dist.py
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch  # noqa: E402

from paper_1709_04057_b200 import capi  # noqa: E402

DISTS = {
    "U(0.05,0.95)": lambda t: t.uniform_(0.05, 0.95),
    "U(-1,1)": lambda t: t.uniform_(-1.0, 1.0),
    "U(0.99,1)": lambda t: t.uniform_(0.99, 1.0),
    "ones": lambda t: t.fill_(1.0),
    "zeros": lambda t: t.zero_(),
}


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1000.0


def main():
    ws = capi.Workspace(0)
    st = torch.cuda.current_stream().cuda_stream
    for name, T, W in (("c4", 1 << 20, 128), ("c2", 65536, 8192)):
        lam = torch.empty(T, W, device="cuda")
        x = torch.empty_like(lam).uniform_(-1, 1)
        dh = torch.empty_like(lam).uniform_(-1, 1)
        h0 = torch.empty(W, device="cuda").uniform_(-1, 1)
        h, hs, dl, dx = (torch.empty_like(lam) for _ in range(4))
        dh0 = torch.empty_like(h0)
        for dn, fill in DISTS.items():
            fill(lam)
            if dn == "ones":  # integer prefix sums stay exact in fp32
                x.copy_(torch.randint(-4, 5, x.shape, device="cuda").float())
            else:
                x.uniform_(-1, 1)
            fwd = lambda: capi.scan(lam.data_ptr(), x.data_ptr(), h0.data_ptr(), h.data_ptr(), T, W,  # noqa: E731
                                    capi.PARALLEL, 4, ws.handle, st)
            bwd = lambda: capi.scan_backward(lam.data_ptr(), h0.data_ptr(), h.data_ptr(), dh.data_ptr(),  # noqa: E731
                                             dl.data_ptr(), dx.data_ptr(), dh0.data_ptr(), T, W,
                                             capi.PARALLEL, 4, ws.handle, st)
            tf, tb = timed(fwd), timed(bwd)
            capi.scan(lam.data_ptr(), x.data_ptr(), h0.data_ptr(), hs.data_ptr(), T, W, capi.SERIAL, 4, None, st)
            fwd()
            err = ((h - hs).abs().max() / hs.abs().max().clamp_min(1.0)).item()
            el = T * W / ((tf + tb) * 1e-6)
            print(f"{name} {dn:13s} fwd {tf:8.1f} us  bwd {tb:8.1f} us  {el:.3e} el/s  err {err:.1e}", flush=True)
        del lam, x, dh, h, hs, dl, dx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
