"""The gated backward scan (linrec_scan_backward_gated_f32): scan_backward on
the adjoint d_h * gate, fused into the TMA backward's staging for the default
configuration and computed as dx = d_h * gate + an in-place scan elsewhere.
Both must equal the plain backward scan on the explicit product: bit-exact in
serial mode, within the reference's 1e-5 normwise in parallel mode (the fused
and unfused products are the same fp32 multiply)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _gated(lam, h0, h, dh, gate, mode):
    from paper_1709_04057_b200 import capi
    T, W = lam.shape
    dx, dl, dh0 = torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(h0)
    capi.check(capi.lib.linrec_scan_backward_gated_f32(lam.data_ptr(), h0.data_ptr(), h.data_ptr(), dh.data_ptr(),
                                                       gate.data_ptr(), dl.data_ptr(), dx.data_ptr(),
                                                       dh0.data_ptr(), T, W, mode, None,
                                                       torch.cuda.current_stream().cuda_stream))
    return dl, dx, dh0


# (T, W): fused TMA default config (C3's cell-scan width, long chains with
# virtual segments), short sequences (CTA-local: unfused), narrow W, serial
@pytest.mark.parametrize("T,W", [(65536, 2048), (20000, 128), (3000, 256), (777, 12), (50, 8192)])
@pytest.mark.parametrize("lo", [0.05, 0.99])
def test_gated_equals_plain_on_product(T, W, lo):
    from paper_1709_04057_b200 import capi
    g = torch.Generator(device="cuda").manual_seed(T + W)
    lam = torch.empty(T, W, device="cuda").uniform_(lo, 1.0 if lo > 0.5 else 0.95, generator=g)
    h = torch.empty(T, W, device="cuda").uniform_(-1, 1, generator=g)
    dh = torch.empty(T, W, device="cuda").uniform_(-1, 1, generator=g)
    gate = torch.empty(T, W, device="cuda").uniform_(0, 1, generator=g)
    h0 = torch.empty(W, device="cuda").uniform_(-1, 1, generator=g)
    prod = dh * gate
    for mode in (capi.SERIAL, capi.PARALLEL):
        dl, dx, dh0 = _gated(lam, h0, h, dh, gate, mode)
        rl, rx, r0 = torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(h0)
        capi.scan_backward(lam.data_ptr(), h0.data_ptr(), h.data_ptr(), prod.data_ptr(), rl.data_ptr(),
                           rx.data_ptr(), r0.data_ptr(), T, W, mode, 4, None,
                           torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        for a, r in ((dl, rl), (dx, rx), (dh0, r0)):
            if mode == capi.SERIAL:
                assert torch.equal(a, r)
            else:
                assert ((a - r).abs().max() / r.abs().max()).item() <= 1e-5
