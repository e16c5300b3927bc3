"""The decay-adaptive stitch's unsplit twin (capi.cpp::unsplit_plan): on wide
split scans (>= 8 channel columns) the deep branch is one unsplit chained
scan per column instead of a reduce pass + seeded scan.  Both branches
against the oracle at the reference's 1e-5 normwise fp32 tolerance, forward
and backward, for decays that never underflow (deep: the twin runs) and the
bench decays (shallow: the split scan + fix-up run), plus the gated backward
(the layers' cell-scan adjoint) through the twin."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _p(t):
    return t.data_ptr()


# (T, W): 8 columns (the threshold), 16 (C3's cell scans), 64 (C2's width)
@pytest.mark.parametrize("T,W", [(16384, 1024), (20000, 2048), (12288, 8192)])
@pytest.mark.parametrize("lo,hi", [(0.99, 1.0), (0.999, 1.0), (0.05, 0.95)])
def test_twin_matches_oracle(oracle, T, W, lo, hi):
    from oracle.oracle import max_rel_error
    from paper_1709_04057_b200 import capi
    assert capi.scan_kernel_count(T, W) == 4  # probe, split scan, twin, fix-up
    rng = np.random.default_rng(T + W)
    lam = rng.uniform(lo, hi, (T, W)).astype(np.float32)
    x = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    h0 = rng.uniform(-1, 1, W).astype(np.float32)
    dh = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    L, X, H0, DH = (torch.from_numpy(a).cuda() for a in (lam, x, h0, dh))
    H, DL, DX, D0 = torch.empty_like(L), torch.empty_like(L), torch.empty_like(L), torch.empty_like(H0)
    capi.scan(_p(L), _p(X), _p(H0), _p(H), T, W)
    capi.scan_backward(_p(L), _p(H0), _p(H), _p(DH), _p(DL), _p(DX), _p(D0), T, W)
    torch.cuda.synchronize()
    cols = np.arange(0, W, W // 64)  # a channel subset keeps the oracle fast
    sub = lambda a: np.ascontiguousarray(a[:, cols])  # noqa: E731
    h_ref = oracle.scan_serial_wide(sub(lam), sub(x), h0[cols])
    g = oracle.scan_backward_wide(sub(lam), h0[cols], oracle.scan_serial(sub(lam), sub(x), h0[cols]), sub(dh))
    assert max_rel_error(H.cpu().numpy()[:, cols], h_ref) <= 1e-5
    assert max_rel_error(DL.cpu().numpy()[:, cols], g[0]) <= 1e-5
    assert max_rel_error(DX.cpu().numpy()[:, cols], g[1]) <= 1e-5
    assert max_rel_error(D0.cpu().numpy()[cols], g[2]) <= 1e-5


def test_twin_gated_backward(oracle):
    """The gated adjoint (dh * gate staged by the fused TMA backward) through
    the twin at slow decays: equal to the oracle's backward on the product."""
    from oracle.oracle import max_rel_error
    from paper_1709_04057_b200 import capi
    T, W = 20000, 2048
    rng = np.random.default_rng(5)
    lam = rng.uniform(0.99, 1.0, (T, W)).astype(np.float32)
    h = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    dh = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    gate = rng.uniform(0, 1, (T, W)).astype(np.float32)
    h0 = rng.uniform(-1, 1, W).astype(np.float32)
    L, Hh, DH, G, H0 = (torch.from_numpy(a).cuda() for a in (lam, h, dh, gate, h0))
    DL, DX, D0 = torch.empty_like(L), torch.empty_like(L), torch.empty_like(H0)
    capi.check(capi.lib.linrec_scan_backward_gated_f32(_p(L), _p(H0), _p(Hh), _p(DH), _p(G), _p(DL), _p(DX),
                                                       _p(D0), T, W, capi.PARALLEL, None,
                                                       torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    cols = np.arange(0, W, W // 64)
    sub = lambda a: np.ascontiguousarray(a[:, cols])  # noqa: E731
    prod = (dh * gate).astype(np.float32)
    g = oracle.scan_backward_wide(sub(lam), h0[cols], sub(h), sub(prod))
    assert max_rel_error(DL.cpu().numpy()[:, cols], g[0]) <= 1e-5
    assert max_rel_error(DX.cpu().numpy()[:, cols], g[1]) <= 1e-5
    assert max_rel_error(D0.cpu().numpy()[cols], g[2]) <= 1e-5
