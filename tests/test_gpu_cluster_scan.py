"""Cluster scans (csrc/cluster_scan.cu: a thread-block cluster splits a short
sequence, CTAs exchanging chunk aggregates through distributed shared
memory) against the oracle: the forward h, the backward dlam, dx, dh0 and the
segment backward's lam_next / g_next carry-in, over the shapes the dispatch
sends there (fp32, 512 <= T <= 4096, W / 4 <= 2 x SMs): the reference's C1
(T = 4096, W = 256), the paper's kernel-table widths (W = 4, 32, 128), ragged
T and W, columns narrower than 32 channels, decays near 1.  Tolerance: the
reference's 1e-5 normwise for fp32 (test_recurrence.cpp:164-171)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _d(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _p(t):
    return None if t is None else t.data_ptr()


SHAPES = [(512, 4), (600, 8), (1000, 32), (4096, 256), (4096, 4), (4096, 32), (4096, 128), (2048, 128),
          (777, 64), (4095, 12), (3000, 1184), (1024, 16), (513, 36), (2049, 1024), (2048, 1024)]


@pytest.mark.parametrize("lo,hi", [(0.05, 0.95), (0.99, 1.0), (-1.0, 1.0)])
@pytest.mark.parametrize("T,W", SHAPES)
def test_cluster_scan_vs_oracle(oracle, T, W, lo, hi):
    from oracle.oracle import max_rel_error
    from paper_1709_04057_b200 import capi
    assert capi.lib.linrec_scan_kernel_count(T, W, 4, 0, capi.PARALLEL) == 1  # one launch
    rng = np.random.default_rng(T * 7 + W)
    lam = rng.uniform(lo, hi, (T, W)).astype(np.float32)
    x = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    h0 = rng.uniform(-1, 1, W).astype(np.float32)
    dh = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    L, X, H0, DH = _d(lam), _d(x), _d(h0), _d(dh)
    H, DL, DX, DH0 = torch.empty_like(L), torch.empty_like(L), torch.empty_like(L), torch.empty_like(H0)
    capi.scan(_p(L), _p(X), _p(H0), _p(H), T, W)
    capi.scan_backward(_p(L), _p(H0), _p(H), _p(DH), _p(DL), _p(DX), _p(DH0), T, W)
    torch.cuda.synchronize()
    h_ref = oracle.scan_serial_wide(lam, x, h0)
    g = oracle.scan_backward_wide(lam, h0, oracle.scan_serial(lam, x, h0), dh)
    assert max_rel_error(H.cpu().numpy(), h_ref) <= 1e-5
    assert max_rel_error(DL.cpu().numpy(), g[0]) <= 1e-5
    assert max_rel_error(DX.cpu().numpy(), g[1]) <= 1e-5
    assert max_rel_error(DH0.cpu().numpy(), g[2]) <= 1e-5


@pytest.mark.parametrize("T,W", [(4096, 256), (1000, 32), (600, 4), (2000, 64)])
def test_cluster_scan_segment_carry_in_and_no_initial(oracle, T, W):
    """scan_backward_segment's lam_next / g_next (the carry entering from the
    rows after the range) and NULL h0 run through the cluster kernels: equal
    to the backward of the longer sequence restricted to the range."""
    from oracle.oracle import max_rel_error
    from paper_1709_04057_b200 import capi
    rng = np.random.default_rng(T + W)
    Tl = T + 37  # the full sequence; the kernel sees rows [0, T) and the carry of the rest
    lam = rng.uniform(0.5, 1.0, (Tl, W)).astype(np.float32)
    x = rng.uniform(-1, 1, (Tl, W)).astype(np.float32)
    dh = rng.uniform(-1, 1, (Tl, W)).astype(np.float32)
    h_full = oracle.scan_serial(lam, x, None)
    g_full = oracle.scan_backward_wide(lam, None, h_full, dh)
    # G at row T of the full backward = the carry entering the range from above
    dx_full = g_full[1]
    L, DH, Hh = _d(lam[:T]), _d(dh[:T]), _d(h_full[:T])
    LN, GN = _d(lam[T]), _d(dx_full[T])
    DL, DX, DH0 = torch.empty_like(L), torch.empty_like(L), torch.empty(W, device="cuda")
    capi.scan_backward_segment(_p(L), None, _p(Hh), _p(DH), _p(LN), _p(GN), _p(DL), _p(DX), _p(DH0), T, W)
    H = torch.empty_like(L)
    capi.scan(_p(L), _p(_d(x[:T])), None, _p(H), T, W)
    torch.cuda.synchronize()
    assert max_rel_error(H.cpu().numpy(), oracle.scan_serial_wide(lam[:T], x[:T], None)) <= 1e-5
    assert max_rel_error(DX.cpu().numpy(), dx_full[:T]) <= 1e-5
    assert max_rel_error(DL.cpu().numpy(), g_full[0][:T]) <= 1e-5
    assert max_rel_error(DH0.cpu().numpy(), g_full[2]) <= 1e-5


def test_cluster_scan_deterministic():
    """Fixed association: bit-identical run to run."""
    from paper_1709_04057_b200 import capi
    g = torch.Generator(device="cuda").manual_seed(3)
    T, W = 4096, 256
    L = torch.rand(T, W, device="cuda", generator=g)
    X = torch.rand(T, W, device="cuda", generator=g) - 0.5
    outs = []
    for _ in range(3):
        H = torch.empty_like(L)
        capi.scan(_p(L), _p(X), None, _p(H), T, W)
        outs.append(H)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
