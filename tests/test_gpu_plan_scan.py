"""The reference's chunked scan with an explicit ChunkPlan on the GPU
(linrec_scan_plan_* / linrec_scan_backward_plan_*, csrc/plan_scan.cu):
BIT-EXACT against the oracle's restatement of scan_parallel / scan_backward
with the same plan (recurrence.hpp:193-245, :365-377), including the
ScanSummaries P, R, C; the reference's hand-executed two-chunk example
(test_recurrence.cpp:75-99); validate_plan's errors (:84-94)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _plan_scan(lam, x, h0, plan):
    from paper_1709_04057_b200 import capi
    T, W = lam.shape[0], int(np.prod(lam.shape[1:]))
    L, X = _dev(lam), _dev(x)
    H0 = None if h0 is None else _dev(h0)
    H = torch.empty_like(L)
    p = len(plan)
    P, R, C = (torch.empty((p,) + lam.shape[1:], dtype=L.dtype, device="cuda") for _ in range(3))
    capi.scan_plan(L.data_ptr(), X.data_ptr(), None if H0 is None else H0.data_ptr(), H.data_ptr(), T, W, plan,
                   P.data_ptr(), R.data_ptr(), C.data_ptr(), lam.itemsize, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return H.cpu().numpy(), P.cpu().numpy(), R.cpu().numpy(), C.cpu().numpy()


def test_two_chunk_example_exposes_p_r_c():
    # test_recurrence.cpp:75-99: T=4, decays 1, impulses 1, h0 = 0, plan_chunks(4, 2)
    lam = np.ones((4, 1, 1)); x = np.ones((4, 1, 1)); h0 = np.zeros((1, 1))
    h, P, R, C = _plan_scan(lam, x, h0, [(1, 2), (3, 4)])
    assert P.ravel().tolist() == [1.0, 1.0]
    assert R.ravel().tolist() == [2.0, 2.0]
    assert C.ravel().tolist() == [2.0, 4.0]
    assert h.ravel().tolist() == [1.0, 2.0, 3.0, 4.0]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("T,B,D,workers", [(1, 1, 3, 1), (10, 2, 3, 4), (997, 3, 17, 7), (4096, 2, 256, 16),
                                           (5, 1, 8, 8), (20000, 1, 40, 3)])
def test_forward_bit_exact_with_the_plan(oracle, dtype, T, B, D, workers):
    rng = np.random.default_rng(T * 7 + D)
    lam = rng.uniform(-1, 1, (T, B, D)).astype(dtype)
    x = rng.uniform(-1, 1, (T, B, D)).astype(dtype)
    h0 = rng.uniform(-1, 1, (B, D)).astype(dtype)
    plan = oracle.plan_chunks(T, workers)
    h, P, R, C = _plan_scan(lam, x, h0, plan)
    rh, rP, rR, rC = oracle.scan_parallel(lam, x, h0, workers=workers, summaries=True)
    for a, b in ((h, rh), (P, rP), (R, rR), (C, rC)):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("T,W,workers", [(1, 4, 1), (10, 6, 4), (3001, 33, 5), (4096, 512, 16)])
def test_backward_bit_exact_with_the_plan(oracle, dtype, T, W, workers):
    from paper_1709_04057_b200 import capi
    rng = np.random.default_rng(T + W)
    lam = rng.uniform(0.05, 0.95, (T, W)).astype(dtype)
    x = rng.uniform(-1, 1, (T, W)).astype(dtype)
    h0 = rng.uniform(-1, 1, (W,)).astype(dtype)
    dh = rng.uniform(-1, 1, (T, W)).astype(dtype)
    h = oracle.scan_serial(lam, x, h0)
    plan = oracle.plan_chunks(T, workers)
    L, H0, H, DH = _dev(lam), _dev(h0), _dev(h), _dev(dh)
    DL, DX, D0 = torch.empty_like(L), torch.empty_like(L), torch.empty_like(H0)
    capi.scan_backward_plan(L.data_ptr(), H0.data_ptr(), H.data_ptr(), DH.data_ptr(), DL.data_ptr(), DX.data_ptr(),
                            D0.data_ptr(), T, W, plan, lam.itemsize, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    rl, rx, r0 = oracle.scan_backward(lam, h0, h, dh, workers=workers)
    assert np.array_equal(DL.cpu().numpy(), rl)
    assert np.array_equal(DX.cpu().numpy(), rx)
    assert np.array_equal(D0.cpu().numpy(), r0)


@pytest.mark.parametrize("plan,msg", [([], "no chunks"), ([(2, 10)], "first chunk must start at step 1"),
                                      ([(1, 9)], "last chunk must end at step T"),
                                      ([(1, 3), (5, 10)], "chunks must be contiguous"),
                                      ([(1, 5), (6, 5), (6, 10)], "chunk start exceeds end")])
def test_plan_errors_match_validate_plan(plan, msg):
    from paper_1709_04057_b200 import capi
    L = torch.ones(10, 4, device="cuda")
    H = torch.empty_like(L)
    with pytest.raises(capi.LinrecError, match=msg):
        capi.scan_plan(L.data_ptr(), L.data_ptr(), None, H.data_ptr(), 10, 4, plan)
