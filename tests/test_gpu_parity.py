"""GPU parity of the sm_100a scans against the CPU oracle and the reference's
golden fixtures (run on a B200: ``pytest -m gpu``).

Bars (BASELINE.json north_star):
* mode "serial" (per-channel kernel) -- BIT-EXACT vs the reference serial scan;
* mode "parallel" (chained scan)     -- normwise max|a-b|/max|ref| <= 1e-5 for
  fp32 and <= 1e-12 for fp64 (oracles.hpp:73-82, test_smoke.py:35), and also
  bounded against an fp64-accumulated serial scan; exact for the dyadic / integer
  identities; bit-identical run to run.
"""
import numpy as np
import pytest

from conftest import RANDOM_CASES, load_golden

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = {np.float32: 1e-5, np.float64: 1e-12}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.fixture(scope="module")
def lr():
    from paper_1709_04057_b200 import linrec
    return linrec


@pytest.fixture(params=["auto", "register"])
def policy(request):
    """Run a test with the TMA persistent kernels (auto) and with the
    register-tiled kernels forced."""
    from paper_1709_04057_b200 import capi
    capi.set_kernel_policy(capi.KERNEL_AUTO if request.param == "auto" else capi.KERNEL_REGISTER)
    yield request.param
    capi.set_kernel_policy(capi.KERNEL_AUTO)


@pytest.fixture(scope="module")
def ops():
    from paper_1709_04057_b200 import torch_ops
    return torch_ops


def rel(a, b):
    from oracle.oracle import max_rel_error
    return max_rel_error(a, b)


def tol_of(a):
    return TOL[np.float32] if a.dtype == np.float32 else TOL[np.float64]


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ---------------------------------------------------------------------------
# golden fixtures produced by the reference itself
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", RANDOM_CASES)
def test_golden_numpy_boundary(lr, name):
    g = load_golden(name)
    lam, x, h0, dh = g["lam"], g["x"], g["h0"], g["dh"]
    tol = tol_of(lam)
    hs = lr.scan(lam, x, h0, mode="serial")
    assert hs.dtype == lam.dtype and hs.shape == lam.shape
    assert np.array_equal(hs, g["h_serial"])
    assert np.array_equal(lr.scan(lam, x, h0, workers=1), g["h_serial"])  # one-chunk plan
    hp = lr.scan(lam, x, h0)
    assert rel(hp, g["h_serial"]) <= tol
    assert rel(hp, g["h_parallel_w4"]) <= tol
    assert rel(lr.scan(lam, x), g["h_zero_initial"]) <= tol
    gs = lr.scan_backward(lam, h0, g["h_serial"], dh, mode="serial")
    for got, key in zip(gs, ("dlam_serial", "dx_serial", "dh0_serial")):
        assert np.array_equal(got, g[key]), key
    gp = lr.scan_backward(lam, h0, g["h_serial"], dh)
    for got, key in zip(gp, ("dlam_serial", "dx_serial", "dh0_serial")):
        assert rel(got, g[key]) <= tol, key


@pytest.mark.parametrize("name", RANDOM_CASES)
def test_golden_device_boundary(ops, policy, name):
    g = load_golden(name)
    lam, x, h0, dh = (cuda(g[k]) for k in ("lam", "x", "h0", "dh"))
    tol = tol_of(g["lam"])
    assert np.array_equal(ops.scan(lam, x, h0, mode="serial").cpu().numpy(), g["h_serial"])
    h = ops.scan(lam, x, h0)
    assert rel(h.cpu().numpy(), g["h_serial"]) <= tol
    hs = cuda(g["h_serial"])
    d = ops.scan_backward(lam, h0, hs, dh, mode="serial")
    for got, key in zip(d, ("dlam_serial", "dx_serial", "dh0_serial")):
        assert np.array_equal(got.cpu().numpy(), g[key]), key
    d = ops.scan_backward(lam, h0, hs, dh)
    for got, key in zip(d, ("dlam_serial", "dx_serial", "dh0_serial")):
        assert rel(got.cpu().numpy(), g[key]) <= tol, key


def test_frozen_dyadic_values(lr, policy):
    g = load_golden("frozen")
    for dt in (np.float64, np.float32):
        lam, x, h0 = (g[k].astype(dt) for k in ("dyadic_lam", "dyadic_x", "dyadic_h0"))
        for mode in ("serial", "parallel"):
            h = lr.scan(lam, x, h0, mode=mode, workers=2)
            assert np.array_equal(h, g["dyadic_h"].astype(dt))
            dlam, dx, dh0 = lr.scan_backward(lam, h0, h, np.ones_like(lam), mode=mode, workers=2)
            assert np.array_equal(dx, g["dyadic_dx"].astype(dt))
            assert np.array_equal(dlam, g["dyadic_dlam"].astype(dt))
            assert np.array_equal(dh0, g["dyadic_dh0"].astype(dt))
        # T = 1 closes the chain rule exactly (test_recurrence.cpp:301-316)
        h = lr.scan(g["t1_lam"], g["t1_x"], g["t1_h0"], workers=2)
        dlam, dx, dh0 = lr.scan_backward(g["t1_lam"], g["t1_h0"], h, g["t1_dh"], workers=2)
        assert np.array_equal(dlam, g["t1_dlam"]) and np.array_equal(dx, g["t1_dh"])
        assert np.array_equal(dh0, g["t1_dh0"])


def test_identities_exact(lr, policy):
    g = load_golden("identities")
    for mode in ("serial", "parallel"):
        assert np.array_equal(lr.scan(g["ones_lam"], g["ones_x"], g["ones_h0"], mode=mode), g["ones_h"])
        assert np.array_equal(lr.scan(g["zeros_lam"], g["zeros_x"], g["zeros_h0"], mode=mode), g["zeros_x"])
    # larger lambda==1 integer prefix sums through many tiles and columns
    T, W = 3000, 260
    rng = np.random.default_rng(0)
    x = rng.integers(-8, 9, size=(T, 1, W)).astype(np.float32)
    h = lr.scan(np.ones_like(x), x)
    assert np.array_equal(h, np.cumsum(x, axis=0, dtype=np.float64).astype(np.float32))


# ---------------------------------------------------------------------------
# the reference's own smoke tests, re-run against the GPU module
# (proj/tests/python/test_smoke.py)
# ---------------------------------------------------------------------------
def smoke_instance(rng, T=33, b=2, n=5, dtype=np.float64):
    decays = rng.uniform(-1.0, 1.0, size=(T, b, n)).astype(dtype)
    impulses = rng.uniform(-1.0, 1.0, size=(T, b, n)).astype(dtype)
    initial = rng.uniform(-1.0, 1.0, size=(b, n)).astype(dtype)
    return decays, impulses, initial


def reference_scan(decays, impulses, initial):
    h = np.empty_like(impulses)
    prev = initial.astype(np.float64)
    for t in range(decays.shape[0]):
        prev = decays[t].astype(np.float64) * prev + impulses[t].astype(np.float64)
        h[t] = prev.astype(h.dtype)
    return h


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_smoke_scan_matches_reference(lr, dtype):
    rng = np.random.default_rng(7)
    decays, impulses, initial = smoke_instance(rng, dtype=dtype)
    h = lr.scan(decays, impulses, initial, workers=4)
    assert h.shape == decays.shape and h.dtype == dtype
    ref = reference_scan(decays, impulses, initial)
    assert np.abs(h - ref).max() / np.abs(ref).max() < TOL[dtype]


def test_smoke_serial_and_single_chunk_bitwise(lr):
    rng = np.random.default_rng(8)
    decays, impulses, initial = smoke_instance(rng, T=17)
    assert np.array_equal(lr.scan(decays, impulses, initial, mode="serial"),
                          lr.scan(decays, impulses, initial, workers=1))


def test_smoke_default_initial_is_zero(lr):
    rng = np.random.default_rng(9)
    decays, impulses, initial = smoke_instance(rng, T=5)
    assert np.array_equal(lr.scan(decays, impulses, np.zeros_like(initial)), lr.scan(decays, impulses))


def test_smoke_backward_matches_finite_differences(lr):
    rng = np.random.default_rng(10)
    decays, impulses, initial = smoke_instance(rng, T=6, b=1, n=3)
    d_h = rng.uniform(-1.0, 1.0, size=decays.shape)
    h = lr.scan(decays, impulses, initial, workers=3)
    d_decays, d_impulses, d_initial = lr.scan_backward(decays, initial, h, d_h, workers=3)
    assert d_decays.shape == decays.shape and d_initial.shape == initial.shape
    eps = 1e-6
    for pos, (arr, grad) in enumerate([(decays, d_decays), (impulses, d_impulses), (initial, d_initial)]):
        idx = tuple(rng.integers(0, s) for s in arr.shape)
        hi_args = [decays, impulses, initial]
        lo_args = [decays, impulses, initial]
        bumped, dipped = arr.copy(), arr.copy()
        bumped[idx] += eps
        dipped[idx] -= eps
        hi_args[pos], lo_args[pos] = bumped, dipped
        fd = ((lr.scan(*hi_args) * d_h).sum() - (lr.scan(*lo_args) * d_h).sum()) / (2 * eps)
        assert grad[idx] == pytest.approx(fd, rel=1e-5, abs=1e-8)


# ---------------------------------------------------------------------------
# shape sweep through the C ABI (every lane split Q, vector / scalar paths,
# ragged tiles) against the oracle
# ---------------------------------------------------------------------------
SWEEP_W = [1, 2, 3, 4, 5, 8, 12, 16, 17, 31, 64, 100, 127, 128, 129, 256, 1000, 1024, 4100]
SWEEP_T = [1, 2, 31, 47, 48, 49, 257, 1000]


@pytest.mark.parametrize("W", SWEEP_W)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_sweep_against_oracle(ops, oracle, policy, W, dtype):
    rng = np.random.default_rng(W)
    for T in SWEEP_T:
        lam = rng.uniform(-1, 1, (T, 1, W)).astype(dtype)
        x = rng.uniform(-1, 1, (T, 1, W)).astype(dtype)
        h0 = rng.uniform(-1, 1, (1, W)).astype(dtype)
        dh = rng.uniform(-1, 1, (T, 1, W)).astype(dtype)
        ref = oracle.scan_serial(lam, x, h0)
        gref = oracle.scan_backward(lam, h0, ref, dh)
        tl, tx, th0, tdh, tref = cuda(lam), cuda(x), cuda(h0), cuda(dh), cuda(ref)
        h = ops.scan(tl, tx, th0).cpu().numpy()
        assert rel(h, ref) <= TOL[dtype], (T, W)
        assert np.array_equal(ops.scan(tl, tx, th0, mode="serial").cpu().numpy(), ref), (T, W)
        for got, want in zip(ops.scan_backward(tl, th0, tref, tdh), gref):
            assert rel(got.cpu().numpy(), want) <= TOL[dtype], (T, W)
        for got, want in zip(ops.scan_backward(tl, th0, tref, tdh, mode="serial"), gref):
            assert np.array_equal(got.cpu().numpy(), want), (T, W)
        if dtype == np.float32:
            wide = oracle.scan_serial_wide(lam, x, h0)
            assert rel(h, wide) <= TOL[dtype]


def test_unaligned_pointers_take_scalar_path(ops, oracle):
    """Views offset by one element are not 16-byte aligned: the VEC=1 kernels."""
    rng = np.random.default_rng(5)
    T, W = 300, 64
    base = torch.from_numpy(rng.uniform(0.05, 0.95, T * W + 1).astype(np.float32)).cuda()
    xb = torch.from_numpy(rng.uniform(-1, 1, T * W + 1).astype(np.float32)).cuda()
    lam = base[1:].view(T, 1, W)
    x = xb[1:].view(T, 1, W)
    h = ops.scan(lam, x)
    ref = oracle.scan_serial(lam.cpu().numpy(), x.cpu().numpy())
    assert rel(h.cpu().numpy(), ref) <= 1e-5


def test_deterministic_run_to_run(ops, policy):
    g = torch.Generator(device="cuda").manual_seed(0)
    T, W = 40000, 512
    lam = torch.rand(T, 1, W, device="cuda", generator=g) * 0.9 + 0.05
    x = torch.rand(T, 1, W, device="cuda", generator=g) * 2 - 1
    dh = torch.rand(T, 1, W, device="cuda", generator=g) * 2 - 1
    h1 = ops.scan(lam, x)
    h2 = ops.scan(lam, x)
    assert torch.equal(h1, h2)
    g1 = ops.scan_backward(lam, None, h1, dh)
    g2 = ops.scan_backward(lam, None, h1, dh)
    assert all(torch.equal(a, b) for a, b in zip(g1, g2))


def test_stress_decay_distributions(ops, oracle, policy):
    rng = np.random.default_rng(11)
    T, W = 20000, 96
    for lo, hi in ((0.99, 1.0), (-1.0, 1.0), (0.05, 0.95), (0.999, 1.0)):
        lam = rng.uniform(lo, hi, (T, 1, W)).astype(np.float32)
        x = rng.uniform(-1, 1, (T, 1, W)).astype(np.float32)
        dh = rng.uniform(-1, 1, (T, 1, W)).astype(np.float32)
        ref = oracle.scan_serial(lam, x)
        wide = oracle.scan_serial_wide(lam, x)
        h = ops.scan(cuda(lam), cuda(x)).cpu().numpy()
        assert rel(h, ref) <= 1e-5 and rel(h, wide) <= 1e-5, (lo, hi)
        gw = oracle.scan_backward_wide(lam, None, ref, dh)
        got = ops.scan_backward(cuda(lam), None, cuda(ref), cuda(dh))
        for a, b in zip(got, gw):
            assert rel(a.cpu().numpy(), b) <= 1e-5, (lo, hi)


# ---------------------------------------------------------------------------
# host (numpy) pipeline with several chunks; segment chaining; workspaces
# ---------------------------------------------------------------------------
def test_host_pipeline_multi_chunk(lr, oracle):
    rng = np.random.default_rng(12)
    T, b, n = 70000, 2, 512  # 280 MB per array -> 5 host chunks of 64 MB
    lam = rng.uniform(0.05, 0.95, (T, b, n)).astype(np.float32)
    x = rng.uniform(-1, 1, (T, b, n)).astype(np.float32)
    h0 = rng.uniform(-1, 1, (b, n)).astype(np.float32)
    dh = rng.uniform(-1, 1, (T, b, n)).astype(np.float32)
    ref = oracle.scan_serial(lam, x, h0)
    assert np.array_equal(lr.scan(lam, x, h0, mode="serial"), ref)
    assert rel(lr.scan(lam, x, h0), ref) <= 1e-5
    gref = oracle.scan_backward(lam, h0, ref, dh)
    for a, r in zip(lr.scan_backward(lam, h0, ref, dh, mode="serial"), gref):
        assert np.array_equal(a, r)
    for a, r in zip(lr.scan_backward(lam, h0, ref, dh), gref):
        assert rel(a, r) <= 1e-5


def test_backward_segments_chain_bit_exactly(oracle, policy):
    from paper_1709_04057_b200 import capi
    rng = np.random.default_rng(13)
    T, W, k = 1000, 36, 377
    lam = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    x = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    h0 = rng.uniform(-1, 1, (W,)).astype(np.float32)
    dh = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    h = oracle.scan_serial(lam, x, h0)
    gref = oracle.scan_backward(lam, h0, h, dh)
    tl, th, tdh, th0 = cuda(lam), cuda(h), cuda(dh), cuda(h0)
    dlam = torch.empty_like(tl)
    dx = torch.empty_like(tl)
    dh0 = torch.empty_like(th0)
    junk = torch.empty_like(th0)
    st = torch.cuda.current_stream().cuda_stream
    for mode in (capi.SERIAL, capi.PARALLEL):
        # tail [k, T) first (true end), then head [0, k) chained through lam[k], G[k]
        capi.scan_backward_segment(tl[k:].data_ptr(), th[k - 1].data_ptr(), th[k:].data_ptr(),
                                   tdh[k:].data_ptr(), None, None, dlam[k:].data_ptr(),
                                   dx[k:].data_ptr(), junk.data_ptr(), T - k, W, mode, 4, None, st)
        capi.scan_backward_segment(tl.data_ptr(), th0.data_ptr(), th.data_ptr(), tdh.data_ptr(),
                                   tl[k].data_ptr(), dx[k].data_ptr(), dlam.data_ptr(), dx.data_ptr(),
                                   dh0.data_ptr(), k, W, mode, 4, None, st)
        got = (dlam.cpu().numpy(), dx.cpu().numpy(), dh0.cpu().numpy())
        for a, r in zip(got, gref):
            if mode == capi.SERIAL:
                assert np.array_equal(a, r)
            else:
                assert rel(a, r) <= 1e-5


def test_workspace_reuse_and_cuda_graph_replay(ops, oracle, policy):
    """Epoch/ticket state lives on the device: a captured graph replays correctly."""
    from paper_1709_04057_b200 import capi
    ws = capi.Workspace(0)
    rng = np.random.default_rng(14)
    shapes = [(5000, 1, 384), (70, 3, 9), (4096, 1, 256), (1, 1, 7)]
    for T, b, n in shapes * 2:  # alternate shapes on one workspace
        lam = rng.uniform(0.05, 0.95, (T, b, n)).astype(np.float32)
        x = rng.uniform(-1, 1, (T, b, n)).astype(np.float32)
        h = ops.scan(cuda(lam), cuda(x), ws=ws).cpu().numpy()
        assert rel(h, oracle.scan_serial(lam, x)) <= 1e-5
    T, W = 8192, 512
    lam = torch.rand(T, 1, W, device="cuda") * 0.9 + 0.05
    x = torch.rand(T, 1, W, device="cuda") * 2 - 1
    out = torch.empty_like(lam)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ops.scan(lam, x, out=out, ws=ws)  # warm-up reserves the workspace
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        ops.scan(lam, x, out=out, ws=ws)
    ref = oracle.scan_serial(lam.cpu().numpy(), x.cpu().numpy())
    for _ in range(3):
        x.mul_(-1.0)
        ref = -ref
        out.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert rel(out.cpu().numpy(), ref) <= 1e-5
    ws.close()


def test_autograd_function(ops, oracle):
    rng = np.random.default_rng(15)
    T, b, n = 500, 2, 40
    lam = cuda(rng.uniform(0.05, 0.95, (T, b, n))).requires_grad_()
    x = cuda(rng.uniform(-1, 1, (T, b, n))).requires_grad_()
    h0 = cuda(rng.uniform(-1, 1, (b, n))).requires_grad_()
    w = cuda(rng.uniform(-1, 1, (T, b, n)))
    (ops.linear_recurrence(lam, x, h0) * w).sum().backward()
    h = oracle.scan_serial(lam.detach().cpu().numpy(), x.detach().cpu().numpy(), h0.detach().cpu().numpy())
    g = oracle.scan_backward(lam.detach().cpu().numpy(), h0.detach().cpu().numpy(), h, w.cpu().numpy())
    for t, r in zip((lam, x, h0), g):
        assert rel(t.grad.cpu().numpy(), r) <= 1e-12


def test_first_nonfinite(oracle):
    from paper_1709_04057_b200 import capi
    a = torch.zeros(9, 2, 4, device="cuda")
    assert capi.first_nonfinite(a.data_ptr(), a.numel()) == -1
    a[5, 1, 2] = float("nan")
    a[7, 0, 0] = float("inf")
    idx = capi.first_nonfinite(a.data_ptr(), a.numel())
    assert idx == 5 * 8 + 1 * 4 + 2 == oracle.first_nonfinite(a.cpu().numpy())


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_check_finite_pinpoints_the_poisoned_element(dtype):
    """test_recurrence.cpp:328-350 through the device path: screening off
    passes garbage through; on, the error names the tensor and the 1-based
    step (t=6), batch (b=1) and feature (n=2) of the NaN in impulses."""
    from paper_1709_04057_b200 import torch_ops
    g = torch.Generator(device="cuda").manual_seed(108)
    lam = torch.empty(9, 2, 4, device="cuda", dtype=dtype).uniform_(0.05, 0.95, generator=g)
    x = torch.empty_like(lam).uniform_(-1, 1, generator=g)
    h0 = torch.empty(2, 4, device="cuda", dtype=dtype).uniform_(-1, 1, generator=g)
    x[5, 1, 2] = float("nan")
    torch_ops.scan(lam, x, h0)  # no throw
    for mode in ("serial", "parallel"):
        with pytest.raises(RuntimeError) as e:
            torch_ops.scan(lam, x, h0, mode=mode, check_finite=True)
        msg = str(e.value)
        assert "non-finite value in impulses" in msg and "t=6" in msg and "b=1" in msg and "n=2" in msg
    x[5, 1, 2] = 0.5
    h0[0, 3] = float("inf")
    with pytest.raises(RuntimeError, match=r"non-finite value in initial at \[b=0, n=3\]"):
        torch_ops.scan(lam, x, h0, check_finite=True)
    h0[0, 3] = 0.0
    h = torch_ops.scan(lam, x, h0, check_finite=True)
    dh = torch.ones_like(h)
    dh[8, 0, 1] = float("-inf")
    with pytest.raises(RuntimeError, match=r"non-finite value in d_h at \[t=9, b=0, n=1\]"):
        torch_ops.scan_backward(lam, h0, h, dh, check_finite=True)
    lam[0, 0, 0] = float("nan")
    with pytest.raises(RuntimeError, match=r"non-finite value in decays at \[t=1, b=0, n=0\]"):
        torch_ops.scan_backward(lam, h0, h, dh, check_finite=True)


def test_torch_ops_shape_contract():
    """h0 / out buffers of the wrong shape are contract errors, not
    out-of-bounds device accesses (the C ABI sees pointers only)."""
    from paper_1709_04057_b200 import torch_ops
    lam = torch.rand(5, 2, 3, device="cuda")
    with pytest.raises(RuntimeError, match=r"initial state \[3\] does not match \[2, 3\]"):
        torch_ops.scan(lam, lam, torch.zeros(3, device="cuda"))
    with pytest.raises(RuntimeError, match="shape mismatch"):
        torch_ops.scan(lam, lam, out=torch.empty(5, 2, 2, device="cuda"))
    h = torch_ops.scan(lam, lam)
    with pytest.raises(RuntimeError, match="shape mismatch"):
        torch_ops.scan_backward(lam, None, h, h, out=(torch.empty_like(h), torch.empty_like(h),
                                                      torch.empty(3, device="cuda")))
    # a non-contiguous h0 works through autograd forward AND backward
    lam_r = lam.clone().requires_grad_()
    h0 = torch.rand(3, 2, device="cuda").t().requires_grad_()
    torch_ops.linear_recurrence(lam_r, lam, h0).sum().backward()
    assert h0.grad.shape == (2, 3)


def test_cuda_array_interface_zero_copy(lr, oracle):
    rng = np.random.default_rng(16)
    lam = rng.uniform(0.05, 0.95, (300, 2, 20)).astype(np.float32)
    x = rng.uniform(-1, 1, (300, 2, 20)).astype(np.float32)
    out = lr.scan(cuda(lam), cuda(x))
    assert isinstance(out, lr.DeviceArray)
    torch.cuda.synchronize()
    h = torch.as_tensor(out, device="cuda").cpu().numpy()
    assert rel(h, oracle.scan_serial(lam, x)) <= 1e-5


@pytest.mark.parametrize("T,W", [(65536, 8192), (1 << 20, 128), (4096, 256), (3000, 1000)])
def test_benchmark_shapes_channel_subset(ops, oracle, T, W):
    """BASELINE configs at full size: every channel is an independent chain, so
    the oracle is run on a strided subset of channels over the FULL T."""
    g = torch.Generator(device="cuda").manual_seed(T + W)
    lam = torch.rand(T, 1, W, device="cuda", generator=g) * 0.9 + 0.05
    x = torch.rand(T, 1, W, device="cuda", generator=g) * 2 - 1
    h0 = torch.rand(1, W, device="cuda", generator=g) * 2 - 1
    dh = torch.rand(T, 1, W, device="cuda", generator=g) * 2 - 1
    h = ops.scan(lam, x, h0)
    dlam, dx, dh0 = ops.scan_backward(lam, h0, h, dh)
    cols = sorted(set(list(range(0, W, max(1, W // 61))) + [W - 1]))
    sub = lambda t: t[..., cols].contiguous().cpu().numpy()  # noqa: E731
    ref = oracle.scan_serial(sub(lam), sub(x), sub(h0))
    assert rel(sub(h), ref) <= 1e-5
    gref = oracle.scan_backward(sub(lam), sub(h0), sub(h), sub(dh))
    for a, r in zip((dlam, dx, dh0), gref):
        assert rel(sub(a), r) <= 1e-5
    # full-tensor properties: finite everywhere, and dx's first row = dh0 / lam_0
    assert torch.isfinite(h).all() and torch.isfinite(dlam).all() and torch.isfinite(dx).all()
    assert rel(dh0.cpu().numpy(), (lam[0] * dx[0]).cpu().numpy()) <= 1e-5


def test_tma_and_register_kernels_agree(ops):
    from paper_1709_04057_b200 import capi
    g = torch.Generator(device="cuda").manual_seed(3)
    T, W = 20000, 2048
    lam = torch.rand(T, 1, W, device="cuda", generator=g) * 0.9 + 0.05
    x = torch.rand(T, 1, W, device="cuda", generator=g) * 2 - 1
    dh = torch.rand(T, 1, W, device="cuda", generator=g) * 2 - 1
    h_auto = ops.scan(lam, x)
    g_auto = ops.scan_backward(lam, None, h_auto, dh)
    capi.set_kernel_policy(capi.KERNEL_REGISTER)
    try:
        h_reg = ops.scan(lam, x)
        g_reg = ops.scan_backward(lam, None, h_auto, dh)
    finally:
        capi.set_kernel_policy(capi.KERNEL_AUTO)
    hs = ops.scan(lam, x, mode="serial")
    for hh in (h_auto, h_reg):
        assert ((hh - hs).abs().max() / hs.abs().max()).item() <= 1e-5
    for a, b in zip(g_auto, g_reg):
        assert ((a - b).abs().max() / b.abs().max()).item() <= 1e-5


@pytest.mark.parametrize("T,W,lo,hi", [
    (300000, 16, 0.05, 0.95),    # 1 column -> virtual T-segments (fix-up of the leading tile)
    (100000, 8, 0.999, 1.0),     # decays ~1: fix-up spans whole segments
    (50000, 3, -1.0, 1.0),       # scalar register kernels with virtual segments
    (1 << 18, 128, 0.5, 1.0),
])
def test_virtual_segments_against_oracle(ops, oracle, policy, T, W, lo, hi):
    rng = np.random.default_rng(T + W)
    lam = rng.uniform(lo, hi, (T, 1, W)).astype(np.float32)
    x = rng.uniform(-1, 1, (T, 1, W)).astype(np.float32)
    h0 = rng.uniform(-1, 1, (1, W)).astype(np.float32)
    dh = rng.uniform(-1, 1, (T, 1, W)).astype(np.float32)
    tl, tx, th0, tdh = cuda(lam), cuda(x), cuda(h0), cuda(dh)
    h = ops.scan(tl, tx, th0)
    wide = oracle.scan_serial_wide(lam, x, h0)
    assert rel(h.cpu().numpy(), wide) <= 1e-5
    assert torch.equal(h, ops.scan(tl, tx, th0))  # deterministic with the stitch too
    ref = oracle.scan_serial(lam, x, h0)
    g = ops.scan_backward(tl, th0, cuda(ref), tdh)
    gw = oracle.scan_backward_wide(lam, h0, ref, dh)
    for a, r in zip(g, gw):
        assert rel(a.cpu().numpy(), r) <= 1e-5


@pytest.mark.parametrize("T,W,lo,hi", [(300000, 16, 0.05, 0.95), (100000, 8, 0.999, 1.0), (50000, 3, -1.0, 1.0)])
def test_virtual_segments_fp64_against_oracle(ops, oracle, T, W, lo, hi):
    """fp64 through the same stitch (the fix-up's in-CTA carry fold in
    double): bit-identical serial reference, 1e-12 normwise."""
    rng = np.random.default_rng(T + W + 1)
    lam = rng.uniform(lo, hi, (T, 1, W))
    x = rng.uniform(-1, 1, (T, 1, W))
    h0 = rng.uniform(-1, 1, (1, W))
    dh = rng.uniform(-1, 1, (T, 1, W))
    tl, tx, th0, tdh = cuda(lam), cuda(x), cuda(h0), cuda(dh)
    h = ops.scan(tl, tx, th0)
    ref = oracle.scan_serial(lam, x, h0)
    assert rel(h.cpu().numpy(), ref) <= 1e-12
    assert torch.equal(h, ops.scan(tl, tx, th0))
    g = ops.scan_backward(tl, th0, cuda(ref), tdh)
    gr = oracle.scan_backward(lam, h0, ref, dh)
    for a, r in zip(g, gr):
        assert rel(a.cpu().numpy(), r) <= 1e-12
