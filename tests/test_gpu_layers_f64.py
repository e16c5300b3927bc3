"""The layers in double precision on the GPU (linrec_*_f64 through
paper_1709_04057_b200.layers with float64 tensors) against the CPU oracle's
double instantiation (oracle/linrec_layers.c, DEFINE_LAYERS(double, ...)),
as the reference's test_layers.cpp runs its layers in double.

Tolerance: 1e-11 normwise (max|a-b|/max|ref|, oracles.hpp:73-82) for every
output, cache and gradient -- fp64 GEMMs and scans whose summation order
differs from the oracle's loops (the reference's own fp64 scan tolerances are
1e-12 / 1e-10, test_recurrence.cpp:150-162, verify.hpp:181)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _d(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _err(a, ref):
    from oracle.oracle import max_rel_error
    return max_rel_error(a.detach().cpu().numpy(), ref)


# {T, b, m, n}: test_layers.cpp's {1,1,1,1}, {7,2,3,4}, {33,3,5,2} plus wider
# and longer ones (the fp64 path takes any width, no padding)
SHAPES = [(1, 1, 1, 1), (7, 2, 3, 4), (33, 3, 5, 2), (40, 2, 8, 6), (129, 5, 36, 20), (300, 4, 64, 96)]


@pytest.mark.parametrize("mode", ["parallel", "serial"])
@pytest.mark.parametrize("T,b,m,n", SHAPES)
def test_gilr_lstm_f64_vs_oracle(oracle, T, b, m, n, mode):
    from oracle.oracle import gilr_lstm_params
    from paper_1709_04057_b200 import layers as L
    rng = np.random.default_rng(T * 100 + n)
    P = gilr_lstm_params(rng, m, n)
    x = rng.uniform(-1, 1, (T, b, m))
    htil0, c0 = rng.uniform(-1, 1, (b, n)), rng.uniform(-1, 1, (b, n))
    dh = rng.uniform(-1, 1, (T, b, n))
    h_ref, cache_ref = oracle.gilr_lstm_forward(P, x, htil0, c0)
    g_ref, dx_ref, dht0_ref, dc0_ref = oracle.gilr_lstm_backward(P, x, htil0, c0, cache_ref, dh)

    p = L.GilrLstmParams(L.GilrParams(_d(P["sU"]), _d(P["sV"]), _d(P["sbg"]), _d(P["sbz"])),
                         _d(P["U"]), _d(P["V"]), _d(P["bias"]))
    cache = L.GilrLstmCache()
    xd, ht0, cc0 = _d(x), _d(htil0), _d(c0)
    h = L.gilr_lstm_forward(p, xd, ht0, cc0, mode=mode, cache=cache)
    grads = L.GilrLstmGrads.zeros_like(p)
    dx, dht0, dc0 = L.gilr_lstm_backward(p, xd, ht0, cc0, cache, _d(dh), grads, mode=mode)
    torch.cuda.synchronize()
    assert h.dtype == torch.float64 and cache.gates.dtype == torch.float64
    assert _err(h, h_ref) < TOL
    assert _err(cache.c, cache_ref["c"]) < TOL
    assert _err(cache.surrogate_h(), cache_ref["htil"]) < TOL
    assert _err(cache.gates_interleaved(), cache_ref["gates"]) < TOL
    for nm, t in zip(["sU", "sV", "sbg", "sbz", "U", "V", "bias"], grads.tensors()):
        assert _err(t, g_ref[nm]) < TOL, nm
    assert _err(dx, dx_ref) < TOL
    assert _err(dht0, dht0_ref) < TOL
    assert _err(dc0, dc0_ref) < TOL


@pytest.mark.parametrize("act", ["tanh", "identity", "relu"])
@pytest.mark.parametrize("T,b,m,n", [(1, 1, 1, 1), (50, 3, 7, 5), (257, 2, 32, 48)])
def test_gilr_f64_vs_oracle(oracle, T, b, m, n, act):
    from paper_1709_04057_b200 import layers as L
    rng = np.random.default_rng(T + 7 * n)
    s = 1 / np.sqrt(m)
    P = {"U": rng.uniform(-s, s, (n, m)), "V": rng.uniform(-s, s, (n, m)), "b_g": rng.uniform(0.5, 1.5, n),
         "b_z": rng.uniform(-0.1, 0.1, n)}
    x, h0, dh = rng.uniform(-1, 1, (T, b, m)), rng.uniform(-1, 1, (b, n)), rng.uniform(-1, 1, (T, b, n))
    a = L.ACT[act]
    h_ref, c_ref = oracle.gilr_forward(P, x, h0, act=a)
    g_ref, dx_ref, dh0_ref = oracle.gilr_backward(P, x, h0, c_ref, h_ref, dh, act=a)
    p = L.GilrParams(_d(P["U"]), _d(P["V"]), _d(P["b_g"]), _d(P["b_z"]), act)
    cache = L.GilrCache()
    xd, h0d = _d(x), _d(h0)
    h = L.gilr_forward(p, xd, h0d, cache=cache)
    grads = L.GilrGrads.zeros_like(p)
    dx, dh0 = L.gilr_backward(p, xd, h0d, cache, _d(dh), grads)
    torch.cuda.synchronize()
    assert _err(h, h_ref) < TOL
    assert _err(cache.g, c_ref["g"]) < TOL and _err(cache.i, c_ref["i"]) < TOL
    for nm, t in zip(["U", "V", "b_g", "b_z"], grads.tensors()):
        assert _err(t, g_ref[nm]) < TOL, nm
    assert _err(dx, dx_ref) < TOL
    assert _err(dh0, dh0_ref) < TOL


@pytest.mark.parametrize("T,b,m,n,k", [(1, 1, 1, 1, 1), (9, 2, 3, 5, 3), (60, 3, 12, 10, 4), (200, 2, 40, 24, 2)])
def test_qrnn_f64_vs_oracle(oracle, T, b, m, n, k):
    from oracle.oracle import qrnn_params
    from paper_1709_04057_b200 import layers as L
    rng = np.random.default_rng(T * 10 + k)
    P = qrnn_params(rng, m, n, k)
    x, c0, dh = rng.uniform(-1, 1, (T, b, m)), rng.uniform(-1, 1, (b, n)), rng.uniform(-1, 1, (T, b, n))
    h_ref, cache_ref = oracle.qrnn_forward(P, x, c0)
    g_ref, dx_ref, dc0_ref = oracle.qrnn_backward(P, x, c0, cache_ref, dh)
    p = L.QrnnParams(_d(P["W"]), _d(P["bias"]))
    cache = L.QrnnCache()
    xd, c0d = _d(x), _d(c0)
    h = L.qrnn_forward(p, xd, c0d, cache=cache)
    grads = L.QrnnGrads.zeros_like(p)
    dx, dc0 = L.qrnn_backward(p, xd, c0d, cache, _d(dh), grads)
    torch.cuda.synchronize()
    assert _err(h, h_ref) < TOL
    assert _err(cache.gates_interleaved(), cache_ref["gates"]) < TOL
    assert _err(cache.c, cache_ref["c"]) < TOL
    assert _err(grads.W, g_ref["W"]) < TOL
    assert _err(grads.bias, g_ref["bias"]) < TOL
    assert _err(dx, dx_ref) < TOL
    assert _err(dc0, dc0_ref) < TOL


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (70, 33, 129), (5, 300, 4000)])
def test_gemm_f64_layouts(M, N, K, a_mn, b_mn):
    """linrec_gemm_f64: C (+)= A(m,k) B(n,k) for every operand layout,
    against a float64 torch matmul (1e-13 normwise), overwrite and accumulate."""
    import ctypes as C
    from paper_1709_04057_b200 import layers as L
    lib = L._bind()
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.rand(M, K, device="cuda", dtype=torch.float64, generator=g) - 0.5
    B = torch.rand(N, K, device="cuda", dtype=torch.float64, generator=g) - 0.5
    Ad = A.t().contiguous() if a_mn else A
    Bd = B.t().contiguous() if b_mn else B
    lda = M if a_mn else K
    ldb = N if b_mn else K
    C0 = torch.rand(M, N, device="cuda", dtype=torch.float64, generator=g)
    Cd = C0.clone()
    st = torch.cuda.current_stream().cuda_stream
    ref = A @ B.t()
    assert lib.linrec_gemm_f64(C.c_void_p(Ad.data_ptr()), a_mn, lda, C.c_void_p(Bd.data_ptr()), b_mn, ldb,
                               C.c_void_p(Cd.data_ptr()), N, M, N, K, 1, st) == 0
    torch.cuda.synchronize()
    assert ((Cd - (C0 + ref)).abs().max() / (C0 + ref).abs().max()).item() < 1e-13
    assert lib.linrec_gemm_f64(C.c_void_p(Ad.data_ptr()), a_mn, lda, C.c_void_p(Bd.data_ptr()), b_mn, ldb,
                               C.c_void_p(Cd.data_ptr()), N, M, N, K, 0, st) == 0
    torch.cuda.synchronize()
    assert ((Cd - ref).abs().max() / ref.abs().max()).item() < 1e-13


def test_f64_dtype_contract():
    """No silent casts: every tensor of a call must share x's dtype."""
    from paper_1709_04057_b200 import layers as L
    gen = torch.Generator().manual_seed(0)
    p = L.gilr_lstm_init(gen, 8, 8, dtype=torch.float64)
    x32 = torch.zeros(4, 1, 8, device="cuda")
    with pytest.raises(TypeError):
        L.gilr_lstm_forward(p, x32)
    x = torch.zeros(4, 1, 8, device="cuda", dtype=torch.float64)
    with pytest.raises(TypeError):
        L.gilr_lstm_forward(p, x, c0=torch.zeros(1, 8, device="cuda"))
    assert L.gilr_lstm_forward(p, x).dtype == torch.float64
