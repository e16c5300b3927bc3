"""C3 at its BASELINE size (configs[2]: GILR-LSTM, T = 65536, B = 4,
m = n = 512): the product's fp32 layer (3xTF32 tcgen05 GEMMs + chained
scans) against an fp64 reference of the same formulas (tests/layer_f64.py),
every output and gradient at the layer tolerance 2e-5 normwise
(tests/test_gpu_layers.py) -- including the weight gradients, whose GEMMs
run over K = T*b = 262,144.  The fp64 reference is first pinned to the
plain-C layer oracle (oracle/linrec_layers.c) at small shapes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NAMES = ["sU", "sV", "sbg", "sbz", "U", "V", "bias"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rel(a, b):
    a, b = a.double(), b.double()
    return ((a - b).abs().max() / b.abs().max()).item()


def _inputs(seed, T, b, m, n):
    from oracle.oracle import gilr_lstm_params
    rng = np.random.default_rng(seed)
    # fp32-representable inputs: the fp32 product and the fp64 reference see the same numbers
    P = {k: v.astype(np.float32).astype(np.float64) for k, v in gilr_lstm_params(rng, m, n).items()}
    g = torch.Generator(device="cuda").manual_seed(seed)
    u = lambda *s: (torch.rand(*s, device="cuda", generator=g) * 2 - 1)  # noqa: E731  (fp32)
    return P, u(T, b, m), u(b, n), u(b, n), u(T, b, n)


@pytest.mark.parametrize("T,b,m,n", [(37, 3, 8, 12), (64, 4, 64, 128), (200, 2, 16, 32)])
def test_f64_composition_matches_c_oracle(oracle, T, b, m, n):
    from layer_f64 import gilr_lstm_f64
    P, x, ht0, c0, dh = _inputs(T + n, T, b, m, n)
    npx = lambda t: t.double().cpu().numpy()  # noqa: E731
    h_ref, cache = oracle.gilr_lstm_forward(P, npx(x), npx(ht0), npx(c0))
    g_ref, dx_ref, dht0_ref, dc0_ref = oracle.gilr_lstm_backward(P, npx(x), npx(ht0), npx(c0), cache, npx(dh))
    Pd = {k: torch.from_numpy(v).cuda() for k, v in P.items()}
    h, g, dx, dht0, dc0 = gilr_lstm_f64(Pd, x.double(), ht0.double(), c0.double(), dh.double())
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    assert _rel(h, t(h_ref)) < 1e-12
    for k in NAMES:
        assert _rel(g[k], t(g_ref[k])) < 1e-12, k
    assert _rel(dx, t(dx_ref)) < 1e-12
    assert _rel(dht0, t(dht0_ref)) < 1e-12
    assert _rel(dc0, t(dc0_ref)) < 1e-12


def test_c3_gilr_lstm_full_size():
    from layer_f64 import gilr_lstm_f64
    from paper_1709_04057_b200 import layers as L
    T, b, m, n = 65536, 4, 512, 512
    P, x, ht0, c0, dh = _inputs(3, T, b, m, n)
    f32 = lambda k: torch.from_numpy(P[k].astype(np.float32)).cuda()  # noqa: E731
    p = L.GilrLstmParams(L.GilrParams(f32("sU"), f32("sV"), f32("sbg"), f32("sbz")), f32("U"), f32("V"),
                         f32("bias"))
    cache = L.GilrLstmCache()
    h = L.gilr_lstm_forward(p, x, ht0, c0, precision="fp32", cache=cache)
    grads = L.GilrLstmGrads.zeros_like(p)
    dx, dht0, dc0 = L.gilr_lstm_backward(p, x, ht0, c0, cache, dh, grads, precision="fp32")
    torch.cuda.synchronize()
    ours = {"h": h, "dx": dx, "dhtil0": dht0, "dc0": dc0}
    ours.update(zip(NAMES, grads.tensors()))
    ours = {k: v.cpu() for k, v in ours.items()}  # free device memory for the fp64 reference
    del h, dx, dht0, dc0, grads, cache
    torch.cuda.empty_cache()
    Pd = {k: torch.from_numpy(v).cuda() for k, v in P.items()}
    h_r, g_r, dx_r, dht0_r, dc0_r = gilr_lstm_f64(Pd, x.double(), ht0.double(), c0.double(), dh.double())
    ref = {"h": h_r, "dx": dx_r, "dhtil0": dht0_r, "dc0": dc0_r}
    ref.update(g_r)
    errs = {k: _rel(ours[k].cuda(), ref[k]) for k in ours}
    bad = {k: e for k, e in errs.items() if not e < 2e-5}
    assert not bad, errs


@pytest.mark.parametrize("M,N", [(2048, 512), (512, 512)])
def test_gemm_weight_gradient_K_262144(M, N):
    """The C3 weight-gradient products: C[M][N] = sum_k A(k, m) B(k, n) over
    K = T*b = 262,144 with MN-major A (dpre^T) and B (x or htil_prev), split-K
    16 -- 3xTF32 with fp32 promotion must stay fp32-grade (<= 1e-5 normwise)
    where plain accumulation in the tensor core drifted to 2e-3."""
    from paper_1709_04057_b200 import capi
    K, splits = 262144, 16
    g = torch.Generator(device="cuda").manual_seed(M + N)
    A = torch.rand(K, M, device="cuda", generator=g) * 2 - 1   # MN-major: [K][M]
    B = torch.rand(K, N, device="cuda", generator=g) * 2 - 1
    C = torch.zeros(M, N, device="cuda")
    scratch = torch.empty(capi.gemm_scratch_bytes(M, N, splits) // 4 + 1, device="cuda")
    capi.gemm(A.data_ptr(), True, M, B.data_ptr(), True, N, C.data_ptr(), N, M, N, K, False, capi.PREC_FP32,
              splits, scratch.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = A.double().t() @ B.double()
    assert _rel(C, ref) <= 1e-5
