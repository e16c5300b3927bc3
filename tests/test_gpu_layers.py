"""GILR / GILR-LSTM layers on the GPU (paper_1709_04057_b200.layers, C ABI
linrec_gilr*_f32) against the CPU oracle (oracle/linrec_layers.c, pinned to
the reference's per-step layer oracle and finite differences by
tests/test_oracle_layers.py), run in float64 on the same inputs.

Tolerances (normwise max|a-b|/max|ref|, the reference metric oracles.hpp:73-82):
  precision "fp32" (3xTF32 + fp32 promotion): 2e-5 for every output and
    gradient -- fp32 activations, fp32 scans and fp32-grade GEMMs;
  precision "tf32": 5e-3 (operands rounded to 10 mantissa bits).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"fp32": 2e-5, "tf32": 5e-3}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _case(seed, T, b, m, n, act="tanh"):
    from oracle.oracle import gilr_lstm_params
    rng = np.random.default_rng(seed)
    P = gilr_lstm_params(rng, m, n)
    x = rng.uniform(-1, 1, (T, b, m))
    htil0 = rng.uniform(-1, 1, (b, n))
    c0 = rng.uniform(-1, 1, (b, n))
    dh = rng.uniform(-1, 1, (T, b, n))
    return P, x, htil0, c0, dh


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _params(P):
    from paper_1709_04057_b200 import layers as L
    return L.GilrLstmParams(L.GilrParams(_dev(P["sU"]), _dev(P["sV"]), _dev(P["sbg"]), _dev(P["sbz"])),
                            _dev(P["U"]), _dev(P["V"]), _dev(P["bias"]))


def _err(a, ref):
    from oracle.oracle import max_rel_error
    return max_rel_error(a.detach().cpu().numpy().astype(np.float64), ref)


SHAPES = [(1, 1, 4, 4), (37, 3, 8, 12), (200, 2, 16, 32), (129, 5, 36, 20), (64, 4, 64, 128),
          # widths that are not multiples of 4 (the reference's test_layers.cpp settings {T, b, m, n}
          # {1,1,1,1}, {7,2,3,4}, {33,3,5,2}; training's 8 -> 6): zero-padded in layers.py
          (1, 1, 1, 1), (7, 2, 3, 4), (33, 3, 5, 2), (40, 2, 8, 6)]


def _aligned(m, n):
    return m % 4 == 0 and n % 4 == 0


@pytest.mark.parametrize("precision", ["fp32", "tf32"])
@pytest.mark.parametrize("T,b,m,n", SHAPES)
def test_gilr_lstm_forward_backward_vs_oracle(oracle, T, b, m, n, precision):
    from paper_1709_04057_b200 import layers as L
    P, x, htil0, c0, dh = _case(T * 1000 + n, T, b, m, n)
    h_ref, cache_ref = oracle.gilr_lstm_forward(P, x, htil0, c0)
    g_ref, dx_ref, dht0_ref, dc0_ref = oracle.gilr_lstm_backward(P, x, htil0, c0, cache_ref, dh)

    p = _params(P)
    cache = L.GilrLstmCache()
    xd, ht0, cc0 = _dev(x), _dev(htil0), _dev(c0)
    h = L.gilr_lstm_forward(p, xd, ht0, cc0, precision=precision, cache=cache)
    grads = L.GilrLstmGrads.zeros_like(p)
    dx, dht0, dc0 = L.gilr_lstm_backward(p, xd, ht0, cc0, cache, _dev(dh), grads, precision=precision)
    torch.cuda.synchronize()
    tol = TOL[precision]
    assert _err(h, h_ref) < tol
    if _aligned(m, n):  # padded runs keep padded (opaque) caches
        assert _err(cache.c, cache_ref["c"]) < tol
        assert _err(cache.surrogate_h(), cache_ref["htil"]) < tol
        assert _err(cache.gates_interleaved(), cache_ref["gates"]) < tol
    names = ["sU", "sV", "sbg", "sbz", "U", "V", "bias"]
    for nm, t in zip(names, grads.tensors()):
        assert _err(t, g_ref[nm]) < tol, nm
    assert _err(dx, dx_ref) < tol
    assert _err(dht0, dht0_ref) < tol
    assert _err(dc0, dc0_ref) < tol


def test_gilr_lstm_serial_mode_and_accumulation(oracle):
    """mode="serial" runs the bit-exact scan kernels; gradients accumulate
    (+=) across calls exactly as the reference's grads do."""
    from paper_1709_04057_b200 import layers as L
    T, b, m, n = 50, 2, 8, 8
    P, x, htil0, c0, dh = _case(7, T, b, m, n)
    h_ref, cache_ref = oracle.gilr_lstm_forward(P, x, htil0, c0)
    g_ref, *_ = oracle.gilr_lstm_backward(P, x, htil0, c0, cache_ref, dh)
    p = _params(P)
    cache = L.GilrLstmCache()
    xd, ht0, cc0 = _dev(x), _dev(htil0), _dev(c0)
    h = L.gilr_lstm_forward(p, xd, ht0, cc0, mode="serial", cache=cache)
    grads = L.GilrLstmGrads.zeros_like(p)
    for _ in range(2):
        L.gilr_lstm_backward(p, xd, ht0, cc0, cache, _dev(dh), grads, mode="serial")
    torch.cuda.synchronize()
    assert _err(h, h_ref) < TOL["fp32"]
    assert _err(grads.V, 2 * g_ref["V"]) < TOL["fp32"]
    assert _err(grads.surrogate.b_g, 2 * g_ref["sbg"]) < TOL["fp32"]


def test_gilr_lstm_deterministic():
    from paper_1709_04057_b200 import layers as L
    T, b, m, n = 300, 4, 32, 64
    P, x, htil0, c0, dh = _case(3, T, b, m, n)
    outs = []
    for _ in range(2):
        p = _params(P)
        cache = L.GilrLstmCache()
        xd = _dev(x)
        h = L.gilr_lstm_forward(p, xd, _dev(htil0), _dev(c0), cache=cache)
        grads = L.GilrLstmGrads.zeros_like(p)
        dx, a, c = L.gilr_lstm_backward(p, xd, _dev(htil0), _dev(c0), cache, _dev(dh), grads)
        outs.append([h, dx, a, c] + grads.tensors())
    torch.cuda.synchronize()
    for u, v in zip(*outs):
        assert torch.equal(u, v)


@pytest.mark.parametrize("act", ["tanh", "identity", "relu"])
@pytest.mark.parametrize("T,b,m,n", [(90, 3, 12, 16), (33, 3, 5, 2), (7, 2, 3, 4)])
def test_gilr_layer_vs_oracle(oracle, act, T, b, m, n):
    """Standalone GILR layer (layers.hpp:78-133) against the oracle's GILR
    (the LSTM's surrogate path), every candidate activation."""
    import ctypes as C
    from oracle.oracle import _ptr
    from paper_1709_04057_b200 import layers as L
    rng = np.random.default_rng(11)
    U, V = rng.uniform(-.5, .5, (n, m)), rng.uniform(-.5, .5, (n, m))
    bg, bz = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    x, h0, dh = rng.uniform(-1, 1, (T, b, m)), rng.uniform(-1, 1, (b, n)), rng.uniform(-1, 1, (T, b, n))
    a = L.ACT[act]
    lib = oracle.lib
    oracle._layer_fns(np.float64)
    g_r, i_r, h_r = (np.empty((T, b, n)) for _ in range(3))
    lib.oracle_gilr_forward_f64(_ptr(x), _ptr(U), _ptr(V), _ptr(bg), _ptr(bz), _ptr(h0), a, _ptr(g_r), _ptr(i_r),
                                _ptr(h_r), T, b, m, n)
    dU, dV, dbg, dbz = np.zeros((n, m)), np.zeros((n, m)), np.zeros(n), np.zeros(n)
    dx_r, dh0_r = np.empty((T, b, m)), np.empty((b, n))
    lib.oracle_gilr_backward_f64(_ptr(x), _ptr(U), _ptr(V), _ptr(h0), a, _ptr(g_r), _ptr(i_r), _ptr(h_r), _ptr(dh),
                                 _ptr(dU), _ptr(dV), _ptr(dbg), _ptr(dbz), _ptr(dx_r), _ptr(dh0_r), T, b, m, n)
    p = L.GilrParams(_dev(U), _dev(V), _dev(bg), _dev(bz), act)
    cache = L.GilrCache()
    xd, h0d = _dev(x), _dev(h0)
    h = L.gilr_forward(p, xd, h0d, cache=cache)
    grads = L.GilrGrads.zeros_like(p)
    dx, dh0 = L.gilr_backward(p, xd, h0d, cache, _dev(dh), grads)
    torch.cuda.synchronize()
    tol = TOL["fp32"]
    assert _err(h, h_r) < tol
    if _aligned(m, n):
        assert _err(cache.g, g_r) < tol and _err(cache.i, i_r) < tol
    for t, r in zip(grads.tensors(), (dU, dV, dbg, dbz)):
        assert _err(t, r) < tol
    assert _err(dx, dx_r) < tol and _err(dh0, dh0_r) < tol


def test_layer_errors():
    from paper_1709_04057_b200 import capi, layers as L
    gen = torch.Generator().manual_seed(0)
    p = L.gilr_lstm_init(gen, 6, 8)  # m = 6: the C ABI wants multiples of 4 (layers.py pads)
    x = torch.zeros(4, 1, 6, device="cuda")
    with pytest.raises(capi.LinrecError, match="multiples of 4"):
        L._gilr_lstm_forward_core(p, x)
    p = L.gilr_lstm_init(gen, 8, 8)
    with pytest.raises(RuntimeError, match="input feature mismatch"):
        L.gilr_lstm_forward(p, torch.zeros(4, 1, 12, device="cuda"))
    with pytest.raises(TypeError):
        L.gilr_lstm_forward(p, torch.zeros(4, 1, 8, device="cuda", dtype=torch.float64))


def test_module_autograd_matches_explicit_backward():
    from paper_1709_04057_b200 import layers as L
    torch.manual_seed(0)
    mod = L.GilrLstm(16, 32, seed=5)
    x = (torch.rand(40, 3, 16, device="cuda") * 2 - 1).requires_grad_(True)
    h = mod(x)
    w = torch.rand_like(h)
    (h * w).sum().backward()
    p = L.GilrLstmParams(L.GilrParams(mod.sU.data, mod.sV.data, mod.sbg.data, mod.sbz.data), mod.U.data, mod.V.data,
                         mod.bias.data)
    cache = L.GilrLstmCache()
    z = torch.zeros(3, 32, device="cuda")
    L.gilr_lstm_forward(p, x.detach(), z, z, cache=cache)
    grads = L.GilrLstmGrads.zeros_like(p)
    dx, _, _ = L.gilr_lstm_backward(p, x.detach(), z, z, cache, w, grads)
    torch.cuda.synchronize()
    assert torch.equal(dx, x.grad)
    assert torch.equal(grads.U, mod.U.grad)


# ---- QRNN ----------------------------------------------------------------------------
QRNN_SHAPES = [(1, 1, 4, 4, 1), (37, 3, 8, 12, 2), (300, 2, 4, 16, 10), (50, 3, 8, 8, 4), (64, 2, 36, 20, 3),
               (200, 2, 16, 32, 10), (129, 4, 64, 128, 2),
               (9, 2, 3, 4, 1), (20, 1, 3, 4, 5), (33, 3, 5, 2, 3)]  # the reference's odd widths: padded


@pytest.mark.parametrize("precision", ["fp32", "tf32"])
@pytest.mark.parametrize("T,b,m,n,k", QRNN_SHAPES)
def test_qrnn_forward_backward_vs_oracle(oracle, T, b, m, n, k, precision):
    from oracle.oracle import qrnn_params
    from paper_1709_04057_b200 import layers as L
    rng = np.random.default_rng(T * 7 + k)
    P = qrnn_params(rng, m, n, k)
    x = rng.uniform(-1, 1, (T, b, m))
    c0 = rng.uniform(-1, 1, (b, n))
    dh = rng.uniform(-1, 1, (T, b, n))
    h_ref, cache_ref = oracle.qrnn_forward(P, x, c0)
    g_ref, dx_ref, dc0_ref = oracle.qrnn_backward(P, x, c0, cache_ref, dh)
    p = L.QrnnParams(_dev(P["W"]), _dev(P["bias"]))
    cache = L.QrnnCache()
    xd, c0d = _dev(x), _dev(c0)
    h = L.qrnn_forward(p, xd, c0d, precision=precision, cache=cache)
    grads = L.QrnnGrads.zeros_like(p)
    dx, dc0 = L.qrnn_backward(p, xd, c0d, cache, _dev(dh), grads, precision=precision)
    torch.cuda.synchronize()
    tol = TOL[precision]
    assert _err(h, h_ref) < tol
    if _aligned(m, n):
        assert _err(cache.gates_interleaved(), cache_ref["gates"]) < tol
        assert _err(cache.c, cache_ref["c"]) < tol
    assert _err(grads.W, g_ref["W"]) < tol
    assert _err(grads.bias, g_ref["bias"]) < tol
    assert _err(dx, dx_ref) < tol
    assert _err(dc0, dc0_ref) < tol


def test_qrnn_errors():
    from paper_1709_04057_b200 import layers as L
    gen = torch.Generator().manual_seed(0)
    p = L.qrnn_init(gen, 8, 8, 5)
    with pytest.raises(RuntimeError, match="window exceeds"):
        L.qrnn_forward(p, torch.zeros(4, 1, 8, device="cuda"))
    with pytest.raises(RuntimeError, match="window must be"):
        L.qrnn_init(gen, 8, 8, 0)
