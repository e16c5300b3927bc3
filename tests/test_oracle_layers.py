"""Pin the GILR-LSTM oracle (oracle/linrec_layers.c) before trusting it:
forward against the reference's own per-step layer oracle
(proj/tests/support/layer_oracles.hpp via oracle/_ref, or the committed
fixture), backward against central finite differences as
proj/tests/test_layers.cpp:198-239 does.  CPU only."""
import os

import numpy as np
import pytest

from conftest import load_golden


def _case(seed=3, T=7, b=2, m=3, n=4):
    from oracle.oracle import gilr_lstm_params
    rng = np.random.default_rng(seed)
    P = gilr_lstm_params(rng, m, n)
    x = rng.uniform(-1, 1, (T, b, m))
    htil0 = rng.uniform(-1, 1, (b, n))
    c0 = rng.uniform(-1, 1, (b, n))
    w = rng.uniform(-1, 1, (T, b, n))
    return P, x, htil0, c0, w


def test_forward_matches_reference_layer_oracle(oracle):
    from oracle.oracle import REF_SO, RefLib, max_rel_error
    g = load_golden("gilr_lstm")
    P = {k[2:]: g[k] for k in g.files if k.startswith("P_")} if hasattr(g, "files") else {k[2:]: v for k, v in g.items() if k.startswith("P_")}
    h, _ = oracle.gilr_lstm_forward(P, g["x"], g["htil0"], g["c0"])
    assert max_rel_error(h, g["h_ref"]) <= 1e-12
    if os.path.exists(REF_SO):  # live check against the reference build
        P2, x, htil0, c0, _ = _case(seed=11, T=9, b=3, m=5, n=6)
        h2, _ = oracle.gilr_lstm_forward(P2, x, htil0, c0)
        assert max_rel_error(h2, RefLib().gilr_lstm_oracle(P2, x, htil0, c0)) <= 1e-12


def test_backward_matches_finite_differences(oracle):
    from oracle.oracle import grads_agree
    P, x, htil0, c0, w = _case()

    def loss(P_, x_, h0_, c0_):
        h, _ = oracle.gilr_lstm_forward(P_, x_, h0_, c0_)
        return float((h * w).sum())

    _, cache = oracle.gilr_lstm_forward(P, x, htil0, c0)
    grads, dx, dhtil0, dc0 = oracle.gilr_lstm_backward(P, x, htil0, c0, cache, w)
    eps = 1e-6

    def fd(arr, idx, rebuild):
        a_hi, a_lo = arr.copy(), arr.copy()
        a_hi[idx] += eps
        a_lo[idx] -= eps
        return (rebuild(a_hi) - rebuild(a_lo)) / (2 * eps)

    for name in P:
        for idx in np.ndindex(P[name].shape):
            num = fd(P[name], idx, lambda a: loss({**P, name: a}, x, htil0, c0))
            assert grads_agree(grads[name][idx], num, 1e-6), (name, idx)
    for idx in np.ndindex(x.shape):
        assert grads_agree(dx[idx], fd(x, idx, lambda a: loss(P, a, htil0, c0)), 1e-6)
    for idx in np.ndindex(htil0.shape):
        assert grads_agree(dhtil0[idx], fd(htil0, idx, lambda a: loss(P, x, a, c0)), 1e-6)
        assert grads_agree(dc0[idx], fd(c0, idx, lambda a: loss(P, x, htil0, a)), 1e-6)


def test_float32_oracle_close_to_float64(oracle):
    from oracle.oracle import max_rel_error
    P, x, htil0, c0, w = _case(seed=5, T=40, b=3, m=8, n=8)
    h64, c64 = oracle.gilr_lstm_forward(P, x, htil0, c0)
    P32 = {k: v.astype(np.float32) for k, v in P.items()}
    h32, c32 = oracle.gilr_lstm_forward(P32, x.astype(np.float32), htil0.astype(np.float32), c0.astype(np.float32))
    assert max_rel_error(h32, h64) < 1e-5
    g64 = oracle.gilr_lstm_backward(P, x, htil0, c0, c64, w)
    g32 = oracle.gilr_lstm_backward(P32, x.astype(np.float32), htil0.astype(np.float32), c0.astype(np.float32),
                                    c32, w.astype(np.float32))
    for k in P:
        assert max_rel_error(g32[0][k], g64[0][k]) < 1e-4, k
    assert max_rel_error(g32[1], g64[1]) < 1e-4


# ---- QRNN (layers.hpp:376-548) ----------------------------------------------------
def test_qrnn_forward_matches_reference_layer_oracle(oracle):
    """Forward against the reference's per-step QRNN (layer_oracles.hpp:84-114),
    windows k = 1, 2, 3 (test_layers.cpp:133-146)."""
    import os
    from oracle.oracle import REF_SO, RefLib, max_rel_error, qrnn_params
    g = load_golden("qrnn")
    for k in (1, 2, 3):
        P = {"W": g[f"k{k}_W"], "bias": g[f"k{k}_bias"]}
        h, _ = oracle.qrnn_forward(P, g[f"k{k}_x"], g[f"k{k}_c0"])
        assert max_rel_error(h, g[f"k{k}_h_ref"]) <= 1e-12, k
    if os.path.exists(REF_SO):
        rng = np.random.default_rng(4)
        P = qrnn_params(rng, 6, 5, 4)
        x = rng.uniform(-1, 1, (9, 2, 6))
        c0 = rng.uniform(-1, 1, (2, 5))
        h, _ = oracle.qrnn_forward(P, x, c0)
        assert max_rel_error(h, RefLib().qrnn_oracle(P, x, c0)) <= 1e-12


@pytest.mark.parametrize("k", [1, 2, 3])
def test_qrnn_backward_matches_finite_differences(oracle, k):
    """test_layers.cpp:241-270: every W, bias, x and c0 entry."""
    from oracle.oracle import grads_agree, qrnn_params
    rng = np.random.default_rng(10 + k)
    T, b, m, n = 6, 2, 3, 4
    P = qrnn_params(rng, m, n, k)
    x = rng.uniform(-1, 1, (T, b, m))
    c0 = rng.uniform(-1, 1, (b, n))
    w = rng.uniform(-1, 1, (T, b, n))

    def loss(P_, x_, c0_):
        h, _ = oracle.qrnn_forward(P_, x_, c0_)
        return float((h * w).sum())

    _, cache = oracle.qrnn_forward(P, x, c0)
    grads, dx, dc0 = oracle.qrnn_backward(P, x, c0, cache, w)
    eps = 1e-6

    def fd(arr, idx, rebuild):
        hi, lo = arr.copy(), arr.copy()
        hi[idx] += eps
        lo[idx] -= eps
        return (rebuild(hi) - rebuild(lo)) / (2 * eps)

    for name in ("W", "bias"):
        for idx in np.ndindex(P[name].shape):
            num = fd(P[name], idx, lambda a: loss({**P, name: a}, x, c0))
            assert grads_agree(grads[name][idx], num, 1e-6), (name, idx)
    for idx in np.ndindex(x.shape):
        assert grads_agree(dx[idx], fd(x, idx, lambda a: loss(P, a, c0)), 1e-6)
    for idx in np.ndindex(c0.shape):
        assert grads_agree(dc0[idx], fd(c0, idx, lambda a: loss(P, x, a)), 1e-6)
