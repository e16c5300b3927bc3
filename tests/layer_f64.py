"""GILR-LSTM forward + backward in float64 on the GPU -- TEST INFRASTRUCTURE.

The plain-C layer oracle (oracle/linrec_layers.c, pinned to the reference's
own per-step layer oracle and to finite differences) is a triple loop: at
the C3 size (T = 65536, b = 4, m = n = 512: ~4e12 flop) it would run for
hours.  This module restates the same formulas -- oracle_gilr_forward /
_backward and oracle_gilr_lstm_forward / _backward, i.e. layers.hpp:78-133
and :245-375 -- as float64 torch matrix products plus the fp64 SERIAL scan
kernels of this repo (bit-identical to the oracle's serial scan), so the
product's fp32 layer can be checked against an fp64 reference at full size.
tests/test_gpu_c3_fullsize.py pins this composition to the C oracle at small
shapes first.  Never imported by the product package.
"""
import torch


def _scan(lam, imp, h0):
    """h_t = lam_t h_{t-1} + imp_t, fp64, serial kernel (recurrence.hpp:169-184)."""
    from paper_1709_04057_b200 import capi
    T = lam.shape[0]
    W = lam[0].numel()
    h = torch.empty_like(lam)
    capi.scan(lam.data_ptr(), imp.data_ptr(), None if h0 is None else h0.data_ptr(), h.data_ptr(), T, W,
              capi.SERIAL, 8, None, torch.cuda.current_stream().cuda_stream)
    return h


def _scan_bwd(lam, h0, h, dh):
    """(dlam, G, dh0) of the serial backward (recurrence.hpp:273-348)."""
    from paper_1709_04057_b200 import capi
    T = lam.shape[0]
    W = lam[0].numel()
    dlam, G = torch.empty_like(lam), torch.empty_like(lam)
    dh0 = torch.empty(lam.shape[1:], dtype=lam.dtype, device=lam.device)
    capi.scan_backward(lam.data_ptr(), None if h0 is None else h0.data_ptr(), h.data_ptr(), dh.data_ptr(),
                       dlam.data_ptr(), G.data_ptr(), dh0.data_ptr(), T, W, capi.SERIAL, 8, None,
                       torch.cuda.current_stream().cuda_stream)
    return dlam, G, dh0


def gilr_lstm_f64(P, x, htil0, c0, dh):
    """P: dict of float64 CUDA tensors sU, sV [n, m], sbg, sbz [n], U [4n, n],
    V [4n, m], bias [4n]; x [T, b, m], htil0, c0 [b, n], dh [T, b, n].
    Returns (h, grads dict, dx, dhtil0, dc0) -- grads from zero."""
    T, b, m = x.shape
    n = P["U"].shape[1]
    R = T * b
    X = x.reshape(R, m)
    # surrogate GILR (gilr_forward :78-100, activation tanh)
    g = torch.sigmoid(X @ P["sU"].t() + P["sbg"])
    i = torch.tanh(X @ P["sV"].t() + P["sbz"])
    htil = _scan(g.view(T, b, n).contiguous(), ((1 - g) * i).view(T, b, n).contiguous(), htil0)
    hp = torch.cat([htil0.view(1, b, n), htil[:-1]]).reshape(R, n)       # shift_right (:213-220)
    pre = X @ P["V"].t() + hp @ P["U"].t() + P["bias"]                    # [R, 4n]: f, i, o, z
    f, ig, o = (torch.sigmoid(pre[:, k * n:(k + 1) * n]) for k in range(3))
    z = torch.tanh(pre[:, 3 * n:])
    c = _scan(f.reshape(T, b, n).contiguous(), (ig * z).reshape(T, b, n).contiguous(), c0)
    C = c.reshape(R, n)
    h = (o * C).view(T, b, n)
    # backward (gilr_lstm_backward :295-375)
    D = dh.reshape(R, n)
    dO = D * C
    dc = (D * o).view(T, b, n).contiguous()
    df, diz, dc0 = _scan_bwd(f.reshape(T, b, n).contiguous(), c0, c, dc)
    df, diz = df.reshape(R, n), diz.reshape(R, n)
    dpre = torch.cat([df * f * (1 - f), diz * z * ig * (1 - ig), dO * o * (1 - o), diz * ig * (1 - z * z)], dim=1)
    grads = {"U": dpre.t() @ hp, "V": dpre.t() @ X, "bias": dpre.sum(0)}
    dx = dpre @ P["V"]
    dhp = dpre @ P["U"]
    dht = torch.cat([dhp[b:], torch.zeros(b, n, dtype=dhp.dtype, device=dhp.device)]).view(T, b, n).contiguous()
    # surrogate backward (gilr_backward :102-133) with d_htil = dhtil_prev shifted
    dl, G, dh0s = _scan_bwd(g.view(T, b, n).contiguous(), htil0, htil, dht)
    dl, G = dl.reshape(R, n), G.reshape(R, n)
    dg = (dl - G * i) * g * (1 - g)
    di = G * (1 - g) * (1 - i * i)
    grads.update(sU=dg.t() @ X, sbg=dg.sum(0), sV=di.t() @ X, sbz=di.sum(0))
    dx = dx + dg @ P["sU"] + di @ P["sV"]
    dhtil0 = dh0s + dhp[:b].view(b, n)
    return h, grads, dx.view(T, b, m), dhtil0, dc0
