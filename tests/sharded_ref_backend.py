"""Reference (CPU, float64) implementation of the primitive contract of
paper_1709_04057_b200.sharded.CudaBackend -- TEST INFRASTRUCTURE.

It restates what each sm_100a segment kernel computes (include/linrec_cuda.h,
csrc/segment.cu) with plain loops, so the CPU test-suite can drive the real
sharding orchestration (SequenceShardedScan) over gloo with world_size > 1.
"""
import numpy as np
import torch


def _np(t):
    return t.detach().numpy()


class RefBackend:
    def __init__(self, rows=5):
        self.rows = rows

    def tile_rows(self, T, W, backward):
        return self.rows

    def prod_rows(self, T, W, backward):
        return -(-T // self.rows)

    def segment_scan(self, lam, x, h0, h, seg_prod, agg, T, W):
        L, X, H = _np(lam).reshape(T, W), _np(x).reshape(T, W), _np(h).reshape(T, W)
        c = np.zeros(W) if h0 is None else _np(h0).reshape(W).copy()
        P = np.ones(W)
        SP = _np(seg_prod)
        for t in range(T):
            if t % self.rows == 0:
                SP[t // self.rows] = P
            c = L[t] * c + X[t]
            P = P * L[t]
            H[t] = c
        A = _np(agg)
        A[0], A[1] = P, c

    def segment_scan_backward(self, lam, hprev, h, dh, lam_next, dlam, dx, dh0, seg_prod, agg, T, W):
        L, H, DH = _np(lam).reshape(T, W), _np(h).reshape(T, W), _np(dh).reshape(T, W)
        DL, DX = _np(dlam).reshape(T, W), _np(dx).reshape(T, W)
        hp = np.zeros(W) if hprev is None else _np(hprev).reshape(W)
        ln = np.zeros(W) if lam_next is None else _np(lam_next).reshape(W)
        ntt = -(-T // self.rows)
        SP = _np(seg_prod)
        G = np.zeros(W)
        P = np.ones(W)
        for t in range(T - 1, -1, -1):
            tile = t // self.rows
            if t == min(T, (tile + 1) * self.rows) - 1:  # top row of the tile
                SP[ntt - 1 - tile] = P
            mu = L[t + 1] if t + 1 < T else ln
            G = mu * G + DH[t]
            P = P * mu
            DX[t] = G
            DL[t] = (H[t - 1] if t >= 1 else hp) * G
        _np(dh0).reshape(W)[:] = L[0] * G
        A = _np(agg)
        A[0], A[1] = L[0] * P, L[0] * G  # (A', B') ready for the exchange

    def compose(self, aggs, first, last, step, seed, out, W):
        AG = _np(aggs)
        c = np.zeros(W) if seed is None else _np(seed).reshape(W).copy()
        q = first
        while q != last:
            c = AG[q, 0] * c + AG[q, 1]
            q += step
        _np(out).reshape(W)[:] = c

    def fixup(self, lam, h, seg_prod, c_in, T, W, rows):
        if c_in is None:  # the scan above is complete: nothing pending without a carry
            return
        L, H, SP, c = _np(lam).reshape(T, W), _np(h).reshape(T, W), _np(seg_prod), _np(c_in).reshape(W)
        for tile in range(-(-T // rows)):
            e = SP[tile] * c
            for t in range(tile * rows, min(T, (tile + 1) * rows)):
                e = L[t] * e
                H[t] += e

    def fixup_backward(self, lam, hprev, h, lam_next, seg_prod, y_in, dlam, dx, T, W, rows):
        if y_in is None:
            return
        L, H, SP = _np(lam).reshape(T, W), _np(h).reshape(T, W), _np(seg_prod)
        DL, DX, y = _np(dlam).reshape(T, W), _np(dx).reshape(T, W), _np(y_in).reshape(W)
        hp = np.zeros(W) if hprev is None else _np(hprev).reshape(W)
        ln = np.zeros(W) if lam_next is None else _np(lam_next).reshape(W)
        ntt = -(-T // rows)
        for tile in range(ntt):
            e = SP[ntt - 1 - tile] * y
            for t in range(min(T, (tile + 1) * rows) - 1, tile * rows - 1, -1):
                mu = L[t + 1] if t + 1 < T else ln
                e = mu * e
                DX[t] += e
                DL[t] += (H[t - 1] if t >= 1 else hp) * e
