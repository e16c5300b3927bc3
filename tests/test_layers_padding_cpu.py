"""The Python layer API's zero padding to the kernels' widths (layers._Pad),
checked on CPU tensors: every gate block keeps its place and unpadding
restores the parameters exactly (the GPU parity of padded layers is in
tests/test_gpu_layers.py)."""
import pytest

torch = pytest.importorskip("torch")


def _layers():
    try:
        from paper_1709_04057_b200 import layers as L
    except ImportError as e:  # the package needs its built .so
        pytest.skip(str(e))
    return L


@pytest.mark.parametrize("m,n", [(1, 1), (3, 4), (5, 2), (8, 6), (4, 4)])
def test_padding_keeps_gate_blocks_and_round_trips(m, n):
    L = _layers()
    g = torch.Generator().manual_seed(m * 10 + n)
    p = L.gilr_lstm_init(g, m, n, 2.5, device="cpu")
    pad = L._Pad(m, n)
    q = pad.lstm(p)
    assert q.V.shape == (4 * pad.n4, pad.m4) and q.U.shape == (4 * pad.n4, pad.n4) and q.bias.shape == (4 * pad.n4,)
    for blk in range(4):  # block blk of the padded tensors holds block blk of the originals, zeros elsewhere
        assert torch.equal(q.V[blk * pad.n4: blk * pad.n4 + n, :m], p.V[blk * n:(blk + 1) * n])
        assert torch.equal(q.bias[blk * pad.n4: blk * pad.n4 + n], p.bias[blk * n:(blk + 1) * n])
        assert float(q.V[blk * pad.n4 + n:(blk + 1) * pad.n4].abs().sum()) == 0.0
    assert float(q.V[:, m:].abs().sum()) == 0.0 and float(q.U[:, n:].abs().sum()) == 0.0
    # unpadding a padded "gradient" restores the original exactly
    acc = torch.zeros_like(p.V)
    pad.add_rows(acc, q.V, 4, m, pad.m4)
    assert torch.equal(acc, p.V)
    accb = torch.zeros_like(p.bias)
    pad.add_vec(accb, q.bias, 4)
    assert torch.equal(accb, p.bias)


def test_qrnn_padding_per_tap():
    L = _layers()
    g = torch.Generator().manual_seed(3)
    p = L.qrnn_init(g, 3, 5, 4, device="cpu")
    pad = L._Pad(3, 5)
    q = pad.qrnn(p)
    assert q.W.shape == (4, 3 * pad.n4, pad.m4)
    for s in range(4):
        for blk in range(3):
            assert torch.equal(q.W[s, blk * pad.n4: blk * pad.n4 + 5, :3], p.W[s, blk * 5:(blk + 1) * 5])
    acc = torch.zeros_like(p.W)
    pad.add_rows(acc.view(3 * 4 * 5, 3), q.W.view(3 * 4 * pad.n4, pad.m4), 3 * 4, 3, pad.m4)
    assert torch.equal(acc, p.W)
