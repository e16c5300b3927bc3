"""Sequence / channel sharding orchestration on CPU: world_size 2 and 3 over
gloo (127.0.0.1), driving paper_1709_04057_b200.sharded with the reference
backend (tests/sharded_ref_backend.py), checked against the unsharded oracle
scan.  The CUDA kernels behind the same primitives are checked on the GPU in
tests/test_gpu_segments.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, T, b, n, rows, use_h0, seed, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1709_04057_b200.sharded import SequenceShardedScan, segment_bounds
        from sharded_ref_backend import RefBackend
        rng = np.random.default_rng(seed)
        lam = rng.uniform(-1.0, 1.0, (T, b, n))
        x = rng.uniform(-1.0, 1.0, (T, b, n))
        h0 = rng.uniform(-1.0, 1.0, (b, n)) if use_h0 else None
        dh = rng.uniform(-1.0, 1.0, (T, b, n))
        s, e = segment_bounds(T, world, rank)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))  # noqa: E731
        L, X, DH = t(lam[s:e]), t(x[s:e]), t(dh[s:e])
        H0 = t(h0) if use_h0 else None
        H = torch.empty_like(L)
        DL, DX = torch.empty_like(L), torch.empty_like(L)
        DH0 = torch.zeros(b, n, dtype=torch.float64)
        runner = SequenceShardedScan(T, b * n, backend=RefBackend(rows), device=torch.device("cpu"))
        # the runner allocates float32 scratch; the reference backend works in float64
        for name in ("seg_prod_f", "seg_prod_b", "agg", "aggs", "c_in", "y_in", "dh0_loc", "ones", "zeros"):
            setattr(runner, name, getattr(runner, name).double())
        runner.forward(L, X, H0, H)
        runner.backward(L, H0, H, DH, DL, DX, DH0)
        # a standalone backward with the halo exchange must agree too
        runner.hprev = None
        DL2, DX2 = torch.empty_like(L), torch.empty_like(L)
        DH02 = torch.zeros(b, n, dtype=torch.float64)
        runner.backward(L, H0, H, DH, DL2, DX2, DH02)
        q.put((rank, s, e, H.numpy(), DL.numpy(), DX.numpy(), DH0.numpy(), DL2.numpy(), DX2.numpy(), DH02.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,T,rows,use_h0", [(2, 23, 5, True), (3, 31, 4, False), (2, 8, 3, True), (3, 9, 2, True)])
def test_sequence_sharded_matches_unsharded(oracle, world, T, rows, use_h0):
    b, n, seed = 2, 3, 100 + world * T
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, b, n, rows, use_h0, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(seed)
    lam = rng.uniform(-1.0, 1.0, (T, b, n))
    x = rng.uniform(-1.0, 1.0, (T, b, n))
    h0 = rng.uniform(-1.0, 1.0, (b, n)) if use_h0 else None
    dh = rng.uniform(-1.0, 1.0, (T, b, n))
    h_ref = oracle.scan_serial(lam, x, h0)
    dl_ref, dx_ref, dh0_ref = oracle.scan_backward(lam, h0, h_ref, dh)
    from oracle.oracle import max_rel_error
    for rank, s, e, H, DL, DX, DH0, DL2, DX2, DH02 in outs:
        assert max_rel_error(H, h_ref[s:e]) < 1e-12, rank
        for a, b_ in ((DL, dl_ref[s:e]), (DX, dx_ref[s:e]), (DL2, dl_ref[s:e]), (DX2, dx_ref[s:e])):
            assert max_rel_error(a, b_) < 1e-12, rank
        if rank == 0:
            assert max_rel_error(DH0, dh0_ref) < 1e-12
            assert max_rel_error(DH02, dh0_ref) < 1e-12


def test_segment_and_channel_bounds():
    from paper_1709_04057_b200.sharded import channel_shard, segment_bounds
    for T in (1, 7, 8, 1 << 20):
        for world in (1, 2, 3, 8):
            b = [segment_bounds(T, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == T
            assert all(e == s2 for (_, e), (s2, _) in zip(b, b[1:]))
            sizes = [e - s for s, e in b]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    assert channel_shard(8192 * 8, 8, 3) == (3 * 8192, 4 * 8192)
