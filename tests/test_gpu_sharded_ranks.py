"""Sequence sharding through the CUDA kernels with REAL ranks: 2 or 3
processes share the one GPU of the test box and exchange carries either over
peer memory (CUDA-IPC mailboxes + release/acquire flags, csrc/p2p.cu -- the
default on one node; here the "peers" are processes on the same device) or
over gloo (host-staged all-gather), running paper_1709_04057_b200.sharded
exactly as bench.py does on a multi-GPU box.  Checked against the oracle."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import ROOT  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, T, W, lo, hi, seed, q, exchange="auto", reps=1, fail_rank=None):
    import sys
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1709_04057_b200.sharded import SequenceShardedScan, segment_bounds
        torch.cuda.set_device(0)
        rng = np.random.default_rng(seed)
        lam = rng.uniform(lo, hi, (T, W)).astype(np.float32)
        x = rng.uniform(-1, 1, (T, W)).astype(np.float32)
        h0 = rng.uniform(-1, 1, (W,)).astype(np.float32)
        dh = rng.uniform(-1, 1, (T, W)).astype(np.float32)
        s, e = segment_bounds(T, world, rank)
        cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        L, X, DH, H0 = cu(lam[s:e]), cu(x[s:e]), cu(dh[s:e]), cu(h0)
        H, DL, DX, DH0 = torch.empty_like(L), torch.empty_like(L), torch.empty_like(L), torch.zeros_like(H0)
        if rank == fail_rank:  # fault injection: this rank's CUDA-IPC mailbox allocation fails
            from paper_1709_04057_b200 import capi
            capi.lib.linrec_ipc_alloc = lambda *a: capi.ERR_CUDA
        run = SequenceShardedScan(T, W, stream=torch.cuda.current_stream(), exchange=exchange)
        want = "collective" if exchange == "collective" or fail_rank is not None else "p2p"
        assert run.exchange == want, (rank, run.exchange)
        for _ in range(reps):  # repeated steps reuse the mailboxes (epochs, acks)
            run.forward(L, X, H0, H)
            run.backward(L, H0, H, DH, DL, DX, DH0)
        torch.cuda.synchronize()
        run.close()
        q.put((rank, s, e, H.cpu().numpy(), DL.cpu().numpy(), DX.cpu().numpy(), DH0.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def _run_ranks(world, T, W, lo, hi, exchange, reps, fail_rank=None):
    import torch.multiprocessing as mp
    seed = T + W
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, W, lo, hi, seed, q, exchange, reps, fail_rank))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return seed, outs


def _check_ranks(oracle, outs, seed, T, W, lo, hi):
    from oracle.oracle import max_rel_error
    rng = np.random.default_rng(seed)
    lam = rng.uniform(lo, hi, (T, W)).astype(np.float32)
    x = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    h0 = rng.uniform(-1, 1, (W,)).astype(np.float32)
    dh = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    h_wide = oracle.scan_serial_wide(lam, x, h0)
    h_ref = oracle.scan_serial(lam, x, h0)
    g = oracle.scan_backward_wide(lam, h0, h_ref, dh)
    for rank, s, e, H, DL, DX, DH0 in outs:
        assert max_rel_error(H, h_wide[s:e]) <= 1e-5, rank
        assert max_rel_error(DL, g[0][s:e]) <= 1e-5, rank
        assert max_rel_error(DX, g[1][s:e]) <= 1e-5, rank
        if rank == 0:
            assert max_rel_error(DH0, g[2]) <= 1e-5


@pytest.mark.parametrize("world,fail_rank", [(2, 1), (3, 0)])
def test_mailbox_failure_falls_back_on_every_rank(oracle, world, fail_rank):
    """exchange="auto": when one rank cannot set up its CUDA-IPC mailbox,
    every rank agrees (an all-reduce of the setup flag) on the all-gather
    exchange instead of hanging in the peer-memory protocol, and the results
    still match the oracle."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    T, W = 20000, 64
    seed, outs = _run_ranks(world, T, W, 0.05, 0.95, "auto", 2, fail_rank)
    _check_ranks(oracle, outs, seed, T, W, 0.05, 0.95)


@pytest.mark.parametrize("exchange,reps", [("p2p", 3), ("collective", 1)])
@pytest.mark.parametrize("world,T,W,lo,hi", [(2, 40000, 128, 0.05, 0.95), (3, 30001, 64, 0.99, 1.0),
                                             (2, 5000, 12, -1.0, 1.0),
                                             (3, 9000, 384, 0.05, 0.95)])  # W > 256: fold kernel publishes
def test_sequence_sharded_ranks_on_gpu(oracle, world, T, W, lo, hi, exchange, reps):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    seed, outs = _run_ranks(world, T, W, lo, hi, exchange, reps)
    _check_ranks(oracle, outs, seed, T, W, lo, hi)


@pytest.mark.parametrize("workload,launch", [("c4", "torchrun"), ("c2", "torchrun"), ("c5", "self")])
def test_bench_two_ranks_sharing_the_gpu(workload, launch):
    """bench.py at --gpus 2 (ranks share the one GPU: gloo for the host-side
    plumbing, CUDA IPC for the carry mailboxes), launched by torchrun or by
    bench.py re-executing itself: one JSON line from rank 0 with the
    whole-job value, every guard passed."""
    import json
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, LINREC_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    args = ["--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", workload, "--no-e2e", "--no-cpu"]
    if launch == "torchrun":
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py")] + args
    else:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py")] + args
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["scaling"] == {"c4": "strong", "c2": "weak", "c5": "strong"}[workload]
    if workload == "c4":
        assert "peer-memory" in d["config"]["parallelism"]
    if workload == "c2":
        # the 1M-step workload beside the headline: 1 GPU and sequence-sharded
        assert d["c4"]["n_gpus"] == 1 and d["c4"]["guard_max_rel_err"] <= 1e-5
        s = d["c4_seq_sharded"]
        assert s["n_gpus"] == 2 and s["exchange"] == "p2p" and s["guard_max_rel_err"] <= 1e-5
        assert s["speedup"] > 0 and s["slow_decay"]["guard_max_rel_err"] <= 1e-5
    if workload == "c5":
        assert [p["sharding"] for p in d["points"]] == ["channel"] * 3 + ["sequence"] * 2
        assert all(p["guard_max_rel_err"] <= 1e-5 for p in d["points"])


def test_bench_refuses_missing_gpus():
    """--gpus N with fewer visible GPUs is an error, not a silent 1-GPU run."""
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n = torch.cuda.device_count() + 1
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "LINREC_BENCH_SHARE_GPU")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "3"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode != 0 and "GPU(s) visible" in (out.stderr + out.stdout)
