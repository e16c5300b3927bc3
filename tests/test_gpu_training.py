"""The training experiment on the B200 (paper_1709_04057_b200.training)
against the CPU oracle (oracle/train_oracle.py, pinned by
tests/test_oracle_training.py):

* generate_batch on the GPU draws the reference's stream bit for bit;
* build_model initialises bit-identically (double draws cast to float);
* a few train_steps follow the fp64 oracle's loss trace and parameters
  (fp32 layers with 3xTF32 GEMMs: 1e-4 relative);
* runs are bit-reproducible; an easy configuration converges.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("T,b,p,counter", [(1, 4, 2, 0), (16, 3, 8, 5), (5, 2, 128, 1000), (300, 7, 12, 3)])
def test_generate_batch_matches_reference_stream(T, b, p, counter):
    from oracle.train_oracle import Rng as ORng, generate_batch as ogen
    from paper_1709_04057_b200.training import Rng, generate_batch
    r = Rng(99).split(2)
    r.counter = counter
    o = ORng(99).split(2)
    o.counter = counter
    batch = generate_batch(r, T, b, p)
    x, y = ogen(o, T, b, p, np.float32)
    torch.cuda.synchronize()
    assert np.array_equal(batch.inputs.cpu().numpy(), x)
    assert np.array_equal(batch.labels.cpu().numpy(), y)
    assert r.counter == o.counter == counter + b * T


def _cfgs(**kw):
    from oracle.train_oracle import TrainConfig as OC
    from paper_1709_04057_b200.training import TrainConfig
    base = dict(seq_len=12, input_dim=8, hidden=8, batch=4, max_iters=6, seed=7)
    base.update(kw)
    return TrainConfig(**base), OC(**base)


def test_build_model_matches_reference_init():
    from oracle.train_oracle import Rng as ORng, build_model as obuild, tensors
    from paper_1709_04057_b200.training import Rng, build_model
    cfg, ocfg = _cfgs()
    m = build_model(cfg, Rng(9).split(1))
    om = obuild(ocfg, ORng(9).split(1), np.float32)
    for a, b in zip(m.tensors(), tensors(om)):
        assert np.array_equal(a.cpu().numpy(), b)
    n, p = cfg.hidden, cfg.input_dim
    expect = 4 * (n * n + n * p + n) + 2 * (n * p + n) + 4 * (n * n + n * n + n) + 2 * (n * n + n) + 2 * n + 2
    assert m.parameter_count() == expect  # test_training.cpp:97-100


@pytest.mark.parametrize("hidden", [8, 6])  # 6: test_training.cpp's hidden width (padded in layers.py)
def test_train_steps_follow_the_oracle(oracle, hidden):
    from oracle.train_oracle import run_experiment as orun
    from paper_1709_04057_b200.training import run_experiment
    cfg, ocfg = _cfgs(max_iters=4, learning_rate=1e-2, hidden=hidden)
    keep = []
    rep = run_experiment(cfg, trainer_out=keep)
    orep, otr = orun(ocfg, oracle=oracle)
    assert rep.iterations == orep.iterations == 4
    for row, (it, loss, acc) in zip(rep.trace, orep.trace):
        assert row.loss == pytest.approx(loss, rel=1e-4)
        assert row.accuracy == acc
    from oracle.train_oracle import tensors
    for a, b in zip(keep[0].model.tensors(), tensors(otr.model)):
        d = np.abs(a.cpu().numpy().astype(np.float64) - b).max() / max(np.abs(b).max(), 1e-30)
        assert d < 1e-4


def test_runs_are_bit_reproducible():
    from paper_1709_04057_b200.training import run_experiment
    cfg, _ = _cfgs(seq_len=64, max_iters=5)
    a = run_experiment(cfg)
    b = run_experiment(cfg)
    assert [(r.loss, r.accuracy) for r in a.trace] == [(r.loss, r.accuracy) for r in b.trace]


def test_easy_problem_converges():
    """Short sequences, few symbols: the detector fires (five perfect batches)."""
    from paper_1709_04057_b200.training import run_experiment
    cfg, _ = _cfgs(seq_len=16, input_dim=4, hidden=16, batch=32, max_iters=600, learning_rate=1e-2, seed=3)
    rep = run_experiment(cfg)
    assert rep.converged, (rep.iterations, rep.trace[-1])


def test_config_errors():
    from paper_1709_04057_b200.training import TrainConfig, run_experiment
    with pytest.raises(RuntimeError, match="unknown arch"):
        run_experiment(TrainConfig(arch="gru"))
    with pytest.raises(RuntimeError, match="counts out of range"):
        run_experiment(TrainConfig(layers=3))


def test_long_sequence_step_follows_the_oracle(oracle):
    """T = 300: the gradient reaching step 1 through both layers and the
    readout matches the fp64 oracle after two Adam steps."""
    from oracle.train_oracle import run_experiment as orun, tensors
    from paper_1709_04057_b200.training import run_experiment
    cfg, ocfg = _cfgs(seq_len=300, max_iters=2, learning_rate=3e-3, gate_bias=3.0)
    keep = []
    rep = run_experiment(cfg, trainer_out=keep)
    orep, otr = orun(ocfg, oracle=oracle)
    for row, (it, loss, acc) in zip(rep.trace, orep.trace):
        assert row.loss == pytest.approx(loss, rel=1e-4)
    for a, b in zip(keep[0].model.tensors(), tensors(otr.model)):
        d = np.abs(a.cpu().numpy().astype(np.float64) - b).max() / max(np.abs(b).max(), 1e-30)
        assert d < 1e-4


def _dp_worker(rank, world, port, q):
    import os
    import sys
    import torch.distributed as dist
    from conftest import ROOT
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1709_04057_b200.training import TrainConfig, run_experiment
        cfg = TrainConfig(seq_len=40, input_dim=8, hidden=8, batch=6, max_iters=4, seed=5, learning_rate=1e-2)
        keep = []
        rep = run_experiment(cfg, trainer_out=keep, group=dist.group.WORLD)
        q.put((rank, [(r.loss, r.accuracy) for r in rep.trace], keep[0].model.params.flat.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_data_parallel_matches_single_gpu():
    """Two ranks sharing the GPU, each holding half of the global batch,
    follow the single-GPU trajectory (gradient sums in a different order:
    1e-5 relative) and stay bit-identical to each other."""
    import socket
    import torch.multiprocessing as mp
    from paper_1709_04057_b200.training import TrainConfig, run_experiment
    cfg = TrainConfig(seq_len=40, input_dim=8, hidden=8, batch=6, max_iters=4, seed=5, learning_rate=1e-2)
    keep = []
    ref = run_experiment(cfg, trainer_out=keep)
    ref_params = keep[0].model.params.flat.cpu().numpy()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, t0, p0), (_, t1, p1) = outs
    assert t0 == t1 and np.array_equal(p0, p1)
    for (l, a), r in zip(t0, ref.trace):
        assert l == pytest.approx(r.loss, rel=1e-5) and a == r.accuracy
    assert np.abs(p0 - ref_params).max() < 1e-5 * max(np.abs(ref_params).max(), 1.0)
