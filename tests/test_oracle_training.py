"""The training-loop oracle (oracle/train_oracle.py) pinned with the
reference's own training test cases (proj/tests/test_training.cpp), CPU only,
plus the product's Rng against the same known-answer values."""
import math

import numpy as np
import pytest


def cfg_tiny():
    from oracle.train_oracle import TrainConfig
    return TrainConfig(seq_len=12, input_dim=8, hidden=8, batch=4, max_iters=6, seed=7)  # test_training.cpp:13-22


def test_rng_known_answers_oracle_and_product():
    """test_rng.cpp:210-223 -- both restatements of rng.hpp."""
    from oracle.train_oracle import Rng as ORng
    from paper_1709_04057_b200.training import Rng as PRng
    for R in (ORng, PRng):
        first = R(42)
        d = first.draws(3) if R is ORng else first.next_u64_array(3)
        assert [int(v) for v in d] == [0xbdd732262feb6e95, 0x28efe333b266f103, 0x47526757130f9f52]
        assert R(42).split(7).seed == 0x583e77c90af5c134
        u = R(42).uniform(1, 0.0, 1.0) if R is ORng else R(42).uniform_array(1, 0.0, 1.0)
        assert float(u[0]) == 0.7415648787718233


def test_generated_batches_are_one_hot_with_sign_labels():
    from oracle.train_oracle import Rng, generate_batch
    rng = Rng(1)
    for T, b, p in ((1, 4, 2), (16, 3, 8), (5, 2, 128)):
        x, y = generate_batch(rng, T, b, p)
        assert x.shape == (T, b, p) and y.shape == (b,)
        assert np.all((x != 0).sum(-1) == 1)
        assert np.all(np.abs(x).max(-1) == 1.0) and np.all(np.abs(x.sum(-1)) == 1.0)
        assert np.all(np.abs(x[0, :, 0]) == 1.0)
        assert np.array_equal(y, (x[0, :, 0] > 0).astype(np.int32))
    with pytest.raises(RuntimeError):
        generate_batch(rng, 4, 2, 1)
    with pytest.raises(RuntimeError):
        generate_batch(rng, 0, 2, 4)


def test_class_balance_near_half():
    from oracle.train_oracle import Rng, generate_batch
    rng = Rng(3)
    pos = sum(int(generate_batch(rng, 1, 4, 2)[1].sum()) for _ in range(2500))
    assert abs(pos / 10000 - 0.5) <= 3 * 0.5 / math.sqrt(10000)


def test_zero_logits_give_ln2_and_adam_and_clip():
    from oracle.train_oracle import Trainer, clip_global_norm, softmax_loss
    loss, _, _ = softmax_loss(np.zeros((4, 2)), np.array([0, 1, 1, 0]))
    assert loss == pytest.approx(math.log(2.0), rel=1e-15)
    # adam hand-computed first step (test_training.cpp:177-189)
    t = Trainer.__new__(Trainer)
    t.cfg, t.step = type("C", (), {"learning_rate": 0.1})(), 0
    t.model = {"layers": [], "W_out": np.array([[1.0]]), "b_out": np.zeros(0)}
    t.m, t.v = [np.zeros(1), np.zeros(0)], [np.zeros(1), np.zeros(0)]
    t.adam([np.array([[0.5]]), np.zeros(0)])
    assert t.model["W_out"][0, 0] == pytest.approx(1.0 - 0.1 * 0.5 / (0.5 + 1e-8), rel=1e-12)
    # global-norm clip (test_training.cpp:191-204)
    a, b = np.array([3.0, 0.0]), np.array([4.0])
    assert clip_global_norm([a, b], 1.0) == pytest.approx(5.0)
    assert a[0] == pytest.approx(0.6, rel=1e-15) and b[0] == pytest.approx(0.8, rel=1e-15)
    c = np.array([0.25])
    clip_global_norm([c], 1.0)
    assert c[0] == 0.25


def test_convergence_detector():
    """test_training.cpp:206-237."""
    from oracle.train_oracle import TrainConfig, run_loop
    cfg = TrainConfig(window=5, max_iters=100)
    assert run_loop(cfg, lambda i: (0.1, 1.0)).iterations == 5
    r = run_loop(cfg, lambda i: (0.1, 0.9 if i == 3 else 1.0))
    assert r.converged and r.iterations == 8
    r = run_loop(cfg, lambda i: (0.1, 0.9))
    assert not r.converged and r.iterations == 100 and "maximum iterations" in r.diagnostic
    r = run_loop(cfg, lambda i: (float("nan") if i == 4 else 0.1, 0.5))
    assert r.diverged and r.iterations == 4 and "iteration 4" in r.diagnostic


def test_one_step_decreases_the_batch_loss(oracle):
    """test_training.cpp:155-175, fp64 oracle."""
    from oracle.train_oracle import Rng, Trainer, generate_batch, softmax_loss
    cfg = cfg_tiny()
    tr = Trainer(cfg, Rng(15), oracle=oracle)
    x, y = generate_batch(Rng(16), cfg.seq_len, cfg.batch, cfg.input_dim)
    before = softmax_loss(tr.forward(x)[-1], y)[0]
    tr.train_step(x, y)
    after = softmax_loss(tr.forward(x)[-1], y)[0]
    assert after < before


def test_experiment_reproducible(oracle):
    from oracle.train_oracle import run_experiment
    a, _ = run_experiment(cfg_tiny(), oracle=oracle)
    b, _ = run_experiment(cfg_tiny(), oracle=oracle)
    assert a.trace == b.trace
