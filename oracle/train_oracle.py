"""CPU oracle of the reference's training experiment -- TEST INFRASTRUCTURE ONLY.

Restates proj/include/linrec/training.hpp (generate_batch :30-43,
build_model :110-123, model_forward :160-190, softmax_loss :193-222,
model_backward :224-246, Adam :248-273, clip_global_norm :275-288,
Trainer :291-333, run_loop :343-380, run_experiment :384-436) on top of the
layer oracle (oracle/linrec_layers.c via oracle.Oracle), with its own
restatement of the reference Rng (rng.hpp:15-52).  Only tests/ and bench.py
may import it; the product never does.

The reference's own training path needs Eigen (absent), so this
restatement is pinned piecewise: the layers by tests/test_oracle_layers.py,
the RNG by the reference's known-answer values (test_rng.cpp:210-223), and
the loss / clip / Adam / convergence pieces by the reference's own test cases
(test_training.cpp:113-237), re-run in tests/test_oracle_training.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .oracle import Oracle

M64 = (1 << 64) - 1


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


class Rng:
    """rng.hpp:15-52."""

    def __init__(self, seed, counter=0):
        self.seed, self.counter = seed & M64, counter

    def split(self, stream):
        with np.errstate(over="ignore"):
            z = np.array([self.seed ^ ((0xD1B54A32D192ED03 * (stream + 1)) & M64)], dtype=np.uint64)
            return Rng(int(_mix(z)[0]))

    def draws(self, count):
        c = np.arange(self.counter + 1, self.counter + 1 + count, dtype=np.uint64)
        self.counter += count
        with np.errstate(over="ignore"):
            return _mix(np.uint64(self.seed) + c * np.uint64(0x9E3779B97F4A7C15))

    def uniform(self, count, lo, hi):
        return lo + (hi - lo) * ((self.draws(count) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)


def generate_batch(rng: Rng, T, b, p, dtype=np.float64):
    if p < 2:
        raise RuntimeError("generate_batch: input_dim must be >= 2")
    if T < 1:
        raise RuntimeError("generate_batch: seq_len must be >= 1")
    x = np.zeros((T, b, p), dtype)
    labels = np.zeros(b, np.int32)
    for r in range(b):  # draw order of the reference: coin, then T-1 below(p)
        d = rng.draws(T)
        pos = bool(d[0] & np.uint64(1))
        labels[r] = 1 if pos else 0
        x[0, r, 0] = 1.0 if pos else -1.0
        hot = (d[1:] % np.uint64(p)).astype(np.int64)
        x[np.arange(1, T), r, hot] = 1.0
    return x, labels


@dataclass
class TrainConfig:
    seq_len: int = 1024
    input_dim: int = 128
    hidden: int = 64
    batch: int = 32
    learning_rate: float = 1e-3
    max_iters: int = 5000
    seed: int = 0
    window: int = 5
    gate_bias: float = 1.0
    clip_norm: float = 1.0


def init_uniform(rng, rows, cols, scale, dtype):
    return rng.uniform(rows * cols, -scale, scale).astype(dtype).reshape(rows, cols)


def build_model(cfg, rng: Rng, dtype=np.float64):
    p, n = cfg.input_dim, cfg.hidden
    layers = []
    for r, m in ((rng.split(101), p), (rng.split(102), n)):
        sub = r.split(1)
        s = 1.0 / math.sqrt(m)
        P = {"sU": init_uniform(sub, n, m, s, dtype), "sV": init_uniform(sub, n, m, s, dtype),
             "sbg": np.full(n, cfg.gate_bias, dtype), "sbz": np.zeros(n, dtype)}
        P["U"] = init_uniform(r, 4 * n, n, 1.0 / math.sqrt(n), dtype)
        P["V"] = init_uniform(r, 4 * n, m, 1.0 / math.sqrt(m), dtype)
        bias = np.zeros(4 * n, dtype)
        bias[:n] = cfg.gate_bias
        P["bias"] = bias
        layers.append(P)
    W_out = init_uniform(rng.split(103), 2, n, 1.0 / math.sqrt(n), dtype)
    return {"layers": layers, "W_out": W_out, "b_out": np.zeros(2, dtype)}


def tensors(model):
    out = []
    for P in model["layers"]:
        out += [P[k] for k in ("sU", "sV", "sbg", "sbz", "U", "V", "bias")]
    return out + [model["W_out"], model["b_out"]]


def softmax_loss(logits, labels):
    b = logits.shape[0]
    loss, correct = 0.0, 0
    d = np.zeros_like(logits)
    for r in range(b):
        a, c = float(logits[r, 0]), float(logits[r, 1])
        mx = max(a, c)
        ea, ec = math.exp(a - mx), math.exp(c - mx)
        z = ea + ec
        y = int(labels[r])
        loss -= math.log((ec if y == 1 else ea) / z)
        correct += int((1 if c > a else 0) == y)
        d[r, 0] = (ea / z - (1.0 if y == 0 else 0.0)) / b
        d[r, 1] = (ec / z - (1.0 if y == 1 else 0.0)) / b
    return loss / b, correct / b, d


class Trainer:
    def __init__(self, cfg, rng, dtype=np.float64, oracle=None):
        self.cfg, self.dtype = cfg, dtype
        self.orc = oracle or Oracle()
        self.model = build_model(cfg, rng, dtype)
        self.m = [np.zeros(t.size) for t in tensors(self.model)]
        self.v = [np.zeros(t.size) for t in tensors(self.model)]
        self.step = 0

    def forward(self, x):
        z = np.zeros((x.shape[1], self.cfg.hidden), self.dtype)
        L1, L2 = self.model["layers"]
        h1, c1 = self.orc.gilr_lstm_forward(L1, x, z, z)
        h2, c2 = self.orc.gilr_lstm_forward(L2, h1, z, z)
        logits = h2[-1] @ self.model["W_out"].T + self.model["b_out"]
        return h1, c1, h2, c2, logits.astype(self.dtype)

    def train_step(self, x, labels):
        cfg, orc, M = self.cfg, self.orc, self.model
        h1, c1, h2, c2, logits = self.forward(x)
        loss, acc, dl = softmax_loss(logits, labels)
        if not math.isfinite(loss):
            return loss, acc
        dl = dl.astype(self.dtype)
        z = np.zeros((x.shape[1], cfg.hidden), self.dtype)
        dW_out = dl.T @ h2[-1]
        db_out = dl.sum(0)
        d_h2 = np.zeros_like(h2)
        d_h2[-1] = dl @ M["W_out"]
        g2, d_h1, _, _ = orc.gilr_lstm_backward(M["layers"][1], h1, z, z, c2, d_h2)
        g1, _, _, _ = orc.gilr_lstm_backward(M["layers"][0], x, z, z, c1, d_h1)
        grads = []
        for g in (g1, g2):
            grads += [g[k] for k in ("sU", "sV", "sbg", "sbz", "U", "V", "bias")]
        grads += [dW_out.astype(self.dtype), db_out.astype(self.dtype)]
        clip_global_norm(grads, cfg.clip_norm)
        self.adam(grads)
        return loss, acc

    def adam(self, grads, beta1=0.9, beta2=0.999, eps=1e-8):
        self.step += 1
        bc1, bc2 = 1.0 - beta1 ** self.step, 1.0 - beta2 ** self.step
        for i, (p, g) in enumerate(zip(tensors(self.model), grads)):
            gj = g.astype(np.float64).ravel()
            self.m[i] = beta1 * self.m[i] + (1.0 - beta1) * gj
            self.v[i] = beta2 * self.v[i] + (1.0 - beta2) * gj * gj
            upd = p.astype(np.float64).ravel() - self.cfg.learning_rate * (self.m[i] / bc1) / (
                np.sqrt(self.v[i] / bc2) + eps)
            p[...] = upd.reshape(p.shape).astype(p.dtype)


def clip_global_norm(grads, max_norm):
    norm = math.sqrt(sum(float(np.sum(g.astype(np.float64) ** 2)) for g in grads))
    if norm > max_norm and norm > 0:
        s = max_norm / norm
        for g in grads:
            g[...] = (g.astype(np.float64) * s).astype(g.dtype)
    return norm


@dataclass
class RunReport:
    converged: bool = False
    diverged: bool = False
    iterations: int = 0
    trace: list = field(default_factory=list)
    diagnostic: str = ""


def run_loop(cfg, step):
    rep, streak = RunReport(), 0
    for it in range(1, cfg.max_iters + 1):
        loss, acc = step(it)
        rep.trace.append((it, loss, acc))
        rep.iterations = it
        if not math.isfinite(loss):
            rep.diverged = True
            rep.diagnostic = f"non-finite loss at iteration {it}; run aborted"
            return rep
        streak = streak + 1 if acc == 1.0 else 0
        if streak >= cfg.window:
            rep.converged = True
            return rep
    rep.diagnostic = "maximum iterations reached without convergence"
    return rep


def run_experiment(cfg, dtype=np.float64, oracle=None):
    root = Rng(cfg.seed)
    trainer = Trainer(cfg, root.split(1), dtype, oracle)
    data = root.split(2)

    def step(_):
        x, y = generate_batch(data, cfg.seq_len, cfg.batch, cfg.input_dim, dtype)
        return trainer.train_step(x, y)
    return run_loop(cfg, step), trainer
