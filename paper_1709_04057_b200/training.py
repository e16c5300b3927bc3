"""The reference's training experiment on the B200 (proj/include/linrec/training.hpp).

Synthetic long-dependency classification (Hochreiter & Schmidhuber problem
2b, the paper's Table 3): one-hot sequences whose first step is +-e1; a
two-layer GILR-LSTM with a linear readout on the final hidden state must
output that sign.  Same names and semantics as the reference:

    Rng                        rng.hpp:15-52 (counter-based splitmix64)
    TrainConfig                training.hpp:46-70
    generate_batch             :30-43   (GPU kernel, same draw stream)
    build_model / Model        :74-123  (same initialisation stream)
    model_forward / backward   :160-246 (GILR-LSTM layers on the GPU)
    softmax_loss               :193-222 (GPU kernel)
    clip_global_norm + Adam    :248-288 (one fused kernel over a flat buffer)
    Trainer.train_step         :297-333
    run_loop / run_experiment  :343-436

Everything numeric runs in liblinrec_cuda.so; the parameters, gradients and
Adam moments each live in ONE flat device buffer (fp32 / fp64) that the layer
calls address by offset.  Only the "gilr-lstm" arch is built (the serial
LSTM baseline is out of scope).

Data parallel over a process group (``run_experiment(cfg, group=...)``, one
rank per GPU): the global batch of cfg.batch rows is split across the ranks,
each rank drawing ITS rows of the same reference stream (row r uses draws
r*T+1 ...), the readout scales by the global batch, and one all-reduce of
the flat gradient buffer (plus the 2-double loss / accuracy) per step makes
every rank's clip + Adam identical -- the same trajectory as one GPU.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import capi
from . import layers as L

_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def _mix(z):
    """splitmix64 finalizer on a numpy uint64 array (wrapping arithmetic)."""
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


class Rng:
    """rng.hpp:15-52: draw k is splitmix64(seed + k * golden), k = 1, 2, ...;
    split() derives an independent child without advancing the parent."""

    def __init__(self, seed: int, counter: int = 0):
        self.seed = seed & _M64
        self.counter = counter

    def split(self, stream: int) -> "Rng":
        with np.errstate(over="ignore"):
            z = np.uint64(self.seed) ^ np.uint64((0xD1B54A32D192ED03 * (stream + 1)) & _M64)
            return Rng(int(_mix(np.array([z], dtype=np.uint64))[0]))

    def next_u64_array(self, count: int) -> np.ndarray:
        c = np.arange(self.counter + 1, self.counter + 1 + count, dtype=np.uint64)
        self.counter += count
        with np.errstate(over="ignore"):
            return _mix(np.uint64(self.seed) + c * np.uint64(_GOLDEN))

    def uniform_array(self, count: int, lo: float, hi: float) -> np.ndarray:
        """uniform(lo, hi) (rng.hpp:39-42), `count` draws in order, float64."""
        u = (self.next_u64_array(count) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        return lo + (hi - lo) * u

    def skip(self, count: int):
        self.counter += count


@dataclass
class TrainConfig:
    """training.hpp:46-70."""
    arch: str = "gilr-lstm"
    seq_len: int = 1024
    input_dim: int = 128
    hidden: int = 64
    layers: int = 2
    batch: int = 32
    learning_rate: float = 1e-3
    optimizer: str = "adam"
    max_iters: int = 5000
    seed: int = 0
    window: int = 5
    gate_bias: float = 1.0
    clip_norm: float = 1.0
    time_data_gen: bool = True
    precision: str = "fp32"  # GEMM precision of the layers (B200 addition)

    def validate(self):
        if (self.seq_len < 1 or self.input_dim < 2 or self.hidden < 1 or self.batch < 1 or self.max_iters < 1
                or self.window < 1 or self.layers != 2):
            raise RuntimeError("TrainConfig: counts out of range")
        if not self.learning_rate > 0:
            raise RuntimeError("TrainConfig: learning rate must be > 0")
        if self.arch not in ("gilr-lstm", "lstm-serial"):
            raise RuntimeError(f'TrainConfig: unknown arch "{self.arch}"')
        if self.arch != "gilr-lstm":
            raise NotImplementedError("only arch gilr-lstm runs on the B200 (the serial LSTM baseline is not built)")


def _init_uniform(rng: Rng, rows: int, cols: int, scale: float) -> np.ndarray:
    """init_uniform (rng.hpp:54-61): row-major draws, double -> float."""
    return rng.uniform_array(rows * cols, -scale, scale).astype(np.float32).reshape(rows, cols)


class FlatBuffer:
    """One device buffer carved into tensor views, each 16-byte aligned."""

    def __init__(self, shapes, dtype, device):
        self.offsets, n = [], 0
        for sh in shapes:
            self.offsets.append(n)
            n += (int(np.prod(sh)) + 3) // 4 * 4
        self.flat = torch.zeros(n, dtype=dtype, device=device)
        self.views = [self.flat.narrow(0, o, int(np.prod(sh))).view(*sh) for o, sh in zip(self.offsets, shapes)]


class Model:
    """Model (training.hpp:74-108) + ModelGrads (:125-147), flat storage."""

    def __init__(self, cfg: TrainConfig, rng: Rng, device="cuda"):
        cfg.validate()
        p_dim, n = cfg.input_dim, cfg.hidden
        self.cfg, self.n, self.device = cfg, n, torch.device(device)
        shapes = []
        for m in (p_dim, n):
            shapes += [(n, m), (n, m), (n,), (n,), (4 * n, n), (4 * n, m), (4 * n,)]
        shapes += [(2, n), (2,)]
        self.params = FlatBuffer(shapes, torch.float32, self.device)
        self.grads = FlatBuffer(shapes, torch.float32, self.device)
        host = []
        r1, r2, r3 = rng.split(101), rng.split(102), rng.split(103)
        for r, m in ((r1, p_dim), (r2, n)):
            # gilr_lstm_init (layers.hpp:165-176) / gilr_init (:42-55)
            sub = r.split(1)
            s = 1.0 / math.sqrt(m)
            sU, sV = _init_uniform(sub, n, m, s), _init_uniform(sub, n, m, s)
            sbg, sbz = np.full(n, cfg.gate_bias, np.float32), np.zeros(n, np.float32)
            U = _init_uniform(r, 4 * n, n, 1.0 / math.sqrt(n))
            V = _init_uniform(r, 4 * n, m, 1.0 / math.sqrt(m))
            bias = np.zeros(4 * n, np.float32)
            bias[:n] = cfg.gate_bias
            host += [sU, sV, sbg, sbz, U, V, bias]
        host += [_init_uniform(r3, 2, n, 1.0 / math.sqrt(n)), np.zeros(2, np.float32)]
        for v, a in zip(self.params.views, host):
            v.copy_(torch.from_numpy(a))
        self.layers = [self._lstm_params(self.params.views[7 * i: 7 * i + 7]) for i in range(2)]
        self.layer_grads = [self._lstm_grads(self.grads.views[7 * i: 7 * i + 7]) for i in range(2)]
        self.W_out, self.b_out = self.params.views[14], self.params.views[15]
        self.dW_out, self.db_out = self.grads.views[14], self.grads.views[15]

    @staticmethod
    def _lstm_params(v):
        return L.GilrLstmParams(L.GilrParams(v[0], v[1], v[2], v[3]), v[4], v[5], v[6])

    @staticmethod
    def _lstm_grads(v):
        return L.GilrLstmGrads(L.GilrGrads(v[0], v[1], v[2], v[3]), v[4], v[5], v[6])

    def tensors(self):
        return self.params.views

    def parameter_count(self):
        return sum(v.numel() for v in self.params.views)


def build_model(cfg: TrainConfig, rng: Rng, device="cuda") -> Model:
    return Model(cfg, rng, device)


def _lib():
    lib = capi.lib
    if not getattr(lib, "_train_bound", False):
        vp, i64 = C.c_void_p, C.c_int64
        lib.linrec_synthetic_batch_f32.argtypes = [C.c_uint64, C.c_uint64, i64, i64, i64, vp, vp, vp]
        lib.linrec_readout_loss_f32.argtypes = [vp] * 7 + [i64, i64, i64, vp]
        lib.linrec_readout_backward_f32.argtypes = [vp] * 6 + [i64, i64, vp]
        lib.linrec_adam_scratch_bytes.restype = C.c_size_t
        lib.linrec_adam_scratch_bytes.argtypes = []
        lib.linrec_clip_adam_f32.argtypes = ([vp] * 4 + [i64] + [C.c_double] * 4 + [i64, C.c_double, vp, vp,
                                                                                     C.c_size_t, vp])
        lib._train_bound = True
    return lib


def _stream(dev):
    return torch.cuda.current_stream(dev).cuda_stream


@dataclass
class SyntheticBatch:
    inputs: torch.Tensor  # [T, b, p] one-hot, device
    labels: torch.Tensor  # [b] int32, device


def generate_batch(rng: Rng, T: int, b: int, p: int, device="cuda", out: SyntheticBatch | None = None,
                   rows: tuple | None = None):
    """training.hpp:30-43 on the GPU: the same draws from the same stream.
    rows = (r0, r1): only rows [r0, r1) of the b-row batch (data-parallel
    shard); the stream still advances by the whole batch."""
    dev = torch.device(device)
    r0, r1 = rows if rows is not None else (0, b)
    bl = r1 - r0
    if out is None or tuple(out.inputs.shape) != (T, bl, p):
        out = SyntheticBatch(torch.empty(T, bl, p, dtype=torch.float32, device=dev),
                             torch.empty(bl, dtype=torch.int32, device=dev))
    capi.check(_lib().linrec_synthetic_batch_f32(rng.seed, rng.counter + r0 * T, T, bl, p, out.inputs.data_ptr(),
                                                 out.labels.data_ptr(), _stream(dev)))
    if p >= 2 and T >= 1:
        rng.skip(b * T)
    return out


class ModelCache:
    """ModelCache (:149-158): per-layer caches, h1, h2, logits, d_logits."""

    def __init__(self):
        self.gl = [L.GilrLstmCache(), L.GilrLstmCache()]
        self.h1 = self.h2 = self.logits = self.d_logits = None
        self.loss_acc = None


def model_forward(m: Model, x, mode="parallel", cache: ModelCache | None = None):
    """model_forward (:160-190): both layers (zero initial states) + readout.
    Returns the cache; logits [b, 2] in cache.logits."""
    cache = cache or ModelCache()
    T, b, _ = x.shape
    prec = m.cfg.precision
    cache.h1 = L.gilr_lstm_forward(m.layers[0], x, None, None, mode=mode, precision=prec, cache=cache.gl[0])
    cache.h2 = L.gilr_lstm_forward(m.layers[1], cache.h1, None, None, mode=mode, precision=prec, cache=cache.gl[1])
    return cache


def softmax_loss(m: Model, cache: ModelCache, labels, b_total=None, group=None):
    """Readout on the last step + softmax_loss (:182-222) on the GPU; leaves
    d_logits in the cache.  Returns (loss, accuracy) as Python floats (over
    the global batch when data parallel: b_total rows, summed over `group`)."""
    T, b, n = cache.h2.shape
    dev = cache.h2.device
    if cache.logits is None or cache.logits.shape[0] != b:
        cache.logits = torch.empty(b, 2, dtype=torch.float32, device=dev)
        cache.d_logits = torch.empty(b, 2, dtype=torch.float32, device=dev)
        cache.loss_acc = torch.empty(2, dtype=torch.float64, device=dev)
    capi.check(_lib().linrec_readout_loss_f32(cache.h2[T - 1].data_ptr(), m.W_out.data_ptr(), m.b_out.data_ptr(),
                                              labels.data_ptr(), cache.logits.data_ptr(), cache.d_logits.data_ptr(),
                                              cache.loss_acc.data_ptr(), b, n, b if b_total is None else b_total,
                                              _stream(dev)))
    if group is not None:
        _all_reduce(cache.loss_acc, group)
    la = cache.loss_acc.cpu()
    return float(la[0]), float(la[1])


def model_backward(m: Model, x, cache: ModelCache, mode="parallel"):
    """model_backward (:224-246): readout, then layer 2, then layer 1;
    gradients accumulate into m.grads."""
    T, b, n = cache.h2.shape
    dev = cache.h2.device
    if getattr(cache, "d_h2", None) is None or tuple(cache.d_h2.shape) != (T, b, n):
        cache.d_h2 = torch.zeros(T, b, n, dtype=torch.float32, device=dev)  # zero except the last step
    capi.check(_lib().linrec_readout_backward_f32(cache.d_logits.data_ptr(), cache.h2[T - 1].data_ptr(),
                                                  m.W_out.data_ptr(), m.dW_out.data_ptr(), m.db_out.data_ptr(),
                                                  cache.d_h2[T - 1].data_ptr(), b, n, _stream(dev)))
    prec = m.cfg.precision
    d_h1, _, _ = L.gilr_lstm_backward(m.layers[1], cache.h1, None, None, cache.gl[1], cache.d_h2, m.layer_grads[1],
                                      mode=mode, precision=prec, want_initial=False)
    L.gilr_lstm_backward(m.layers[0], x, None, None, cache.gl[0], d_h1, m.layer_grads[0], mode=mode,
                         precision=prec, want_initial=False)


def _all_reduce(t, group):
    """Sum over the data-parallel group: NCCL on device buffers; gloo (CPU
    tests, ranks sharing one GPU) through a host copy."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(t, group=group)
    else:
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)


class Adam:
    """Adam (:248-273) with global-norm clipping (:275-288), fp64 moments,
    fused over the model's flat parameter buffer."""

    def __init__(self, model: Model, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps
        self.step = 0
        flat = model.params.flat
        self.m = torch.zeros(flat.numel(), dtype=torch.float64, device=flat.device)
        self.v = torch.zeros_like(self.m)
        self.scratch = torch.empty(_lib().linrec_adam_scratch_bytes() // 8 + 1, dtype=torch.float64,
                                   device=flat.device)
        self.norm = torch.zeros(1, dtype=torch.float64, device=flat.device)

    def clip_and_update(self, model: Model, clip_norm: float):
        self.step += 1
        p, g = model.params.flat, model.grads.flat
        capi.check(_lib().linrec_clip_adam_f32(p.data_ptr(), g.data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                                               p.numel(), self.lr, self.beta1, self.beta2, self.eps, self.step,
                                               clip_norm, self.norm.data_ptr(), self.scratch.data_ptr(),
                                               self.scratch.numel() * 8, _stream(p.device)))


class Trainer:
    """Trainer (:291-333); `group` makes it data parallel (see module doc)."""

    def __init__(self, cfg: TrainConfig, rng: Rng, device="cuda", group=None):
        self.cfg = cfg
        self.group = group
        self.model = build_model(cfg, rng, device)
        self.opt = Adam(self.model, lr=cfg.learning_rate)
        self.clip_norm = cfg.clip_norm
        self.cache = ModelCache()

    def train_step(self, batch: SyntheticBatch, mode="parallel"):
        m = self.model
        model_forward(m, batch.inputs, mode, self.cache)
        loss, acc = softmax_loss(m, self.cache, batch.labels, self.cfg.batch, self.group)
        if not math.isfinite(loss):
            return loss, acc  # caller handles divergence
        m.grads.flat.zero_()
        model_backward(m, batch.inputs, self.cache, mode)
        if self.group is not None:
            _all_reduce(m.grads.flat, self.group)  # the one exchange of the step
        self.opt.clip_and_update(m, self.clip_norm)
        return loss, acc


@dataclass
class TraceRow:
    iteration: int
    loss: float
    accuracy: float
    elapsed_seconds: float


@dataclass
class RunReport:
    converged: bool = False
    diverged: bool = False
    iterations: int = 0
    elapsed_seconds: float = 0.0
    trace: list = field(default_factory=list)
    diagnostic: str = ""


def run_loop(cfg: TrainConfig, step, clock=None) -> RunReport:
    """run_loop (:343-380): step(iter) -> (loss, acc) until `window`
    consecutive perfect rows, divergence or max_iters."""
    report = RunReport()
    streak = 0
    start = time.perf_counter()
    clock = clock or (lambda: time.perf_counter() - start)
    for it in range(1, cfg.max_iters + 1):
        loss, acc = step(it)
        elapsed = clock()
        report.trace.append(TraceRow(it, loss, acc, elapsed))
        report.iterations, report.elapsed_seconds = it, elapsed
        if not math.isfinite(loss):
            report.diverged = True
            report.diagnostic = f"non-finite loss at iteration {it}; run aborted"
            return report
        streak = streak + 1 if acc == 1.0 else 0
        if streak >= cfg.window:
            report.converged = True
            return report
    report.diagnostic = "maximum iterations reached without convergence"
    return report


def run_experiment(cfg: TrainConfig, mode="parallel", device="cuda", trainer_out: list | None = None,
                   group=None) -> RunReport:
    """run_experiment (:384-436): fresh batches every iteration from
    root.split(2), parameters from root.split(1).  With a process group the
    global batch is split across its ranks (data parallel)."""
    cfg.validate()
    rows = None
    if group is not None:
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        if world == 1:
            group = None
        else:
            if cfg.batch < world:
                raise RuntimeError("data parallel: batch must be >= the number of ranks")
            base, rem = divmod(cfg.batch, world)
            r0 = rank * base + min(rank, rem)
            rows = (r0, r0 + base + (1 if rank < rem else 0))
    root = Rng(cfg.seed)
    param_rng, data_rng = root.split(1), root.split(2)
    trainer = Trainer(cfg, param_rng, device, group)
    if trainer_out is not None:
        trainer_out.append(trainer)
    batch = None
    dev = torch.device(device)

    if cfg.time_data_gen:
        def step(_):
            nonlocal batch
            batch = generate_batch(data_rng, cfg.seq_len, cfg.batch, cfg.input_dim, dev, batch, rows)
            return trainer.train_step(batch, mode)
        return run_loop(cfg, step)

    timed = [0.0]

    def step_k(_):  # kernel-only accounting: data generation outside the stopwatch
        nonlocal batch
        batch = generate_batch(data_rng, cfg.seq_len, cfg.batch, cfg.input_dim, dev, batch, rows)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        r = trainer.train_step(batch, mode)
        torch.cuda.synchronize(dev)
        timed[0] += time.perf_counter() - t0
        return r
    return run_loop(cfg, step_k, lambda: timed[0])
