"""Developer probe: magnitudes through one training step at a long sequence
(where does a non-finite value first appear?).  Usage: train_probe.py T gate_bias"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch  # noqa: E402

from paper_1709_04057_b200 import training as TR  # noqa: E402

T, gb = int(sys.argv[1]), float(sys.argv[2])
cfg = TR.TrainConfig(seq_len=T, hidden=64, input_dim=128, batch=32, learning_rate=3e-3, gate_bias=gb, max_iters=3)
tr = TR.Trainer(cfg, TR.Rng(cfg.seed).split(1))
rng = TR.Rng(cfg.seed).split(2)
batch = TR.generate_batch(rng, T, cfg.batch, cfg.input_dim, device=torch.device("cuda", 0))
cache = TR.model_forward(tr.model, batch.inputs)
mx = lambda t: (t.abs().max().item(), bool(torch.isfinite(t).all()))  # noqa: E731
print("x", mx(batch.inputs))
for i, c in enumerate(cache.gl):
    print(f"layer {i}: htil", mx(c.htil), "gates", mx(c.gates), "c", mx(c.c))
print("h1", mx(cache.h1), "h2", mx(cache.h2))
loss, acc = TR.softmax_loss(tr.model, cache, batch.labels)
print("loss", loss, "logits", cache.logits[:4].tolist())
tr.model.grads.flat.zero_()
TR.model_backward(tr.model, batch.inputs, tr.cache if hasattr(tr, "cache") and tr.cache is cache else cache)
g = tr.model.grads
for i, v in enumerate(g.views):
    print("grad", i, tuple(v.shape), mx(v))
tr.opt.clip_and_update(tr.model, tr.clip_norm)
print("norm", tr.opt.norm.item(), "params", mx(tr.model.params.flat))
cache2 = TR.model_forward(tr.model, batch.inputs)
print("h2 after step", mx(cache2.h2))
