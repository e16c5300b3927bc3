import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_1709_04057_b200 import training as TR
T, gb, lr, iters = int(sys.argv[1]), float(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
cfg = TR.TrainConfig(seq_len=T, hidden=64, input_dim=128, batch=32, learning_rate=lr, gate_bias=gb, max_iters=iters)
rep = TR.run_experiment(cfg)
for r in rep.trace[:10]: print(r.iteration, r.loss, r.accuracy)
print(rep.converged, rep.diverged, rep.iterations, rep.diagnostic)
