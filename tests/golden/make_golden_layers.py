"""Generate the layer fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run here (where /root/reference exists) after ``make -C oracle ref``:

    python tests/golden/make_golden_layers.py

The outputs come from the reference's own per-step layer oracles
(proj/tests/support/layer_oracles.hpp: gilr_lstm :52-82, qrnn :84-114),
compiled unmodified into oracle/_ref/liblinrec_ref.so.  They pin the forward
pass of the C restatement (oracle/linrec_layers.c) on the GPU box, where
/root/reference does not exist:

  gilr_lstm.npz   T=17 b=3 m=5 n=6, random htil0 / c0
  qrnn.npz        T=13 b=2 m=5 n=4 for windows k = 1, 2, 3 (k=3 > the first
                  rows' history: the zero-padded causal window)
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.oracle import RefLib, gilr_lstm_params, qrnn_params  # noqa: E402


def main():
    ref = RefLib()
    rng = np.random.default_rng(20171)
    T, b, m, n = 17, 3, 5, 6
    P = gilr_lstm_params(rng, m, n)
    x = rng.uniform(-1, 1, (T, b, m))
    htil0 = rng.uniform(-1, 1, (b, n))
    c0 = rng.uniform(-1, 1, (b, n))
    h = ref.gilr_lstm_oracle(P, x, htil0, c0)
    np.savez(os.path.join(HERE, "gilr_lstm.npz"), x=x, htil0=htil0, c0=c0, h_ref=h,
             **{f"P_{k}": v for k, v in P.items()})

    out = {}
    T, b, m, n = 13, 2, 5, 4
    for k in (1, 2, 3):
        P = qrnn_params(rng, m, n, k)
        x = rng.uniform(-1, 1, (T, b, m))
        c0 = rng.uniform(-1, 1, (b, n))
        out[f"k{k}_W"] = P["W"]
        out[f"k{k}_bias"] = P["bias"]
        out[f"k{k}_x"] = x
        out[f"k{k}_c0"] = c0
        out[f"k{k}_h_ref"] = ref.qrnn_oracle(P, x, c0)
    np.savez(os.path.join(HERE, "qrnn.npz"), **out)
    print("wrote gilr_lstm.npz, qrnn.npz")


if __name__ == "__main__":
    main()
