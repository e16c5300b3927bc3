"""Host memcpy bandwidth on this machine: numpy copies (GIL released) split
over k threads, pageable->pinned (input staging) and pinned->fresh pageable
(output staging incl. first-touch page faults).  Sizing for the e2e path."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

N = 512 << 20  # bytes per copy
src = np.ones(N // 4, np.float32)
pin = torch.empty(N // 4, dtype=torch.float32, pin_memory=True).numpy()
try:
    print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
except OSError:
    pass
for k in (1, 2, 4, 8, 12, 16):
    ex = ThreadPoolExecutor(k)
    parts = np.array_split(np.arange(N // 4), k)

    def cp(dst, s):
        list(ex.map(lambda p: np.copyto(dst[p[0]:p[-1] + 1], s[p[0]:p[-1] + 1]), parts))
    cp(pin, src)
    t = time.perf_counter()
    for _ in range(3):
        cp(pin, src)
    a = 3 * N / (time.perf_counter() - t) / 1e9
    t = time.perf_counter()
    for _ in range(3):
        dst = np.empty(N // 4, np.float32)
        cp(dst, pin)
        del dst
    b = 3 * N / (time.perf_counter() - t) / 1e9
    print(f"threads {k:2d}: pageable->pinned {a:6.1f} GB/s   pinned->fresh pageable {b:6.1f} GB/s", flush=True)
