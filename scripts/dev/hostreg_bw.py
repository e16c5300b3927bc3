"""Dev probe: cudaHostRegister / Unregister throughput on pageable numpy memory (the alternative to staging
pageable inputs through pinned bounce buffers)."""
import ctypes
import time
import numpy as np
cudart = ctypes.CDLL("libcudart.so")
for mb in (64, 256, 2048):
    a = np.ones(mb << 18, np.float32)  # mb MiB
    t = time.perf_counter()
    rc = cudart.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(a.nbytes), 0)
    t1 = time.perf_counter()
    rc2 = cudart.cudaHostUnregister(ctypes.c_void_p(a.ctypes.data))
    t2 = time.perf_counter()
    print(f"{mb} MiB: register {a.nbytes / (t1 - t) / 1e9:.1f} GB/s (rc {rc}), unregister {a.nbytes / (t2 - t1) / 1e9:.1f} GB/s (rc {rc2})")
