"""Host packing throughput of seed_stage_requests (n = 1024 Atari frames of 28 KB from
4096 per-actor host buffers into pinned staging + chunked H2D) vs worker threads, and
the plain pinned H2D of the packed bytes (usage: python scripts/probe_stager.py)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_06591_b200 import _lib as L  # noqa: E402

lib = L.load()
n, ob, NA = 1024, 84 * 84 * 4, 4096
frames = np.random.default_rng(0).integers(0, 256, size=(NA, ob), dtype=np.uint8)
ids = np.random.default_rng(1).choice(NA, n, replace=False).astype(np.int32)
ptrs = (C.c_void_p * n)(*[frames[i].ctypes.data for i in ids])
pin = torch.empty(n * ob, dtype=torch.uint8).pin_memory()
dev = torch.empty(n * ob, dtype=torch.uint8, device="cuda")
st = torch.cuda.Stream()
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
for threads in (1, 4, 8, 12, 16):
    h = C.c_void_p()
    lib.seed_stager_create(threads, C.byref(h))
    for chunk in (64, 128, 1024):
        ts = []
        for it in range(12):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = lib.seed_stage_requests(h, n, ptrs, C.c_size_t(ob), None, None, None,
                                        C.c_void_p(pin.data_ptr()), None, C.c_void_p(dev.data_ptr()),
                                        None, chunk, C.c_void_p(st.cuda_stream))
            st.synchronize()
            ts.append((time.perf_counter() - t) * 1e6)
            assert r == 0, r
        ts = sorted(ts[2:])
        print(f"threads {threads:2d} chunk {chunk:4d}: p50 {ts[len(ts)//2]:8.1f} us  min {ts[0]:8.1f} us"
              f"  ({n * ob / ts[len(ts)//2] / 1e3:.1f} GB/s)")
    lib.seed_stager_destroy(h)
t = time.perf_counter()
for _ in range(5):
    dev.copy_(pin, non_blocking=True)
torch.cuda.synchronize()
print("pinned H2D alone", (time.perf_counter() - t) / 5 * 1e6, "us")
