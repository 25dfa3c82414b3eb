"""Probe: pageable -> device staging rate of device.h2d_into for several ring
chunk sizes / depths / copy-thread counts (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_03209_b200 import device as D  # noqa: E402

dev = torch.device("cuda", 0)
X = np.random.default_rng(0).standard_normal((1_000_000, 256))
out = torch.empty(X.shape, dtype=torch.float64, device=dev)
Xp = torch.from_numpy(X).pin_memory()
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); out.copy_(Xp, non_blocking=True); torch.cuda.synchronize()
print(f"pinned: {X.nbytes / (time.perf_counter() - t) / 1e9:.1f} GB/s", flush=True)
for chunk_mb in (32, 64, 128):
    for depth in (3, 4, 6):
        for threads in (8, 16, 32):
            D.STAGE_CHUNK = chunk_mb << 20
            D.STAGE_DEPTH = depth
            D._RINGS.clear()
            if D._POOL is not None:
                D._POOL.shutdown()
            D._POOL = None
            os.environ["B200MAP_STAGE_THREADS"] = str(threads)
            best = 1e9
            for _ in range(3):
                torch.cuda.synchronize(); t = time.perf_counter()
                D.h2d_into(out, X)
                torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
            print(f"chunk {chunk_mb} MB depth {depth} threads {threads}: {X.nbytes / best / 1e9:.1f} GB/s", flush=True)
