"""Ceiling of the pageable -> pinned staging copy on this box: N threads x np.copyto over 4 MB pieces of a 1 GB
pageable buffer into pinned memory (what device.pageable_arena does), without any GPU transfer."""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

size = 1 << 30
src = np.random.default_rng(0).integers(0, 256, size=size, dtype=np.uint8)
dst_t = torch.empty(size, dtype=torch.uint8, pin_memory=True)
dst = dst_t.numpy()
out = {"cpus": os.cpu_count()}
for piece_mb in (1, 4, 16):
    piece = piece_mb << 20
    for threads in (1, 2, 4, 8, 12, 16):
        pool = ThreadPoolExecutor(max_workers=threads)
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            tasks = [pool.submit(np.copyto, dst[o:o + piece], src[o:o + piece]) for o in range(0, size, piece)]
            for t in tasks:
                t.result()
            best = min(best, time.perf_counter() - t0)
        pool.shutdown()
        out[f"piece{piece_mb}MB_t{threads}_gbs"] = round(size / best / 1e9, 1)
# pinned -> device alone, for reference
d = torch.empty(size, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    d.copy_(dst_t, non_blocking=True)
torch.cuda.synchronize()
out["pinned_h2d_gbs"] = round(3 * size / (time.perf_counter() - t0) / 1e9, 1)
print(json.dumps(out))
