"""pageable_to_device alone (no hashing): one numpy array of 64 MB ... 2 GB through the pinned staging ring; GB/s by
size, with the C copy pool and (SNT_NO_COPY_POOL=1) the Python pool. Also the raw copy_many rate into pinned memory."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import device as dev  # noqa: E402

out = {"copy_pool": dev._copy_pool is not None}
d = torch.device("cuda")
for mb in (64, 256, 652, 2048):
    src = np.random.default_rng(0).integers(0, 256, size=mb << 20, dtype=np.uint8)
    dst = torch.empty(src.size, dtype=torch.uint8, device=d)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.pageable_to_device(src, dst)
        ts.append(time.perf_counter() - t0)
    out[f"{mb}MB"] = {"ms": round(min(ts) * 1e3, 2), "gbs": round(src.size / min(ts) / 1e9, 1)}
    if mb == 652 and dev._hostpack is not None:
        pin = torch.empty(src.size, dtype=torch.uint8, pin_memory=True)
        for thr in (4, 8, 12, 16):
            ts = []
            for _ in range(4):
                t0 = time.perf_counter()
                dev._hostpack.copy_many([pin.data_ptr(), src.ctypes.data, src.size], -1, thr)
                ts.append(time.perf_counter() - t0)
            out[f"copy_many_{thr}thr_gbs"] = round(src.size / min(ts) / 1e9, 1)
        t0 = time.perf_counter()
        dst.copy_(pin, non_blocking=True)
        torch.cuda.synchronize()
        out["pinned_h2d_652MB_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
        del pin
    del src, dst
print(json.dumps(out))
