"""Step-by-step wall clock of one pageable_to_device call (64 MB and 652 MB): acquire, copy_many per slot, issue."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import device as dev  # noqa: E402

d = torch.device("cuda")
for mb in (64, 652):
    src = np.random.default_rng(0).integers(0, 256, size=mb << 20, dtype=np.uint8)
    dst = torch.empty(src.size, dtype=torch.uint8, device=d)
    dev.pageable_to_device(src, dst)
    dev.pageable_to_device(src, dst)
    ring = dev.StagingRing.get(dev.staging_threads(1))
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    log = []
    t00 = time.perf_counter()
    base = src.ctypes.data
    for off in range(0, src.size, dev.STAGE_SLOT_BYTES):
        n = min(dev.STAGE_SLOT_BYTES, src.size - off)
        t0 = time.perf_counter()
        slot = ring.acquire()
        t1 = time.perf_counter()
        dev._hostpack.copy_many([ring.bufs[slot].data_ptr(), base + off, n], -1, ring.threads)
        t2 = time.perf_counter()
        dst[off:off + n].copy_(ring.bufs[slot][:n], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        ring.events[slot] = ev
        t3 = time.perf_counter()
        log.append((round((t1 - t0) * 1e3, 3), round((t2 - t1) * 1e3, 3), round((t3 - t2) * 1e3, 3)))
    t4 = time.perf_counter()
    stream.synchronize()
    t5 = time.perf_counter()
    print(json.dumps({"mb": mb, "total_ms": round((t5 - t00) * 1e3, 2), "final_sync_ms": round((t5 - t4) * 1e3, 2),
                      "acquire_copy_issue_ms_per_slot": log[:24]}))
