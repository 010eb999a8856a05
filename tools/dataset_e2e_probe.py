"""Per-call wall clock of the dataset end-to-end step bench.py times (rows + shard from pinned host memory -> HBM, one
launch, digests back): distribution over 30 calls for the CIFAR-shaped set and the hellaswag-shaped pool, and a
cProfile of ten calls (stderr)."""
import cProfile
import io
import json
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2510_00554_b200 import dataset as dsm, device as dev  # noqa: E402

out = {}
for name, make in (("cifar", bench.cifar_shaped), ("pool", bench.hellaswag_shaped)):
    shard, offs, lens, ids, src, n_src = make(np)
    shard_h = torch.from_numpy(shard).pin_memory()

    def step():
        d = dsm.DeviceDataset.from_host(shard_h, offs, lens, ids, src, list(range(n_src)))
        acc = dev.LatticeAccumulator(n_src)
        d.accumulate(acc)
        return acc.digests()

    for _ in range(3):
        step()
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        step()
        ts.append((time.perf_counter() - t0) * 1e3)
    ts_sorted = sorted(ts)
    out[name] = {"min_ms": round(ts_sorted[0], 3), "median_ms": round(ts_sorted[15], 3), "max_ms": round(ts_sorted[-1], 3),
                 "first10": [round(t, 2) for t in ts[:10]], "link_floor_ms": round((shard.nbytes + 28 * len(ids)) / 55.6e6, 3)}
    prof = cProfile.Profile()
    prof.enable()
    for _ in range(10):
        step()
    prof.disable()
    s = io.StringIO()
    pstats.Stats(prof, stream=s).sort_stats("tottime").print_stats(12)
    print(name, s.getvalue()[:3500], file=sys.stderr)
print(json.dumps(out))
