"""Latency of one LtHash launch over a small batch (rows of 3,072 bytes and ragged token arrays): the four-lanes-per-item
kernel (default schedule, n <= LT_QUAD_MAX_ITEMS) against one thread per item (SNT_SCHEDULE_GRID).
SNT_QUAD_FORCE=1 is not needed: sizes above the threshold show where the default switches over."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import _native, dataset as dsm, device as dev  # noqa: E402

lib = _native.load()


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best * 1e3


out = {}
rng = np.random.default_rng(0)
for shape in ("rows3072", "ragged"):
    for n in (1, 128, 2048, 4096, 8192, 12288, 16384, 24576, 32768):
        lens = np.full(n, 3072, dtype=np.uint64) if shape == "rows3072" else \
            (np.clip(np.rint(rng.lognormal(np.log(90.0), 0.4, n)), 16, 256).astype(np.uint64) * np.uint64(4))
        offs = np.zeros(n, dtype=np.uint64)
        np.cumsum(lens[:-1], out=offs[1:])
        shard = rng.integers(0, 256, size=int(lens.sum()) + 16, dtype=np.uint8)
        ds = dsm.DeviceDataset.from_host(shard, offs, lens, np.arange(n, dtype=np.uint64), rng.integers(0, 16, size=n), list(range(16)))
        acc = dev.LatticeAccumulator(16)
        res = {}
        ref = None
        for name, sched in (("default", _native.SCHEDULE_PERSISTENT), ("grid", _native.SCHEDULE_GRID), ("chains", _native.SCHEDULE_FUSED)):
            lib.snt_merkle_schedule(sched)
            acc.zero_()
            ds.accumulate(acc)
            got = acc.digests()
            assert ref is None or got == ref
            ref = got
            res[name + "_us"] = round(timed(lambda: ds.accumulate(acc)), 1)
        lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT)
        out[f"{shape}_n{n}"] = res
print(json.dumps(out))
