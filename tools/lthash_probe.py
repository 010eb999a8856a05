"""Times the LtHash launch on the CIFAR10-shaped (50,000 x 3,072 B) and hellaswag-shaped (40,000 ragged) sets under both
schedules (persistent chains / plain grid).  python tools/lthash_probe.py [reps]"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import _native, dataset as dsm, device as dev  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
lib = _native.load()


def timed(fn):
    for _ in range(3):
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
    return best


def cifar():
    n, ln, n_src = 50_000, 3072, 16
    data = np.random.default_rng(0).integers(0, 256, size=n * ln, dtype=np.uint8)
    r1 = np.random.default_rng(1)
    src = r1.choice(n_src, size=n, p=r1.dirichlet(np.ones(n_src)))
    return data, np.arange(n, dtype=np.uint64) * ln, np.full(n, ln, dtype=np.uint64), np.arange(n, dtype=np.uint64), src, n_src


def hellaswag():
    n, n_cur = 40_000, 16
    lens_tok = np.clip(np.rint(np.random.default_rng(2).lognormal(np.log(90.0), 0.4, n)), 16, 256).astype(np.int64)
    lengths = (lens_tok * 4).astype(np.uint64)
    offsets = np.zeros(n, dtype=np.uint64)
    np.cumsum(lengths[:-1], out=offsets[1:])
    tokens = np.random.default_rng(2).integers(0, 50257, size=int(lens_tok.sum()), dtype=np.int32)
    r3 = np.random.default_rng(3)
    return tokens.view(np.uint8), offsets, lengths, np.arange(n, dtype=np.uint64), r3.choice(n_cur, size=n, p=r3.dirichlet(np.ones(n_cur))), n_cur


out = {"lib": os.path.basename(os.environ.get("SNT_LIB_PATH", "default"))}
for name, make in (("cifar10_shaped", cifar), ("hellaswag_shaped", hellaswag)):
    shard, offs, lens, ids, src, n_src = make()
    ds = dsm.DeviceDataset.from_host(shard, offs, lens, ids, src, list(range(n_src)))
    acc = dev.LatticeAccumulator(n_src)
    ref = None
    for sname, sched in (("chains", _native.SCHEDULE_FUSED), ("grid", _native.SCHEDULE_GRID)):
        lib.snt_merkle_schedule(sched)
        ms = timed(lambda: ds.accumulate(acc))
        acc.zero_()
        ds.accumulate(acc)
        got = acc.digests()
        assert ref is None or got == ref
        ref = got
        out[f"{name}_{sname}_us"] = round(ms * 1e3, 1)
    lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT)
print(json.dumps(out))
