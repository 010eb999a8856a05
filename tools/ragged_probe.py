"""LtHash over variable-length samples: arrival order vs length-sorted order (warp lanes then run the same
number of BLAKE2b compressions). hellaswag-shaped token samples, 2 M of them."""
import json, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import dataset as dsm, device as dev

n, n_src = 2_000_000, 16
rng = np.random.default_rng(2)
lens = (np.clip(np.rint(rng.lognormal(np.log(90.0), 0.4, n)), 16, 256).astype(np.int64) * 4).astype(np.uint64)
offs = np.zeros(n, dtype=np.uint64); np.cumsum(lens[:-1], out=offs[1:])
shard = torch.randint(0, 256, (int(lens.sum()),), dtype=torch.uint8, device="cuda")
ids = np.arange(n, dtype=np.uint64); src = rng.integers(0, n_src, size=n)
ds = dsm.DeviceDataset(shard, torch.from_numpy(offs.view(np.int64)).cuda(), torch.from_numpy(lens.view(np.int64)).cuda(),
                       torch.from_numpy(ids.view(np.int64)).cuda(), torch.from_numpy(src.astype(np.int32)).cuda(), list(range(n_src)))

def timed(d):
    acc = dev.LatticeAccumulator(n_src)
    for _ in range(2):
        acc.zero_(); d.accumulate(acc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        acc.zero_(); d.accumulate(acc)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 5, acc.digests()[0]

t_plain, dig_plain = timed(ds)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
order = torch.argsort(ds.lengths)
sorted_ds = dsm.DeviceDataset(shard, ds.offsets[order], ds.lengths[order], ds.ids[order], ds.slots[order], list(range(n_src)))
e1.record(); torch.cuda.synchronize()
t_sort = e0.elapsed_time(e1)
t_sorted, dig_sorted = timed(sorted_ds)
print(json.dumps({"samples": n, "bytes": int(lens.sum()), "arrival_order_ms": round(t_plain, 3), "sorted_ms": round(t_sorted, 3),
                  "sort_cost_ms": round(t_sort, 3), "same_digest": dig_plain == dig_sorted,
                  "msamples_per_s": [round(n / t_plain / 1e3, 1), round(n / t_sorted / 1e3, 1)]}))
