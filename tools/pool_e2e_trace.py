"""Why the hellaswag-shaped pool's end-to-end step is bimodal (0.44 ms for the first calls, 1.25 ms afterwards): CUDA
event times of the shard transfer, the rows transfer and the LtHash launch inside consecutive DeviceDataset.from_host
steps (fresh device and pinned allocations per step, as bench.py's e2e leg does), and the same with persistent buffers."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2510_00554_b200 import dataset as dsm, device as dev  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "cifar-first":
    c = bench.cifar_shaped(np)
    c_h = torch.from_numpy(c[0]).pin_memory()
    for _ in range(8):
        cd = dsm.DeviceDataset.from_host(c_h, c[1], c[2], c[3], c[4], list(range(c[5])))
        ca = dev.LatticeAccumulator(c[5])
        cd.accumulate(ca)
        ca.digests()
    del cd, ca
shard, offs, lens, ids, src, n_src = bench.hellaswag_shaped(np)
shard_h = torch.from_numpy(shard).pin_memory()
n = len(ids)
out = {}
for mode in ("fresh",):
    rows = []
    held = []
    for i in range(24):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        t0 = time.perf_counter()
        ev[0].record()
        shard_t = shard_h.to("cuda", non_blocking=True)
        ev[1].record()
        t1 = time.perf_counter()
        d = dsm.DeviceDataset.from_host(shard_t, offs, lens, ids, src, list(range(n_src)))
        ev[2].record()
        t2 = time.perf_counter()
        acc = dev.LatticeAccumulator(n_src)
        d.accumulate(acc)
        ev[3].record()
        res = acc.digests()
        t3 = time.perf_counter()
        rows.append([round((t3 - t0) * 1e3, 3), round(ev[0].elapsed_time(ev[1]), 3), round(ev[1].elapsed_time(ev[2]), 3),
                     round(ev[2].elapsed_time(ev[3]), 3), round((t1 - t0) * 1e3, 3), round((t2 - t1) * 1e3, 3), round((t3 - t2) * 1e3, 3)])
        if mode != "fresh":
            held.append((shard_t, d, acc))
    out[mode] = {"columns": "wall, gpu shard h2d, gpu rows h2d, gpu kernel, host .to(), host from_host, host accumulate+digests",
                 "steps": rows}
print(json.dumps(out))
