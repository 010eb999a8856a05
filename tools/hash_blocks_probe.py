"""Host cost of the reference-shaped hash_blocks / merkle_root calls on host blocks: 128 MiB cut into 8 KiB
memoryview slices (what the reference's BlockTable hands to hash_blocks, merkle.py:93-114), digests checked
against hashlib; SNT_NO_HOSTPACK=1 times the pure-Python packing for comparison."""
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2510_00554_b200 as snt  # noqa: E402
from paper_2510_00554_b200 import device as _dev  # noqa: E402

if os.environ.get("SNT_NO_HOSTPACK"):
    _dev._hostpack = None
total, bs = 128 << 20, 8192
buf = np.random.default_rng(0).integers(0, 256, size=total, dtype=np.uint8).tobytes()
view = memoryview(buf)
blocks = [view[i:i + bs] for i in range(0, total, bs)]
alg = snt.CompressionAlg.SHA256
ts, tr = [], []
for _ in range(4):
    t0 = time.perf_counter()
    leaves = snt.hash_blocks(alg, blocks)
    t1 = time.perf_counter()
    root = snt.merkle_root(alg, leaves)
    t2 = time.perf_counter()
    ts.append(t1 - t0)
    tr.append(t2 - t1)
for i in (0, 1, len(blocks) - 1):
    assert bytes(leaves.data[32 * i:32 * i + 32]) == hashlib.sha256(blocks[i]).digest()
print(json.dumps({"hostpack": _dev._hostpack is not None, "blocks": len(blocks), "hash_blocks_ms": round(min(ts) * 1e3, 2),
                  "gbs": round(total / min(ts) / 1e9, 2), "merkle_root_ms": round(min(tr) * 1e3, 2), "root": root.hex()[:16]}))
