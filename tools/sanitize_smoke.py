"""Small pass over every kernel path for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py

All three Merkle schedules (persistent chains + reducer, fused single launch, grid) on ragged / unaligned models
whose SMs get more chains than worker warps (so the parked-state FIFO runs), shard ranges with forced levels, and
the LtHash kernels (grid, forced chains, persistent lanes, four lanes per item). SANITIZE_ONLY=lthash skips the Merkle part. Results are checked against hashlib, so a silent corruption fails too.
"""
import hashlib
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import _native, device as dev  # noqa: E402

lib = _native.load()
H = {"sha256": hashlib.sha256, "blake2b": hashlib.blake2b, "sha3-256": hashlib.sha3_256}


def merkle_root(alg, leaves):
    dl = H[alg]().digest_size
    level = leaves
    while len(level) > 1:
        if len(level) % 2:
            level = level + [bytes(dl)]
        level = [H[alg](level[i] + level[i + 1]).digest() for i in range(0, len(level), 2)]
    return level[0]


rng = np.random.default_rng(1)
sms = torch.cuda.get_device_properties(0).multi_processor_count
bs = 64
n_leaves = sms * 32 * 9 + 77                      # ~9 chains per SM at 4-8 warps: time slicing on every SM
arena_h = rng.integers(0, 256, size=n_leaves * bs + 4096, dtype=np.uint8)
arena = torch.from_numpy(arena_h).cuda()
cuts = [0, 1000 * bs + 16, 1000 * bs + 16 + 7 * bs + 5, 1000 * bs + 16 + 7 * bs + 5 + 3, n_leaves * bs - 40]
cuts[2] += (-cuts[2]) % 16 + 1                    # third tensor at an odd address
views = [arena[a:b] for a, b in zip(cuts[:-1], cuts[1:])]
host = [arena_h[a:b].tobytes() for a, b in zip(cuts[:-1], cuts[1:])]
blocks = [t[o:o + bs] for t in host for o in range(0, len(t), bs)]
plan = dev.ModelPlan(views, bs)
assert plan.leaf_count == len(blocks)
for alg in (() if os.environ.get("SANITIZE_ONLY") == "lthash" else ("sha256", "blake2b", "sha3-256")):
    want_leaves = [H[alg](b).digest() for b in blocks]
    want_root = merkle_root(alg, want_leaves)
    for schedule in (_native.SCHEDULE_PERSISTENT, _native.SCHEDULE_FUSED, _native.SCHEDULE_GRID):
        lib.snt_merkle_schedule(schedule)
        h = dev.MerkleModelHasher(plan, alg)
        for _ in range(2):
            h.run()
        assert h.leaf_bytes() == b"".join(want_leaves), (alg, schedule)
        assert h.out_bytes() == want_root, (alg, schedule)
        k = 6
        first, last = 1 << k, min(plan.leaf_count, 5 << k)
        hs = dev.MerkleModelHasher(plan, alg, first, last, k)
        hs.run()
        dl = len(want_root)
        got = hs.out_bytes()
        for j in range((last - first) >> k):
            sub = want_leaves[first + (j << k):first + ((j + 1) << k)]
            assert got[j * dl:(j + 1) * dl] == merkle_root(alg, sub), (alg, schedule, "shard", j)
lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT)

n, n_src = sms * 32 * 5 + 9, 7
lens = rng.integers(0, 900, size=n).astype(np.uint64)
offs = np.zeros(n, dtype=np.uint64)
np.cumsum(lens[:-1] + 1, out=offs[1:])
shard_h = rng.integers(0, 256, size=int(offs[-1] + lens[-1]) + 16, dtype=np.uint8)
slots = rng.integers(0, n_src, size=n).astype(np.int32)
ids = np.arange(n, dtype=np.uint64) * 7
want = np.zeros((n_src, 32), dtype=np.uint64)
sb = shard_h.tobytes()
for i in range(n):
    d = hashlib.blake2b(int(ids[i]).to_bytes(8, "little") + sb[int(offs[i]):int(offs[i] + lens[i])]).digest()
    want[slots[i]] += np.frombuffer(d, dtype="<u2")
want = (want & 0xFFFF).astype("<u2").tobytes()
d_args = [torch.from_numpy(shard_h).cuda()] + [torch.from_numpy(a.view(np.int64)).cuda() for a in (offs, lens, ids)] + \
         [torch.from_numpy(slots).cuda()]
for schedule in (_native.SCHEDULE_FUSED, _native.SCHEDULE_GRID, _native.SCHEDULE_PERSISTENT):   # chains, grid, lanes
    lib.snt_merkle_schedule(schedule)
    acc = dev.LatticeAccumulator(n_src)
    acc.add_samples(*d_args)
    out, counts, status = acc.digests()
    assert out == want and status == 0 and sum(counts) == n, schedule
lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT)
# a small launch: the four-lanes-per-item kernel (the first 1,000 samples in two calls, then the rest through the lanes)
acc = dev.LatticeAccumulator(n_src)
for a, b in ((0, 700), (700, 1000), (1000, n)):
    acc.add_samples(d_args[0], *(t[a:b] for t in d_args[1:]))
out, counts, status = acc.digests()
assert out == want and status == 0 and sum(counts) == n, "quad + lanes"
print("sanitize smoke ok")
