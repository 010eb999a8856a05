"""Times the three schedules of snt_merkle_schedule (persistent leaf kernel + reducer launches, the single fused
launch, round 1's leaf grid + reducer) for one architecture.

    python tools/fused_probe.py gpt2 sha256 [reps]
Prints one JSON line; SNT_LIB_PATH selects an alternative build of the library.
"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import _native, device as dev, shapes  # noqa: E402


def timed(fn, reps):
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


arch = sys.argv[1] if len(sys.argv) > 1 else "gpt2"
alg = sys.argv[2] if len(sys.argv) > 2 else "sha256"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
lib = _native.load()
sd = shapes.synthetic_state_dict(arch, torch.device("cuda"))
plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], 8192)
h = dev.MerkleModelHasher(plan, alg)
out = {"lib": os.path.basename(os.environ.get("SNT_LIB_PATH", "default")), "arch": arch, "alg": alg,
       "leaves": plan.leaf_count, "bytes": plan.total_bytes}
root = None
for name, schedule in (("persistent", _native.SCHEDULE_PERSISTENT), ("fused", _native.SCHEDULE_FUSED), ("grid", _native.SCHEDULE_GRID)):
    lib.snt_merkle_schedule(schedule)
    ms = timed(h.run, reps)
    leaf_ms = timed(h.run_leaves_only, reps)
    got = h.out_bytes().hex()
    assert root is None or got == root or os.environ.get("SNT_FUSED_NOTREE")
    root = root or got
    out[name] = {"ms": round(ms, 4), "gbs": round(plan.total_bytes / ms / 1e6, 1), "leaf_stage_ms": round(leaf_ms, 4)}
lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT)
out["root"] = root[:16]
print(json.dumps(out))
