"""Per-rank GPU time of the sharded GPT2-XL hash for world = 1, 2, 4, 8, measured on ONE GPU.

Each rank's work (leaf range + shard reduce, then the top reduce over all shard roots) is timed with
CUDA events for the slowest rank of every world size; the all-gather itself (a few KB over NVLink, one
NCCL call) cannot run here and is not included. This is a projection aid for DESIGN.md, not a bench line.
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import device as dev, distributed as dd, shapes  # noqa: E402


def timed(fn, reps=10):
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


sd = shapes.synthetic_state_dict("gpt2-xl", torch.device("cuda"))
plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], 8192)
backend = dd.CudaBackend(plan, "sha256")
out = {}
for world in (1, 2, 4, 8):
    sp = dd.plan_shards(plan.leaf_count, world)
    roots = torch.zeros(sp.n_shards * 32, dtype=torch.uint8, device="cuda")
    worst = 0.0
    for rank in range(world):
        a, b = sp.leaf_range(rank)

        def step():
            backend.shard_roots_padded(a, b, sp.levels, sp.shard_count(0))
            backend.root_of(roots, sp.n_shards)

        worst = max(worst, timed(step))
    out[f"world{world}"] = {"slowest_rank_ms": round(worst, 4), "shards_per_rank": sp.shard_count(0),
                            "projected_gbs": round(plan.total_bytes / worst / 1e6, 1)}
base = out["world1"]["slowest_rank_ms"]
for k, v in out.items():
    v["projected_speedup"] = round(base / v["slowest_rank_ms"], 2)
print(json.dumps(out))
