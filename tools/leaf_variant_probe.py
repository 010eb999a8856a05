"""Times snt_merkle_leaves (SHA-256) for the library named by SNT_LIB_PATH on the GPT2-XL and GPT-2 layouts."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import device as dev, shapes  # noqa: E402

out = {"lib": os.path.basename(os.environ.get("SNT_LIB_PATH", "default"))}
for arch in ("gpt2-xl", "gpt2"):
    sd = shapes.synthetic_state_dict(arch, torch.device("cuda"))
    plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], 8192)
    h = dev.MerkleModelHasher(plan, "sha256")
    for _ in range(3):
        h.run_leaves_only()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            h.run_leaves_only()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 10)
    out[arch] = {"leaf_ms": round(best, 4), "gbs": round(plan.total_bytes / best / 1e6, 1)}
    del sd, plan, h
print(json.dumps(out))
