"""Where do the last few percent of the SHA-256 leaf kernel go? Times snt_merkle_leaves on
(a) one contiguous tensor of 799,954 full leaves, (b) the same bytes cut into 581 equal tensors,
(c) the GPT2-XL state-dict layout (388 ragged tensors)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import device as dev, shapes  # noqa: E402


def time_leaves(tensors, alg="sha256", steps=10):
    plan = dev.ModelPlan(tensors, 8192)
    h = dev.MerkleModelHasher(plan, alg)
    for _ in range(3):
        h.run_leaves_only()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        h.run_leaves_only()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return {"ms": round(ms, 4), "gbs": round(plan.total_bytes / ms / 1e6, 1), "leaves": plan.leaf_count}


n = 799_954
big = torch.randint(0, 256, (n * 8192,), dtype=torch.uint8, device="cuda")
out = {"contiguous": time_leaves([big])}
per = (n // 581) * 8192
out["581_equal_tensors"] = time_leaves([big[i * per:(i + 1) * per] for i in range(581)])
del big
sd = shapes.synthetic_state_dict("gpt2-xl", torch.device("cuda"))
out["gpt2xl_layout"] = time_leaves([dev.as_device_bytes(t) for _, t in sd])
print(json.dumps(out))
