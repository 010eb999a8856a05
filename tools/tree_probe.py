"""Times the tree stage alone (snt_merkle_root over n digests) and the leaf stage for SNT_LIB_PATH."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import device as dev, shapes  # noqa: E402


def timed(fn, reps=20):
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
    return round(best * 1000, 1)


out = {"lib": os.path.basename(os.environ.get("SNT_LIB_PATH", "default"))}
for alg in ("sha256", "blake2b", "sha3-256"):
    for n in (799_954, 79_672):
        nodes = torch.randint(0, 256, (n * dev.DIGEST_LEN[alg],), dtype=torch.uint8, device="cuda")
        out[f"tree_us_{alg}_{n}"] = timed(lambda: dev.merkle_root_device(alg, nodes, n))
sd = shapes.synthetic_state_dict("gpt2-xl", torch.device("cuda"))
plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], 8192)
h = dev.MerkleModelHasher(plan, "sha256")
out["leaf_us_gpt2xl"] = timed(h.run_leaves_only, 10)
out["step_us_gpt2xl"] = timed(h.run, 10)
print(json.dumps(out))
