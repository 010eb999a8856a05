"""Times the BLAKE2b leaf stage and whole hash (library named by SNT_LIB_PATH) on BERT-large, VGG19 and GPT2-XL layouts,
and checks the root against the default library's.  python tools/b2b_variant_probe.py"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import device as dev, shapes  # noqa: E402


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


out = {"lib": os.path.basename(os.environ.get("SNT_LIB_PATH", "default"))}
for arch in sys.argv[1:] or ("bert-large", "vgg19", "gpt2-xl"):
    sd = shapes.synthetic_state_dict(arch, torch.device("cuda"))
    plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], 8192)
    h = dev.MerkleModelHasher(plan, "blake2b")
    out[arch] = {"leaf_ms": round(timed(h.run_leaves_only), 4), "hash_ms": round(timed(h.run), 4),
                 "root": h.out_bytes().hex()[:16]}
    out[arch]["gbs"] = round(plan.total_bytes / out[arch]["hash_ms"] / 1e6, 1)
    del sd, plan, h
print(json.dumps(out))
