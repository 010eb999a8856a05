"""hash_model on pinned host tensors (GPT2-XL, GPT-2 small) by size of the copy/hash groups (model.STAGE_CHUNK_BYTES)."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2510_00554_b200 as pkg  # noqa: E402
from paper_2510_00554_b200 import model as mm, shapes  # noqa: E402

out = {}
for arch in sys.argv[1:] or ("gpt2", "gpt2-xl"):
    sd = shapes.synthetic_state_dict(arch, torch.device("cuda"))
    seen, entries = {}, []
    for name, t in sd:
        if t.data_ptr() not in seen:
            h = torch.empty(t.numel() * 4, dtype=torch.uint8).pin_memory()
            h.copy_(t.reshape(-1).view(torch.uint8))
            seen[t.data_ptr()] = h
        entries.append((name, seen[t.data_ptr()]))
    del sd
    torch.cuda.empty_cache()
    model = pkg.TensorMap(entries)
    cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.SHA256)
    out[arch] = {}
    for mb in (256, 128, 64, 32, 16):
        mm.STAGE_CHUNK_BYTES = mb << 20
        for _ in range(2):
            pkg.hash_model(cfg, model)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            pkg.hash_model(cfg, model)
            ts.append(time.perf_counter() - t0)
        out[arch][f"group{mb}MB_ms"] = round(min(ts) * 1e3, 3)
    del model, entries, seen
print(json.dumps(out))
