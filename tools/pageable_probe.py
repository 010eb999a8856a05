"""hash_model on a model held as ordinary Python bytes (what load_model returns): pageable host memory."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2510_00554_b200 as pkg
from paper_2510_00554_b200 import shapes
out = {}
for arch in (sys.argv[1:] or ("gpt2", "bert-large", "gpt2-xl")):
    rng = np.random.default_rng(0)
    entries = []
    for name, shape, alias in shapes.ARCHITECTURES[arch]():
        if alias is not None:
            entries.append((name, dict(entries)[alias])); continue
        entries.append((name, rng.integers(0, 256, size=shapes.numel(shape) * 4, dtype=np.uint8).tobytes()))
    model = pkg.TensorMap(entries)
    cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.SHA256)
    out[arch] = {"bytes": model.total_bytes}
    from paper_2510_00554_b200 import device as dv
    for slot_mb, slots in ((32, 4), (64, 4), (128, 3)):      # transfer size of the staging ring
        dv.STAGE_SLOT_BYTES, dv.STAGE_RING_SLOTS = slot_mb << 20, slots
        pkg.hash_model(cfg, model)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter(); r = pkg.hash_model(cfg, model); ts.append(time.perf_counter() - t0)
        out[arch][f"slot{slot_mb}MBx{slots}"] = {"ms": round(min(ts) * 1e3, 2), "gbs": round(model.total_bytes / min(ts) / 1e9, 2)}
print(json.dumps(out))
