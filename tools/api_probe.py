"""Host overhead of the drop-in call on device-resident models: hash_model(cfg, TensorMap(CUDA tensors)) per call
against the kernels alone (MerkleModelHasher.run), with a cProfile of the call path.  python tools/api_probe.py [arch]"""
import cProfile
import io
import json
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2510_00554_b200 as pkg  # noqa: E402
from paper_2510_00554_b200 import device as dev, shapes  # noqa: E402

out = {}
for arch in sys.argv[1:] or ["gpt2", "gpt2-xl"]:
    sd = shapes.synthetic_state_dict(arch, torch.device("cuda"))
    model = pkg.TensorMap(list(sd))
    cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.SHA256)
    plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], 8192)
    h = dev.MerkleModelHasher(plan, "sha256")
    for _ in range(5):
        h.run()
        pkg.hash_model(cfg, model)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        h.run()
    e1.record()
    torch.cuda.synchronize()
    kernels_ms = e0.elapsed_time(e1) / 50
    t0 = time.perf_counter()
    for _ in range(50):
        pkg.hash_model(cfg, model)
    api_ms = (time.perf_counter() - t0) / 50 * 1e3
    prof = cProfile.Profile()
    prof.enable()
    for _ in range(50):
        pkg.hash_model(cfg, model)
    prof.disable()
    s = io.StringIO()
    pstats.Stats(prof, stream=s).sort_stats("cumulative").print_stats(12)
    out[arch] = {"kernels_ms": round(kernels_ms, 4), "hash_model_ms": round(api_ms, 4),
                 "overhead_pct": round((api_ms / kernels_ms - 1) * 100, 1)}
    print(s.getvalue()[:2500], file=sys.stderr)
    del sd, model, plan, h
print(json.dumps(out))
