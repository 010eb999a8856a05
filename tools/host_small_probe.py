"""Where hash_model on a host-resident GPT-2-small-sized state dict (pageable numpy / pinned tensors) spends its wall
clock: best of 5 calls and a cProfile of one call (stderr)."""
import cProfile
import io
import json
import pstats
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2510_00554_b200 as snt  # noqa: E402
from paper_2510_00554_b200 import shapes  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "gpt2"
sd = shapes.synthetic_state_dict(arch, torch.device("cuda"), seed=0)
host_np = [(k, v.cpu().numpy()) for k, v in sd]
host_pin = [(k, v.cpu().pin_memory()) for k, v in sd]
nbytes = sum(v.nbytes for _, v in host_np)
cfg = snt.HashConfig(snt.Construction.MERKLE, snt.Strategy.IN_PLACE, snt.CompressionAlg.SHA256, 8192)
out = {"arch": arch, "bytes": nbytes}
for name, items in (("pageable", host_np), ("pinned", host_pin)):
    ts = []
    for _ in range(6):
        tm = snt.TensorMap(items)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = snt.hash_model(cfg, tm)
        ts.append(time.perf_counter() - t0)
    out[f"{name}_ms"] = round(min(ts) * 1e3, 2)
    out[f"{name}_gbs"] = round(nbytes / min(ts) / 1e9, 1)
    prof = cProfile.Profile()
    tm = snt.TensorMap(items)
    prof.enable()
    snt.hash_model(cfg, tm)
    prof.disable()
    s = io.StringIO()
    pstats.Stats(prof, stream=s).sort_stats("tottime").print_stats(18)
    print(name, s.getvalue()[:5000], file=sys.stderr)
out["root"] = r.model_digest.hex()[:16]
print(json.dumps(out))
