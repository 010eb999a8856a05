"""The file-level flow of sign-model / verify-model (cli.py:109, :154): load_model(manifest) + hash_model on a
checkpoint written to disk (page cache), this package against the reference package (oracle/_ref, checker only);
digests compared. python tools/checkpoint_file_probe.py [arch] [--reference]"""
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
import paper_2510_00554_b200 as snt  # noqa: E402
from paper_2510_00554_b200 import shapes  # noqa: E402

arch = next((a for a in sys.argv[1:] if not a.startswith("-")), "gpt2")
sd = shapes.synthetic_state_dict(arch, torch.device("cuda"), seed=0)
out = {"arch": arch}
with tempfile.TemporaryDirectory(dir="/dev/shm" if Path("/dev/shm").is_dir() else None) as tmp:
    tmp = Path(tmp)
    records, pos = [], 0
    with open(tmp / "model.bin", "wb") as f:
        for name, t in sd:
            b = t.cpu().numpy().tobytes()
            f.write(b)
            records.append({"name": name, "offset": pos, "length": len(b)})
            pos += len(b)
    (tmp / "model.json").write_text(json.dumps({"tensors": records, "data": "model.bin"}))
    del sd
    torch.cuda.empty_cache()
    out["bytes"] = pos
    cfg = snt.HashConfig(snt.Construction.MERKLE, snt.Strategy.IN_PLACE, snt.CompressionAlg.SHA256, 8192)
    best = None
    for _ in range(3):
        t0 = time.perf_counter()
        model = snt.load_model(tmp / "model.json")
        t1 = time.perf_counter()
        res = snt.hash_model(cfg, model)
        t2 = time.perf_counter()
        del model
        if best is None or t2 - t0 < best[0]:
            best = (t2 - t0, t1 - t0, t2 - t1)
    out["ours"] = {"total_ms": round(best[0] * 1e3, 1), "load_model_ms": round(best[1] * 1e3, 1), "hash_model_ms": round(best[2] * 1e3, 1),
                   "gbs": round(pos / best[0] / 1e9, 2)}
    if "--reference" in sys.argv:
        import sentinel as ref  # noqa: E402

        rcfg = ref.HashConfig(ref.Construction.MERKLE, ref.Strategy.IN_PLACE, ref.CompressionAlg.SHA256, 8192)
        t0 = time.perf_counter()
        rmodel = ref.load_model(tmp / "model.json")
        t1 = time.perf_counter()
        want = ref.hash_model(rcfg, rmodel)
        t2 = time.perf_counter()
        out["reference"] = {"total_ms": round((t2 - t0) * 1e3, 1), "load_model_ms": round((t1 - t0) * 1e3, 1),
                            "hash_model_ms": round((t2 - t1) * 1e3, 1)}
        assert want.model_digest.hex() == res.model_digest.hex() and want.block_count == res.block_count
        out["parity"] = "root and block count identical"
    out["root"] = res.model_digest.hex()[:16]
print(json.dumps(out))
