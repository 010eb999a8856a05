"""hash_model wall clock for every construction x strategy from HOST memory (pageable numpy arrays, as a checkpoint
loaded by a drop-in user) and from HBM-resident tensors, GPT-2-small-shaped state dict, against the reference package
(oracle/_ref, checker only) on the same bytes; digests (model, per-layer) compared before anything is printed."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
import paper_2510_00554_b200 as snt  # noqa: E402
import sentinel as ref  # noqa: E402
from paper_2510_00554_b200 import shapes  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "gpt2"
tensors = dict(shapes.synthetic_state_dict(arch, torch.device("cuda"), seed=0))
host = {k: v.cpu().numpy() for k, v in tensors.items()}
nbytes = sum(v.nbytes for v in host.values())
out = {"arch": arch, "bytes": nbytes, "rows": []}
combos = [("merkle", "in-place", "sha256", False), ("merkle", "per-layer", "sha256", False), ("merkle", "coalesced", "sha256", False),
          ("lattice", "in-place", "blake2b", False), ("lattice", "per-layer", "blake2b", False), ("lattice", "per-layer", "blake2b", True),
          ("lattice", "coalesced", "blake2b", False)]
for cons, strat, alg, ordered in combos:
    cfg = snt.HashConfig(snt.Construction(cons), snt.Strategy(strat), snt.CompressionAlg(alg), 8192, ordered)
    rcfg = ref.HashConfig(ref.Construction(cons), ref.Strategy(strat), ref.CompressionAlg(alg), 8192, ordered)
    t0 = time.perf_counter()
    want = ref.hash_model(rcfg, ref.TensorMap([(k, memoryview(v).cast("B")) for k, v in host.items()]))
    t_ref = time.perf_counter() - t0
    row = {"construction": cons, "strategy": strat, "ordered": ordered, "reference_ms": round(t_ref * 1e3, 1)}
    for where, tm_of in (("host", lambda: snt.TensorMap(list(host.items()))), ("hbm", lambda: snt.TensorMap(list(tensors.items())))):
        ts = []
        for _ in range(4):
            tm = tm_of()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            got = snt.hash_model(cfg, tm)
            ts.append(time.perf_counter() - t0)
        assert got.model_digest.hex() == want.model_digest.hex(), (cons, strat, where)
        assert (got.layer_digests is None) == (want.layer_digests is None)
        if got.layer_digests is not None:
            assert {k: d.hex() for k, d in got.layer_digests.items()} == {k: d.hex() for k, d in want.layer_digests.items()}
        assert got.block_count == want.block_count and got.aux_data_bytes == want.aux_data_bytes
        row[f"{where}_ms"] = round(min(ts) * 1e3, 2)
    row["speedup_host"] = round(row["reference_ms"] / row["host_ms"], 1)
    out["rows"].append(row)
print(json.dumps(out))
