"""hash_model end to end (host wall clock) on the smaller BASELINE models: tensors in pinned host memory, in pageable
memory (numpy) and resident on the GPU, against the H2D floor of the link."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2510_00554_b200 as pkg  # noqa: E402
from paper_2510_00554_b200 import shapes  # noqa: E402


def best_of(fn, n=5):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


out = {}
for arch, alg in (("gpt2", "sha256"), ("vgg19", "blake2b"), ("bert-large", "sha3-256")):
    sd = shapes.synthetic_state_dict(arch, torch.device("cuda"))
    cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.from_name(alg))
    seen, pinned, pageable = {}, [], []
    for name, t in sd:
        k = t.data_ptr()
        if k not in seen:
            h = torch.empty(t.numel() * 4, dtype=torch.uint8).pin_memory()
            h.copy_(t.reshape(-1).view(torch.uint8))
            seen[k] = (h, np.array(h.numpy()))
        pinned.append((name, seen[k][0]))
        pageable.append((name, seen[k][1]))
    torch.cuda.synchronize()
    nbytes = sum(t.numel() * 4 for _, t in sd)
    m_dev, m_pin, m_page = pkg.TensorMap(list(sd)), pkg.TensorMap(pinned), pkg.TensorMap(pageable)
    root = pkg.hash_model(cfg, m_dev).model_digest.data
    assert pkg.hash_model(cfg, m_pin).model_digest.data == root and pkg.hash_model(cfg, m_page).model_digest.data == root
    big = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    hbig = torch.empty(nbytes, dtype=torch.uint8).pin_memory()

    def h2d():
        big.copy_(hbig, non_blocking=True)
        torch.cuda.synchronize()

    out[f"{arch}:{alg}"] = {"bytes": nbytes, "resident_ms": round(best_of(lambda: pkg.hash_model(cfg, m_dev)) * 1e3, 3),
                            "pinned_ms": round(best_of(lambda: pkg.hash_model(cfg, m_pin)) * 1e3, 3),
                            "pageable_ms": round(best_of(lambda: pkg.hash_model(cfg, m_page)) * 1e3, 3),
                            "one_h2d_copy_ms": round(best_of(h2d) * 1e3, 3)}
    del sd, m_dev, m_pin, m_page, pinned, pageable, seen, big, hbig
    torch.cuda.empty_cache()
print(json.dumps(out))
