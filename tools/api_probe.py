import sys, time, json
sys.path.insert(0, '/root/repo')
import torch
import paper_2510_00554_b200 as pkg
from paper_2510_00554_b200 import shapes
out = {}
for arch in ("gpt2", "gpt2-xl"):
    sd = shapes.synthetic_state_dict(arch, torch.device("cuda"), seed=0)
    model = pkg.TensorMap([(n, t) for n, t in sd])
    cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.SHA256)
    for _ in range(3):
        r = pkg.hash_model(cfg, model)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); r = pkg.hash_model(cfg, model); ts.append(time.perf_counter() - t0)
    out[arch] = {"hash_model_cuda_tensors_ms_median": round(sorted(ts)[5] * 1e3, 3), "min": round(min(ts) * 1e3, 3), "digest": r.digest_hex()[:16]}
    del sd, model
print(json.dumps(out))
