import sys, time, cProfile, pstats, io
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parent.parent))
import torch
import paper_2510_00554_b200 as pkg
from paper_2510_00554_b200 import shapes
sd = shapes.synthetic_state_dict("gpt2-xl", torch.device("cuda"))
seen = {}
entries = []
for name, t in sd:
    if t.data_ptr() not in seen:
        h = torch.empty(t.numel()*4, dtype=torch.uint8).pin_memory(); h.copy_(t.reshape(-1).view(torch.uint8)); seen[t.data_ptr()] = h
    entries.append((name, seen[t.data_ptr()]))
del sd; torch.cuda.empty_cache()
model = pkg.TensorMap(entries)
cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.SHA256)
for _ in range(2): pkg.hash_model(cfg, model)
t0=time.perf_counter(); pkg.hash_model(cfg, model); print('e2e ms', (time.perf_counter()-t0)*1e3)
t0=time.perf_counter(); [b.is_pinned() for _, b in entries]; print('is_pinned loop ms', (time.perf_counter()-t0)*1e3)
pr=cProfile.Profile(); pr.enable(); pkg.hash_model(cfg, model); pr.disable()
s=io.StringIO(); pstats.Stats(pr,stream=s).sort_stats('tottime').print_stats(14); print(s.getvalue()[:3000])
