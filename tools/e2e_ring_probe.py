"""hash_model on pinned host tensors by ring depth (STAGE_RING_GROUPS), piece size and small-tensor threshold."""
import sys, time, json
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parent.parent))
import torch
import paper_2510_00554_b200 as pkg
from paper_2510_00554_b200 import shapes, model as mm
arch = sys.argv[1] if len(sys.argv) > 1 else "gpt2-xl"
sd = shapes.synthetic_state_dict(arch, torch.device("cuda"))
seen, entries = {}, []
for name, t in sd:
    if t.data_ptr() not in seen:
        h = torch.empty(t.numel()*4, dtype=torch.uint8).pin_memory(); h.copy_(t.reshape(-1).view(torch.uint8)); seen[t.data_ptr()] = h
    entries.append((name, seen[t.data_ptr()]))
del sd; torch.cuda.empty_cache()
model = pkg.TensorMap(entries)
cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.SHA256)
for rg, piece, small in ((3, 64, 64), (8, 64, 64), (30, 64, 64), (3, 256, 64), (3, 16, 64), (3, 64, 0), (3, 64, 1024)):
    mm.STAGE_RING_GROUPS, mm.STAGE_PIECE_BYTES, mm.SMALL_H2D_BYTES = rg, piece << 20, small << 10
    ts=[]
    for _ in range(7):
        t0=time.perf_counter(); pkg.hash_model(cfg, model); ts.append(round((time.perf_counter()-t0)*1e3,2))
    print(rg, piece, small, sorted(ts)[:3], mm.LAST_HOST_STAGING["ring_bytes"] >> 20, mm.LAST_HOST_STAGING["groups"])
