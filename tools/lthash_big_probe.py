import sys, json, time
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2510_00554_b200 import _native, dataset as dsm, device as dev, shapes
lib = _native.load()
def timed(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1) / reps)
    return best
out = {}
for arch in ("bert-large", "gpt2"):
    sd = shapes.synthetic_state_dict(arch, torch.device("cuda"))
    plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], 8192)
    acc = dev.LatticeAccumulator(1)
    for name, s in (("chains", 1), ("grid", 2)):
        lib.snt_merkle_schedule(s)
        out[f"lattice_model_{arch}_{name}_ms"] = round(timed(lambda: acc.add_model_leaves(plan, 0, plan.leaf_count)), 4)
    del sd, plan
rng = np.random.default_rng(5)
n = 2_000_000
lens_tok = np.clip(np.rint(rng.lognormal(np.log(90.0), 0.4, n)), 16, 256).astype(np.int64)
lens = (lens_tok * 4).astype(np.uint64); offs = np.zeros(n, dtype=np.uint64); np.cumsum(lens[:-1], out=offs[1:])
shard = rng.integers(0, 256, size=int(lens.sum()), dtype=np.uint8)
ds = dsm.DeviceDataset.from_host(shard, offs, lens, np.arange(n, dtype=np.uint64), rng.integers(0, 16, size=n), list(range(16)))
dss = ds.sorted_by_length()
acc = dev.LatticeAccumulator(16)
for name, s in (("chains", 1), ("grid", 2)):
    lib.snt_merkle_schedule(s)
    out[f"ragged2M_{name}_ms"] = round(timed(lambda: ds.accumulate(acc)), 4)
    out[f"ragged2M_sorted_{name}_ms"] = round(timed(lambda: dss.accumulate(acc)), 4)
lib.snt_merkle_schedule(0)
torch.cuda.synchronize(); t0 = time.perf_counter(); d2 = ds.sorted_by_length(); torch.cuda.synchronize()
out["sort_warm_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
print(json.dumps(out))
