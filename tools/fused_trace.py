"""Per-SM timeline of one fused launch: when each persistent CTA started and finished, how many group
reductions and chain slices it ran.  python tools/fused_trace.py gpt2-xl sha256"""
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import _native, device as dev, shapes  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "gpt2"
alg = sys.argv[2] if len(sys.argv) > 2 else "sha256"
lib = _native.load()
if arch.startswith("flat:"):          # one contiguous tensor of that many leaves
    sd = [("flat", torch.randint(0, 256, (int(arch[5:]) * 8192,), dtype=torch.uint8, device="cuda"))]
else:
    sd = shapes.synthetic_state_dict(arch, torch.device("cuda"))
plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], 8192)
h = dev.MerkleModelHasher(plan, alg)
for _ in range(3):
    h.run()
torch.cuda.synchronize()
sms = torch.cuda.get_device_properties(0).multi_processor_count
trace = torch.zeros(6 * sms, dtype=torch.int64, device="cuda")
lib.snt_debug_fused_trace(ctypes.c_void_p(trace.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
h.run()
e1.record()
torch.cuda.synchronize()
lib.snt_debug_fused_trace(None)
t = trace.cpu().numpy().reshape(sms, 6).astype(np.int64)
t0 = t[:, 0].min()
start, end, leaf_end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 4] - t0) / 1e3
out = {"arch": arch, "alg": alg, "kernel_ms": round(e0.elapsed_time(e1), 4),
       "start_us": [round(float(start.min()), 1), round(float(start.max()), 1)],
       "last_chain_us_min_med_max": [round(float(np.min(leaf_end)), 1), round(float(np.median(leaf_end)), 1), round(float(np.max(leaf_end)), 1)],
       "end_us_min_med_max": [round(float(np.min(end)), 1), round(float(np.median(end)), 1), round(float(np.max(end)), 1)],
       "reductions_min_med_max": [int(t[:, 2].min()), int(np.median(t[:, 2])), int(t[:, 2].max())],
       "slices_min_med_max": [int(t[:, 3].min()), int(np.median(t[:, 3])), int(t[:, 3].max())]}
print(json.dumps(out))
order = np.argsort(end)
print("slowest CTAs (cta, end_us, reductions, slices):", [(int(i), round(float(end[i]), 1), int(t[i, 2]), int(t[i, 3])) for i in order[-8:]])
print("fastest CTAs (cta, end_us, reductions, slices):", [(int(i), round(float(end[i]), 1), int(t[i, 2]), int(t[i, 3])) for i in order[:8]])
import os
tagname = "_flip" if os.environ.get("SNT_FUSED_FLIP") else ""
np.save("gpurun_out/fused_trace_%s_%s%s.npy" % (arch, alg, tagname), t)
