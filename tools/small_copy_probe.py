"""Cost of the small tensors of a state dict on the copy engine: GPT2-XL has 388 tensors below 64 KB. Times (CUDA
events) one batch of cudaMemcpyAsync for them (snt_memcpy_h2d_batch) against ONE gather launch that reads the pinned
host memory through the unified address space (snt_gather_spans with host source addresses)."""
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import _native, device as dev, shapes  # noqa: E402

lib = _native.load()
out = {}
for arch in ("gpt2", "gpt2-xl"):
    layout = shapes.ARCHITECTURES[arch]()
    sizes = [shapes.numel(s) * 4 for _, s, alias in layout if alias is None]
    for limit_kb in (64, 1024):
        small = [s for s in sizes if s < limit_kb << 10]
        hosts = [torch.empty(s, dtype=torch.uint8).pin_memory() for s in small]
        total = sum(-(-s // 256) * 256 for s in small)
        arena = torch.empty(total, dtype=torch.uint8, device="cuda")
        offs, o = [], 0
        for s in small:
            offs.append(o)
            o += -(-s // 256) * 256
        k = len(small)
        dst = (ctypes.c_void_p * k)(*[arena.data_ptr() + x for x in offs])
        src = (ctypes.c_void_p * k)(*[h.data_ptr() for h in hosts])
        ln = (ctypes.c_uint64 * k)(*small)
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

        def dma():
            lib.snt_memcpy_h2d_batch(dst, src, ln, k, stream)

        src_addr = np.array([h.data_ptr() for h in hosts], dtype=np.uint64)

        def gather():
            dev.gather_spans(src_addr, np.array(small, dtype=np.uint64), np.array(offs, dtype=np.uint64), 0, arena)

        res = {}
        for name, fn in (("dma_batch", dma), ("gather_uva", gather)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                fn()
            e1.record()
            torch.cuda.synchronize()
            res[name + "_us"] = round(e0.elapsed_time(e1) / 5 * 1e3, 1)
        out[f"{arch}_below_{limit_kb}KB"] = {"tensors": k, "bytes": sum(small), **res}
print(json.dumps(out))
