"""The transfer floor of a GPT2-XL state dict: the product's 203 copies (64 MB pieces, small tensors left out) issued alone, all 581 tensors whole, and one 6.55 GB copy."""
import sys, time, json, ctypes
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parent.parent))
import torch
from paper_2510_00554_b200 import shapes, _native
lib = _native.load()
layout = shapes.ARCHITECTURES["gpt2-xl"]()
sizes = [shapes.numel(s) * 4 for _, s, alias in layout]          # tied lm_head copied again, like the product does
hosts = {}
srcs = []
for (name, s, alias), n in zip(layout, sizes):
    key = alias or name
    if key not in hosts:
        hosts[key] = torch.empty(n, dtype=torch.uint8).pin_memory()
    srcs.append(hosts[key])
PIECE = 64 << 20
arena = torch.empty(sum(-(-n // 256) * 256 for n in sizes), dtype=torch.uint8, device="cuda")
for mode in ("all_tensors_whole", "big_only_in_64MB_pieces"):
    dst, src, ln = [], [], []
    off = 0
    for h, n in zip(srcs, sizes):
        if mode == "all_tensors_whole":
            dst.append(arena.data_ptr() + off); src.append(h.data_ptr()); ln.append(n)
        elif n >= (64 << 10):
            for o in range(0, n, PIECE):
                dst.append(arena.data_ptr() + off + o); src.append(h.data_ptr() + o); ln.append(min(PIECE, n - o))
        off += -(-n // 256) * 256
    k = len(dst)
    a = ((ctypes.c_void_p * k)(*dst), (ctypes.c_void_p * k)(*src), (ctypes.c_uint64 * k)(*ln))
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        lib.snt_memcpy_h2d_batch(a[0], a[1], a[2], k, st)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    print(mode, k, "copies", round(best * 1e3, 2), "ms", round(sum(ln) / best / 1e9, 2), "GB/s")
big = torch.empty(sum(sizes), dtype=torch.uint8).pin_memory()
d = torch.empty(sum(sizes), dtype=torch.uint8, device="cuda")
best = 1e9
for _ in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(big, non_blocking=True); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
print("one copy", round(best * 1e3, 2), "ms")
