"""LtHash launch on CIFAR10-shaped (50,000 x 3,072 B), hellaswag-shaped (40,000 ragged) and a 2 M-sample ragged set:
plain grid / warp chains / persistent lanes (W warps per CTA swept). Every result is compared with the grid's.
python tools/lthash_lanes_probe.py [reps]"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import _native, dataset as dsm, device as dev  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 20
lib = _native.load()


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best


def cifar():
    n, ln, n_src = 50_000, 3072, 16
    data = np.random.default_rng(0).integers(0, 256, size=n * ln, dtype=np.uint8)
    r1 = np.random.default_rng(1)
    src = r1.choice(n_src, size=n, p=r1.dirichlet(np.ones(n_src)))
    return data, np.arange(n, dtype=np.uint64) * ln, np.full(n, ln, dtype=np.uint64), np.arange(n, dtype=np.uint64), src, n_src


def ragged(n, seed):
    n_cur = 16
    lens_tok = np.clip(np.rint(np.random.default_rng(seed).lognormal(np.log(90.0), 0.4, n)), 16, 256).astype(np.int64)
    lengths = (lens_tok * 4).astype(np.uint64)
    offsets = np.zeros(n, dtype=np.uint64)
    np.cumsum(lengths[:-1], out=offsets[1:])
    tokens = np.random.default_rng(seed).integers(0, 50257, size=int(lens_tok.sum()), dtype=np.int32)
    r3 = np.random.default_rng(seed + 1)
    return tokens.view(np.uint8), offsets, lengths, np.arange(n, dtype=np.uint64), r3.choice(n_cur, size=n, p=r3.dirichlet(np.ones(n_cur))), n_cur


def main():
    only = os.environ.get("PROBE_ONLY", "").split(":") if os.environ.get("PROBE_ONLY") else None   # e.g. ragged_2M:lanes_w12
    out = {}
    for name, make in (("cifar10_shaped", cifar), ("hellaswag_40k", lambda: ragged(40_000, 2)), ("ragged_2M", lambda: ragged(2_000_000, 5))):
        if only and name != only[0]:
            continue
        shard, offs, lens, ids, src, n_src = make()
        ds = dsm.DeviceDataset.from_host(shard, offs, lens, ids, src, list(range(n_src)))
        acc = dev.LatticeAccumulator(n_src)
        variants = [("grid", _native.SCHEDULE_GRID, None), ("chains", _native.SCHEDULE_FUSED, None)]
        variants += [(f"lanes_w{w}", _native.SCHEDULE_PERSISTENT, w) for w in (4, 8, 12, 16)]
        variants += [("lanes_auto", _native.SCHEDULE_PERSISTENT, 0)]
        ref = None
        for vname, sched, w in variants:
            if only and len(only) > 1 and vname not in (only[1], "grid"):
                continue
            lib.snt_merkle_schedule(sched)
            if w:
                os.environ["SNT_LT_LANES_WARPS"] = str(w)
            else:
                os.environ.pop("SNT_LT_LANES_WARPS", None)
            acc.zero_()
            dig = torch.zeros(ds.n_samples * 64, dtype=torch.uint8, device="cuda")
            ds.accumulate(acc, digests=dig)
            got = (acc.digests(), bytes(dig.cpu().numpy().tobytes()))
            if ref is None:
                ref = got
            ok = got == ref
            ms = timed(lambda: ds.accumulate(acc))
            out[f"{name}_{vname}_us"] = round(ms * 1e3, 1)
            if not ok:
                out[f"{name}_{vname}_MISMATCH"] = True
        if name == "ragged_2M":
            lib.snt_merkle_schedule(_native.SCHEDULE_GRID)
            dss = ds.sorted_by_length()
            out["ragged_2M_sorted_grid_us"] = round(timed(lambda: dss.accumulate(acc)) * 1e3, 1)
        lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT)
        os.environ.pop("SNT_LT_LANES_WARPS", None)
        del ds, acc
    print(json.dumps(out))


if __name__ == "__main__":
    main()
