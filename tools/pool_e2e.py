#!/usr/bin/env python
"""BASELINE config 5: multi-curator pool, LtHash per curator + GPT2-XL Merkle root, sign/verify end to end.

    python tools/pool_e2e.py                      # one GPU
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tools/pool_e2e.py         # N GPUs (one rank per GPU, NCCL)

Workload: a hellaswag-shaped token dataset -- 40,000 samples,
token count clip(round(lognormal(ln 90, 0.4)), 16, 256) with default_rng(2), int32 tokens in [0, 50257),
one flat shard + offsets -- from 16 curators (Dirichlet(1) with default_rng(3)), one P-256 key per curator;
and a random-init fp32 GPT2-XL state dict. Per run:

  dataset  pinned host shard -> HBM, one LtHash launch over this rank's sample range, one all-reduce of
           the lane sums (N > 1), digests back to the host;
  model    SHA-256 Merkle in-place root of the resident state dict (leaf ranges sharded over ranks,
           one all-gather of shard roots at N > 1);
  host     one in-toto statement per curator + one for the model: ECDSA P-256 sign, then verify against
           the recomputed digests (rank 0).

Prints one JSON line with the wall time of each part (max over ranks for the GPU parts). This is an
end-to-end walk of the public API, not the bench contract's line (bench.py is).
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2510_00554_b200 as pkg  # noqa: E402
from paper_2510_00554_b200 import attestation as att  # noqa: E402
from paper_2510_00554_b200 import dataset as dsm, device as dev, distributed as dd, shapes  # noqa: E402
from paper_2510_00554_b200.model import INDEX_ENCODING  # noqa: E402

N_SAMPLES, N_CURATORS, VOCAB = 40_000, 16, 50257


def hellaswag_shaped():
    lens_tok = np.clip(np.rint(np.random.default_rng(2).lognormal(np.log(90.0), 0.4, N_SAMPLES)), 16, 256).astype(np.int64)
    lengths = (lens_tok * 4).astype(np.uint64)
    offsets = np.zeros(N_SAMPLES, dtype=np.uint64)
    np.cumsum(lengths[:-1], out=offsets[1:])
    tokens = np.random.default_rng(2).integers(0, VOCAB, size=int(lens_tok.sum()), dtype=np.int32)
    r3 = np.random.default_rng(3)
    curator = r3.choice(N_CURATORS, size=N_SAMPLES, p=r3.dirichlet(np.ones(N_CURATORS)))
    return tokens.view(np.uint8), offsets, lengths, np.arange(N_SAMPLES, dtype=np.uint64), curator


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)

    def sync_max(seconds: float) -> float:
        torch.cuda.synchronize()
        if world == 1:
            return seconds
        t = torch.tensor([seconds], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- inputs (not timed): pinned shard on the host, model resident in HBM
    shard, offsets, lengths, ids, curator = hellaswag_shaped()
    shard_pinned = torch.from_numpy(shard.copy()).pin_memory()
    a, b = dd.sample_ranges(N_SAMPLES, world)[rank]
    lo, hi = int(offsets[a]), int(offsets[b - 1] + lengths[b - 1]) if b > a else int(offsets[a])
    sd = shapes.synthetic_state_dict("gpt2-xl", device, seed=0)
    plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], 8192)
    sp = dd.plan_shards(plan.leaf_count, world)
    backend = dd.CudaBackend(plan, "sha256")
    keys = [att.KeyPair.generate() for _ in range(N_CURATORS)]
    model_key = att.KeyPair.generate()

    def dataset_pass():
        ds = dsm.DeviceDataset.from_host(shard_pinned[lo:hi], offsets[a:b] - np.uint64(lo), lengths[a:b], ids[a:b],
                                         curator[a:b], list(range(N_CURATORS)))
        acc = dev.LatticeAccumulator(N_CURATORS)
        ds.accumulate(acc)
        t_coll = 0.0
        if world > 1:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dd.allreduce_lattice(acc.state)
            torch.cuda.synchronize()
            t_coll = time.perf_counter() - t0
        out, counts, status = acc.digests()
        assert status == 0
        return out, counts, t_coll

    def model_pass():
        return backend.to_bytes(dd.sharded_merkle_root(backend, sp, rank, world))

    for _ in range(2):                      # warm-up: allocator, first-launch attributes, NCCL channels
        dataset_pass()
        model_pass()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    t0 = time.perf_counter()
    digests, counts, t_coll = dataset_pass()
    t_dataset = sync_max(time.perf_counter() - t0)
    t0 = time.perf_counter()
    root = model_pass()
    t_model = sync_max(time.perf_counter() - t0)

    line = None
    if rank == 0:
        t0 = time.perf_counter()
        bundles = []
        for c in range(N_CURATORS):
            stmt = att.Statement([att.Subject(f"pool.json:source:{c}", {"lthash": digests[64 * c:64 * c + 64].hex()})],
                                 att.DATASET_PREDICATE_TYPE,
                                 {"source_id": c, "sample_count": counts[c], "cover_labels": False,
                                  "index_encoding": INDEX_ENCODING})
            bundles.append(att.sign_bundle(stmt, keys[c]))
        cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.SHA256)
        model_bundle = att.sign_bundle(att.Statement([att.Subject("gpt2-xl", {"sha256": root.hex()})],
                                                     att.MODEL_PREDICATE_TYPE, cfg.predicate()), model_key)
        t_sign = time.perf_counter() - t0
        t0 = time.perf_counter()
        verdicts = [att.verify_bundle(bundles[c], {f"pool.json:source:{c}": {"lthash": digests[64 * c:64 * c + 64].hex()}})
                    for c in range(N_CURATORS)]
        verdicts.append(att.verify_bundle(model_bundle, {"gpt2-xl": {"sha256": root.hex()}}))
        t_verify = time.perf_counter() - t0
        assert all(v is att.Verdict.OK for v in verdicts), verdicts
        assert sum(counts) == N_SAMPLES
        line = {
            "workload": "hellaswag-shaped pool (40,000 samples, 16 curators) LtHash + GPT2-XL SHA-256 Merkle, sign/verify",
            "n_gpus": world, "samples": N_SAMPLES, "dataset_bytes": int(lengths.sum()), "model_bytes": plan.total_bytes,
            "dataset_hash_ms": round(t_dataset * 1e3, 3), "dataset_allreduce_ms": round(t_coll * 1e3, 3),
            "dataset_h2d_bytes": int(hi - lo) + 28 * (b - a),
            "model_hash_ms": round(t_model * 1e3, 3),
            "ecdsa_sign_ms": round(t_sign * 1e3, 3), "ecdsa_verify_ms": round(t_verify * 1e3, 3),
            "bundles": N_CURATORS + 1, "all_verified": True,
            "total_ms": round((t_dataset + t_model + t_sign + t_verify) * 1e3, 3),
            "samples_per_s_end_to_end": round(N_SAMPLES / t_dataset, 1),
            "model_root": root.hex(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
