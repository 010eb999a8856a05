"""One warm and one captured launch of every leaf / LtHash kernel the bench's configurations use, in a fixed order, for
    ncu --set full --clock-control none --import-source on -k regex:"merkle_fused|lthash" -o gpurun_out/x python tools/ncu_targets.py
The order printed on stdout (two launches per line) maps the captured launches to configurations."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_2510_00554_b200 import dataset as dsm, device as dev, shapes  # noqa: E402
from lthash_lanes_probe import cifar, ragged  # noqa: E402  (PROBE_ONLY=none keeps the probe itself from running)

want = sys.argv[1:] or ["gpt2:sha256", "gpt2-model:sha256", "vgg19:blake2b", "vgg19:sha3-256", "bert-large:blake2b",
                        "bert-large:sha3-256", "gpt2:lattice", "cifar", "pool", "gpt2-xl:sha256"]
for item in want:
    if ":" in item:
        arch, alg = item.split(":")
        sd = shapes.synthetic_state_dict(arch, torch.device("cuda"))
        plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], 8192)
        if alg == "lattice":
            acc = dev.LatticeAccumulator(1)
            for _ in range(2):
                acc.add_model_leaves(plan, 0, plan.leaf_count)
        else:
            h = dev.MerkleModelHasher(plan, alg)
            for _ in range(2):
                h.run_leaves_only()
        torch.cuda.synchronize()
        print(item, plan.total_bytes, flush=True)
        del sd, plan
    else:
        shard, offs, lens, ids, src, n_src = cifar() if item == "cifar" else ragged(40_000, 2)
        ds = dsm.DeviceDataset.from_host(shard, offs, lens, ids, src, list(range(n_src)))
        acc = dev.LatticeAccumulator(n_src)
        for _ in range(2):
            ds.accumulate(acc)
        torch.cuda.synchronize()
        print(item, int(lens.sum()), flush=True)
    torch.cuda.empty_cache()
