#!/usr/bin/env python
"""Benchmark of the hashing hot path on B200 (contract: see the repo brief / DESIGN.md).

    python bench.py --gpus N --steps K --warmup W            # this repo's CUDA engine
    python bench.py --impl reference --gpus N --steps K ...  # the reference's CPU path (oracle port)

One "step" = one pass of the hot path over one batch of synthetic input:
the SHA-256 Merkle in-place hash of a random-init fp32 GPT2-XL state dict
(581 tensors, 6,552,089,600 bytes, 799,954 leaves of 8 KiB) down to the root.
`value` is whole-job throughput in GB/s (10^9 tensor bytes per second) with the
tensors resident in HBM; `e2e` is the same metric through the public
`hash_model(cfg, TensorMap(host tensors))` call, host->device copies included.
The CIFAR10-shaped LtHash dataset metric (samples/s) rides along under "dataset".

Multi-GPU (torchrun, one rank per GPU): the model is replicated, each rank hashes a
contiguous run of 1024-leaf shards, one all-gather of shard roots, every rank
finishes the top of the tree -> strong scaling of one model hash.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "gpt2xl_sha256_merkle_inplace_hash_throughput"
UNIT = "GB/s"
WORKLOAD = "GPT2-XL (1.5B, random-init fp32, 581 tensors, 6.55 GB) SHA-256 Merkle in-place hash, block 8192"
SHA256_OPS_PER_LEAF = 180_600      # 128 x 1400 + 904 + byte swaps, 8 KiB leaf
# ALU-pipe instructions the leaf kernel actually executes per 8 KiB leaf (SASS of merkle_leaf_kernel<0>:
# 576 SHF.W + 96 SHF + 352 LOP3 + 16 PRMT per data block, 384 SHF.W + 256 LOP3 for the constant padding
# block); every addition runs as an IMAD on the FMA pipe (616 per data block).
SHA256_ALU_INSTR_PER_LEAF = 128 * 1040 + 640


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--arch", default="gpt2-xl")
    ap.add_argument("--alg", default="sha256")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dataset", action="store_true")
    ap.add_argument("--no-intpeak", action="store_true")
    ap.add_argument("--cpu-sample-mb", type=int, default=1024)
    return ap.parse_args()


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples nvidia-smi SM clocks / throttle reasons while the timed region runs."""

    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                                      "-i", str(self.index)], capture_output=True, text=True, timeout=5).stdout
                parts = [x.strip() for x in out.strip().split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = [n for i, n in enumerate(names) if any(s[3 + i].lower().startswith("active") for s in self.samples)]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU side

def host_model_sample(arch: str, max_bytes: int, seed: int = 0):
    """The first tensors of the architecture's state dict up to ~max_bytes, random bytes (host)."""
    import numpy as np

    from paper_2510_00554_b200 import shapes

    rng = np.random.default_rng(seed)
    tensors, total = [], 0
    for _name, shape, alias in shapes.ARCHITECTURES[arch]():
        if alias is not None:
            continue
        nbytes = shapes.numel(shape) * 4
        if tensors and total + nbytes > max_bytes:
            break
        tensors.append(rng.integers(0, 256, size=nbytes, dtype=np.uint8))
        total += nbytes
    return tensors, total


def cpu_baseline_python(alg: str, tensors, total: int, workers: int, repeats: int = 1):
    """The oracle port of the reference (hashlib + thread pool), GB/s."""
    from oracle import sentinel_oracle as orc

    best = None
    for _ in range(repeats):
        t0 = time.perf_counter()
        orc.inplace_merkle(alg, tensors, 8192, workers=workers)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return total / best / 1e9, best


def cpu_baseline_c(alg: str, tensors, total: int, threads: int, repeats: int = 2):
    from oracle import c_oracle

    tl = c_oracle.TensorList(tensors)
    best = None
    for _ in range(repeats):
        t0 = time.perf_counter()
        c_oracle.inplace_merkle(alg, tl, 8192, threads)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return total / best / 1e9, best


def run_reference(args):
    """--impl reference: the reference's CPU path (its oracle port) on this box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    sample_bytes = min(args.cpu_sample_mb, 512) << 20
    tensors, total = host_model_sample(args.arch, sample_bytes)
    for _ in range(min(args.warmup, 1)):
        cpu_baseline_python(args.alg, tensors, total, cores)
    times = []
    for _ in range(max(1, min(args.steps, 10))):
        _, dt = cpu_baseline_python(args.alg, tensors, total, cores)
        times.append(dt)
    dt = statistics.median(times)
    value = total / dt / 1e9
    c_gbs, _ = cpu_baseline_c(args.alg, tensors, total, cores)
    sample = (f"first {len(tensors)} tensors of the {args.arch} state dict ({total / 1e6:.0f} MB, random bytes), "
              f"Python/hashlib port with a {cores}-thread pool, median of {len(times)} passes")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(times), "warmup": min(args.warmup, 1), "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": sample},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "c_port_all_threads_gbs": round(c_gbs, 3)},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU side

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2510_00554_b200 as pkg
    from paper_2510_00554_b200 import _native, dataset as dsm, device as dev, distributed as dd, shapes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    # debugging aid: several ranks sharing GPU 0 (gloo collectives through the host); never a bench number
    same_gpu = os.environ.get("SNT_BENCH_RANKS_SHARE_GPU0") == "1"
    if same_gpu:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    lib = _native.load()
    device = torch.device("cuda", local_rank)
    hbm_peak, peak_src = measured_peaks()

    # ---- workload: random-init fp32 state dict, every tensor its own allocation
    sd = shapes.synthetic_state_dict(args.arch, device, seed=0)
    flat = [dev.as_device_bytes(t) for _, t in sd]
    plan = dev.ModelPlan(flat, 8192)
    total_bytes, n_leaves = plan.total_bytes, plan.leaf_count
    sp = dd.plan_shards(n_leaves, world)
    backend = dd.CudaBackend(plan, args.alg)
    whole = dev.MerkleModelHasher(plan, args.alg) if world == 1 else None

    def step():
        if world == 1:
            whole.run()
            return whole.out
        return dd.sharded_merkle_root(backend, sp, rank, world)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        root_t = step()
    barrier()
    launches0 = int(lib.snt_debug_launch_count())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        ev0.record()
        for _ in range(args.steps):
            root_t = step()
        ev1.record()
        barrier()
        ms_total = ev0.elapsed_time(ev1)
        launches = int(lib.snt_debug_launch_count()) - launches0
        # keep the sampler alive for a few more passes so short runs still get clock samples
        t_end = time.time() + 1.0
        while time.time() < t_end:
            step()
        torch.cuda.synchronize()
    root_hex = root_t.cpu().numpy().tobytes().hex()
    if world > 1:
        t = torch.tensor([ms_total], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = total_bytes / (ms_step * 1e-3) / 1e9

    # ---- dominant kernel (leaf hashing) alone, CUDA events on the launching stream
    begin, end = sp.leaf_range(rank)
    leaf_hasher = whole if world == 1 else dev.MerkleModelHasher(plan, args.alg, begin, end, sp.levels)
    for _ in range(2):
        leaf_hasher.run_leaves_only()
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record()
    for _ in range(args.steps):
        leaf_hasher.run_leaves_only()
    k1.record()
    torch.cuda.synchronize()
    leaf_ms = k0.elapsed_time(k1) / args.steps
    my_leaves = end - begin
    my_bytes = total_bytes * my_leaves / n_leaves
    achieved = my_bytes / (leaf_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": f"merkle_leaf_kernel<{args.alg}>", "achieved": round(achieved, 1),
                "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": None,
                "peak_source": peak_src, "kernel_ms": round(leaf_ms, 4),
                "share_of_step": round(leaf_ms / ms_step, 4),
                "note": "binding roofline is the integer ALU pipe (see int_pipe); HBM fraction reported per contract"}
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            whole = json.loads(prof.read_text()).get(f"merkle_leaf_kernel<{args.alg}>:{args.arch}")
            # per launch, like `achieved`: a rank's launch covers its share of the leaves
            roofline["traffic"] = whole if (whole is None or world == 1) else int(whole * my_leaves / n_leaves)
        except Exception:
            pass

    # ---- integer-pipe roofline: measured on this box by tools/intpeak
    int_pipe = None
    intpeak_bin = ROOT / "tools" / "_build" / "intpeak"
    if rank == 0 and intpeak_bin.exists() and args.alg == "sha256" and not args.no_intpeak:
        try:
            out = subprocess.run([str(intpeak_bin)], capture_output=True, text=True, timeout=120).stdout
            peaks = json.loads(out.strip().splitlines()[-1])
            alu_peak = max(peaks["lop3_tops"], peaks["shf_tops"], peaks["iadd3_tops"])
            ops = SHA256_OPS_PER_LEAF * my_leaves / (leaf_ms * 1e-3) / 1e12
            alu_ops = SHA256_ALU_INSTR_PER_LEAF * my_leaves / (leaf_ms * 1e-3) / 1e12
            ceiling = peaks.get("sha256_fma_regs_gbs") or peaks["sha256_regs_gbs"]
            int_pipe = {"achieved_tops": round(ops, 3), "alu_peak_tops": round(alu_peak, 3),
                        "frac_of_alu_peak": round(ops / alu_peak, 4),
                        "alu_pipe_tops": round(alu_ops, 3), "alu_pipe_utilisation": round(alu_ops / alu_peak, 4),
                        "compute_only_gbs": ceiling, "compute_only_stock_gbs": peaks.get("sha256_regs_gbs"),
                        "frac_of_compute_only": round(achieved / ceiling, 4),
                        "ops_model": "180,600 32-bit ops per 8 KiB leaf (SURVEY.md 8(d)); the kernel issues "
                                     f"{SHA256_ALU_INSTR_PER_LEAF:,} of them on the ALU pipe and the additions as "
                                     "IMAD on the FMA pipe, so achieved_tops may exceed the ALU-only peak",
                        "microbench": peaks}
            # the unit that actually binds this kernel, next to the contractual HBM fraction
            roofline["binding_unit"] = "integer ALU pipe (SHF/LOP3/PRMT at 64 lanes/clk/SM)"
            roofline["binding_unit_frac"] = int_pipe["alu_pipe_utilisation"]
        except Exception as exc:       # the microbenchmark is evidence, not a dependency
            int_pipe = {"error": str(exc)}

    # ---- the public call on tensors that already live in HBM: hash_model(cfg, TensorMap(cuda tensors)),
    #      host wall clock per call (plan build + 3 launches + 32-byte readback); explains value vs e2e
    api_resident = None
    if world == 1:
        cfg_r = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.from_name(args.alg))
        model_r = pkg.TensorMap([(name, t) for name, t in sd])
        for _ in range(2):
            got_r = pkg.hash_model(cfg_r, model_r).model_digest.data
        assert got_r.hex() == root_hex, "hash_model on resident tensors differs from the planned hasher"
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pkg.hash_model(cfg_r, model_r)
        dt_r = (time.perf_counter() - t0) / args.steps
        api_resident = {"value": round(total_bytes / dt_r / 1e9, 2), "unit": UNIT, "ms_per_call": round(dt_r * 1e3, 4),
                        "api": "hash_model(cfg, TensorMap(CUDA tensors)), host wall clock"}
        del model_r

    # ---- end to end through the public API: pinned host tensors -> hash_model -> root bytes
    e2e = None
    if not args.no_e2e:
        cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.from_name(args.alg))
        host_entries = []
        seen = {}
        first_leaf = 0
        my_a, my_b = sp.leaf_range(rank)
        for name, t in sd:
            nbytes = t.numel() * 4
            next_leaf = first_leaf + -(-nbytes // 8192)
            mine = world == 1 or (first_leaf < my_b and next_leaf > my_a)
            key = (t.data_ptr(), mine)
            if key not in seen:
                if mine:
                    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
                    h.copy_(t.reshape(-1).view(torch.uint8))
                else:
                    h = torch.empty(nbytes, dtype=torch.uint8)   # never read by this rank: not pinned, not touched
                seen[key] = h
            host_entries.append((name, seen[key]))
            first_leaf = next_leaf
        torch.cuda.synchronize()
        if world == 1:
            model = pkg.TensorMap(host_entries)

            def e2e_step():
                return pkg.hash_model(cfg, model).model_digest.data
            h2d = total_bytes
        else:
            model = pkg.TensorMap(host_entries)

            def e2e_step():
                return dd.hash_model_sharded(cfg, model, rank, world).model_digest.data
            h2d = dd.staged_bytes(model, 8192, *sp.leaf_range(rank))
        got = e2e_step()
        assert got.hex() == root_hex, "e2e digest differs from the device-resident digest"
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        barrier()
        dt = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([dt], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": round(total_bytes / dt / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": 32, "ms_per_step": round(dt * 1e3, 3), "steps": args.e2e_steps,
               "api": "hash_model(HashConfig(MERKLE, IN_PLACE, SHA256, 8192), TensorMap(pinned host tensors))"}
        del host_entries, seen, model

    # ---- CIFAR10-shaped LtHash dataset (BASELINE config 3), samples/s
    dataset = None
    if not args.no_dataset:
        n, ln, n_src = 50_000, 3072, 16
        rng = np.random.default_rng(0)
        shard_h = torch.from_numpy(rng.integers(0, 256, size=n * ln, dtype=np.uint8)).pin_memory()
        src = np.random.default_rng(1).choice(n_src, size=n, p=np.random.default_rng(1).dirichlet(np.ones(n_src)))
        offs = np.arange(n, dtype=np.uint64) * ln
        lens = np.full(n, ln, dtype=np.uint64)
        ids = np.arange(n, dtype=np.uint64)
        dset = dsm.DeviceDataset.from_host(shard_h, offs, lens, ids, src, list(range(n_src)))
        a, b = dd.sample_ranges(n, world)[rank]
        acc = dev.LatticeAccumulator(n_src)

        def ds_step():
            acc.zero_()
            dset.accumulate(acc, a, b)
            if world > 1:
                dd.allreduce_lattice(acc.acc, acc.counts)

        for _ in range(args.warmup):
            ds_step()
        barrier()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record()
        for _ in range(args.steps):
            ds_step()
        d1.record()
        barrier()
        ds_ms = d0.elapsed_time(d1) / args.steps
        if world > 1:
            t = torch.tensor([ds_ms], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ds_ms = float(t.item())
        # e2e: shard rows from pinned host memory each step, digests back to the host
        def ds_e2e():
            d = dsm.DeviceDataset.from_host(shard_h[a * ln:b * ln], offs[:b - a], lens[a:b], ids[a:b], src[a:b],
                                            list(range(n_src)))
            acc2 = dev.LatticeAccumulator(n_src)
            d.accumulate(acc2)
            if world > 1:
                dd.allreduce_lattice(acc2.acc, acc2.counts)
            return acc2.digests()
        ds_e2e()
        barrier()
        t0 = time.perf_counter()
        for _ in range(5):
            ds_e2e()
        barrier()
        ds_dt = (time.perf_counter() - t0) / 5
        dataset = {"metric": "cifar10_shaped_lthash_samples_per_s", "value": round(n / (ds_ms * 1e-3), 1),

                   "unit": "samples/s", "ms_per_step": round(ds_ms, 4), "samples": n, "bytes": n * ln,
                   "gbs": round(n * ln / (ds_ms * 1e-3) / 1e9, 2),
                   "e2e": {"value": round(n / ds_dt, 1), "unit": "samples/s", "ms_per_step": round(ds_dt * 1e3, 3),
                           "h2d_bytes_per_step": int((b - a) * (ln + 28)), "d2h_bytes_per_step": n_src * 72}}

    # ---- CPU baseline on this box's host cores (rank 0, N=1 only), bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        tensors, total = host_model_sample(args.arch, args.cpu_sample_mb << 20)
        c_gbs, c_dt = cpu_baseline_c(args.alg, tensors, total, cores)
        py_tensors, py_total = host_model_sample(args.arch, min(args.cpu_sample_mb, 512) << 20)
        py_gbs, py_dt = cpu_baseline_python(args.alg, py_tensors, py_total, cores)
        py1_gbs, _ = cpu_baseline_python(args.alg, py_tensors[:1], py_tensors[0].size, 1)
        cpu = {"value": round(py_gbs, 4), "unit": UNIT, "cores": cores, "kind": "port",
               "sample": (f"Python/hashlib port of the reference with a {cores}-thread pool over the first "
                          f"{len(py_tensors)} tensors ({py_total / 1e6:.0f} MB) of the same state-dict layout"),
               "single_thread_gbs": round(py1_gbs, 4),
               "c_port": {"value": round(c_gbs, 3), "unit": UNIT, "threads": cores, "sample_mb": round(total / 1e6),
                          "note": "plain-C oracle, pthreads over contiguous leaf ranges, SHA-NI if the CPU has it"}}

    if rank == 0:
        line = {
            "metric": METRIC if (args.arch, args.alg) == ("gpt2-xl", "sha256")
            else f"{args.arch}_{args.alg}_merkle_inplace_hash_throughput".replace("-", ""),
            "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD if args.arch == "gpt2-xl" and args.alg == "sha256"
                       else f"{args.arch} {args.alg} Merkle in-place hash, block 8192",
                       "bytes": total_bytes, "leaves": n_leaves, "tensors": len(sd),
                       "parallelism": f"leaf-range sharding x{world}, shard = 2^{sp.levels} leaves",
                       "l2_policy": "inputs (6.55 GB per pass) larger than the 126 MB L2",
                       "root": root_hex},
            **({"debug": "ranks share GPU 0 over gloo; not a measurement"} if same_gpu else {}),
            "e2e": e2e, "api_device_resident": api_resident, "gpu_launches": launches, "clocks": clocks.summary(), "roofline": roofline,
            "int_pipe": int_pipe, "cpu_baseline": cpu, "dataset": dataset,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
