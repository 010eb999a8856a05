#!/usr/bin/env python
"""Benchmark of the hashing hot path on B200 (contract: see the repo brief / DESIGN.md section 6).

    python bench.py --gpus N --steps K --warmup W            # this repo's CUDA engine
    python bench.py --impl reference --gpus N --steps K ...  # the UNMODIFIED reference package on the host cores

One "step" = one pass of the hot path over one batch of synthetic input: the SHA-256 Merkle in-place hash
of a random-init fp32 GPT2-XL state dict (581 tensors, 6,552,089,600 bytes, 799,954 leaves of 8 KiB) down
to the root. `value` is whole-job throughput in GB/s (10^9 tensor bytes per second) with the tensors
resident in HBM; `e2e` is the same metric through the public `hash_model(cfg, TensorMap(host tensors))`
call, host->device copies included. Every other BASELINE.json configuration rides along under "configs"
(GPT-2 small SHA-256; BERT-large and VGG19 x {BLAKE2b, SHA3-256}; CIFAR10-shaped LtHash; the
hellaswag-shaped pool of config 5), each with its own roofline and CPU reference. Beside `e2e` (page-locked host
tensors) the line carries `e2e_pageable_host` (ordinary numpy arrays) and `e2e_checkpoint_file` (`load_model` +
`hash_model` on a checkpoint file the bench writes to tmpfs); the dataset configurations add `process_batch_api`
(the reference's loader loop), `manifest_api` (`digest_dataset` on manifest + shard file) and `streaming_api`.

Parity is checked before any time is printed: the reference package
(`oracle/_ref/sentinel`, staged by build()) hashes the D2H copy of the very bytes the GPU hashed; roots,
leaf digests (sampled) and per-source lattice digests must be bit-identical or the run aborts.

Multi-GPU (`--gpus N`, N > 1): when not already under torchrun the script re-launches itself with one
rank per GPU (`python -m torch.distributed.run`); the model is replicated, each rank hashes a
contiguous run of 1024-leaf shards, one NCCL all-gather of shard roots, every rank finishes the top of
the tree -> strong scaling of one model hash. NCCL_DEBUG=INFO is set so the communicator lines land on
stderr.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
BLOCK = 8192
# Root of the seed-0 GPT2-XL state dict of shapes.synthetic_state_dict generated on a CUDA device (torch's
# Philox stream): both arms hash these very bytes, the reference arm checks its root against this pin.
PINNED_ROOTS = {("gpt2-xl", "sha256"): "d11fec86b65f2f91ce084c01ba14010fcec9e4a2f07bd2497ba4aca7fdfa9d41"}

# Instructions one thread issues per 8 KiB leaf, from the SASS of the persistent kernel
# (profiles/r2_sass_report.txt, tools/sass_report.py): the aligned SHA-256 loop is 1,046 ALU-pipe + 603
# FMA-pipe (IMAD) instructions per 64-byte block, the constant padding block 640 + 512; one BLAKE2b block
# (128 B, message staging included) 2,066 + 226; one Keccak round 181 ALU, 24 rounds + ~110 of absorb per
# 136-byte block, no additions.
ALU_PER_LEAF = {"sha256": 128 * 1046 + 640, "blake2b": 64 * 2066, "sha3-256": 61 * (24 * 181 + 110)}
FMA_PER_LEAF = {"sha256": 128 * 603 + 512, "blake2b": 64 * 226, "sha3-256": 0}
LT_ALU_PER_BLOCK, LT_FMA_PER_BLOCK = 2150, 276        # lthash kernel, one 128-byte BLAKE2b block of a sample
SHA256_OPS_PER_LEAF = 180_600                         # SURVEY.md section 8(d) op model (128 x 1400 + 904 + swaps)


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
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-intpeak", action="store_true")
    ap.add_argument("--reference-budget-s", type=float, default=200.0,
                    help="--impl reference: wall-clock budget of the timed passes; above it a prefix of the model is hashed")
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


# ----------------------------------------------------------------------------- the reference package (CPU)

def load_reference():
    """The unmodified reference package staged under oracle/_ref by build(); None if it did not travel."""
    ref_dir = ROOT / "oracle" / "_ref"
    if not (ref_dir / "sentinel" / "__init__.py").exists():
        try:
            from paper_2510_00554_b200 import build

            build.stage_reference()
        except Exception:
            pass
    if not (ref_dir / "sentinel" / "__init__.py").exists():
        return None
    if str(ref_dir) not in sys.path:
        sys.path.insert(0, str(ref_dir))
    import sentinel

    return sentinel


def host_views(sd):
    """Host copies of the device tensors: [(name, uint8 numpy array)], tied entries shared."""
    import torch

    seen, out = {}, []
    for name, t in sd:
        key = t.data_ptr()
        if key not in seen:
            seen[key] = t.reshape(-1).view(torch.uint8).cpu().numpy()
        out.append((name, seen[key]))
    return out


def reference_model(ref, host):
    return ref.TensorMap([(name, memoryview(arr)) for name, arr in host])


def reference_cfg(ref, alg):
    return ref.HashConfig(ref.Construction.MERKLE, ref.Strategy.IN_PLACE, ref.CompressionAlg.from_name(alg), BLOCK)


def timed_cpu(fn, repeats=1):
    best, out = None, None
    for _ in range(repeats):
        t0 = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, out


def reference_leaf_digests(ref, alg, host, max_bytes):
    """hash_blocks(...).data of the reference over the first tensors (<= max_bytes): bytes, leaf count, tensor count."""
    entries, total = [], 0
    for name, arr in host:
        if entries and total + arr.size > max_bytes:
            break
        entries.append((name, memoryview(arr)))
        total += arr.size
    tm = ref.TensorMap(entries)
    table = ref.BlockTable.build(tm, BLOCK)
    views = [memoryview(buf) for _, buf in tm.entries]
    blocks = [views[t][off:off + ln] for _, t, off, ln in table.rows]
    buf = ref.hash_blocks(ref.CompressionAlg.from_name(alg), blocks, os.cpu_count() or 1)
    return bytes(buf.data), len(blocks), len(entries)


# ----------------------------------------------------------------------------- --impl reference

def run_reference(args):
    """The reference's own CPU implementation of the path, all host threads, on the bytes the GPU arm hashes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch

    from paper_2510_00554_b200 import shapes

    cores = os.cpu_count() or 1
    ref = load_reference()
    on_cuda = torch.cuda.is_available()
    device = torch.device("cuda", 0) if on_cuda else torch.device("cpu")
    sd = shapes.synthetic_state_dict(args.arch, device, seed=0)
    host = host_views(sd)
    total_bytes = sum(arr.size for _, arr in host)
    n_leaves = sum(-(-arr.size // BLOCK) for _, arr in host)
    del sd
    if on_cuda:
        torch.cuda.empty_cache()
    if ref is not None:
        kind = "reference"
        cfg = reference_cfg(ref, args.alg)

        def one_pass(h):
            return ref.hash_model(cfg, reference_model(ref, h), workers=cores).model_digest.data.hex()
    else:                                   # the staged copy did not travel: the oracle port stands in, and says so
        kind = "port"
        from oracle import sentinel_oracle as orc

        def one_pass(h):
            return orc.inplace_merkle(args.alg, [a for _, a in h], BLOCK, workers=cores).hex()

    # first (untimed) pass: the root check, and the per-pass cost that decides between the full model and a prefix
    t_first, root = timed_cpu(lambda: one_pass(host))
    pinned = PINNED_ROOTS.get((args.arch, args.alg)) if on_cuda else None
    root_ok = None if pinned is None else (root == pinned)
    if root_ok is False:
        print(f"bench.py: reference root {root} differs from the pinned root {pinned}", file=sys.stderr)
    passes = max(0, args.warmup - 1) + args.steps
    sample_host, sample_bytes, sample_note = host, total_bytes, "the full state dict"
    if passes * t_first > args.reference_budget_s:
        want = total_bytes * args.reference_budget_s / (passes * t_first)
        sample_host, sample_bytes = [], 0
        for name, arr in host:
            if sample_host and sample_bytes + arr.size > want:
                break
            sample_host.append((name, arr))
            sample_bytes += arr.size
        sample_note = f"the first {len(sample_host)} tensors ({sample_bytes / 1e6:.0f} MB) of the state dict"
    for _ in range(max(0, args.warmup - 1)):
        one_pass(sample_host)
    times = []
    for _ in range(args.steps):
        dt, _ = timed_cpu(lambda: one_pass(sample_host))
        times.append(dt)
    dt = statistics.median(times)
    value = sample_bytes / dt / 1e9
    sample = (f"{'reference package sentinel.hash_model' if kind == 'reference' else 'oracle port'}"
              f"(MERKLE, IN_PLACE, {args.alg}, 8192, workers={cores}) over {sample_note}, "
              f"bytes = D2H copy of the GPU arm's tensors" + ("" if on_cuda else " (no CUDA device: CPU generator)"))
    headline = (args.arch, args.alg) == ("gpt2-xl", "sha256")
    line = {
        "impl": "reference",
        "metric": METRIC if headline else f"{args.arch}_{args.alg}_merkle_inplace_hash_throughput".replace("-", ""),
        "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": WORKLOAD if headline else f"{args.arch} {args.alg} Merkle in-place hash, block {BLOCK}",
                   "bytes": total_bytes, "leaves": n_leaves, "tensors": len(host),
                   "root": root, "root_matches_pinned": root_ok, "sample": sample, "sample_bytes": sample_bytes},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU side helpers

def cuda_time_ms(fn, steps, warmup=2):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def run_intpeak():
    exe = ROOT / "tools" / "_build" / "intpeak"
    if not exe.exists():
        return None
    try:
        out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120).stdout
        return json.loads(out.strip().splitlines()[-1])
    except Exception as exc:                   # the microbenchmark is evidence, not a dependency
        return {"error": str(exc)}


def model_roofline(alg, arch, kernel_ms, leaves, nbytes, step_ms, hbm_peak, peak_src, peaks, traffic):
    """Roofline of the leaf-stage launch (the dominant kernel): HBM fraction per contract, and the unit that binds."""
    achieved = nbytes / (kernel_ms * 1e-3) / 1e9
    r = {"bound": "hbm", "kernel": f"merkle_fused_kernel<{alg}> (persistent leaf stage)", "achieved": round(achieved, 1),
         "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
         "peak_source": peak_src, "kernel_ms": round(kernel_ms, 4), "share_of_step": round(kernel_ms / step_ms, 4),
         "algorithmic_bytes": nbytes}
    if peaks and "error" not in peaks:
        alu_peak = max(peaks["lop3_tops"], peaks["shf_tops"], peaks["iadd3_tops"])
        fma_peak = peaks.get("imad_tops", alu_peak)
        alu = ALU_PER_LEAF[alg] * leaves / (kernel_ms * 1e-3) / 1e12
        fma = FMA_PER_LEAF[alg] * leaves / (kernel_ms * 1e-3) / 1e12
        r.update({"binding_unit": "integer ALU pipe (SHF / LOP3 / PRMT / IADD3, 64 lanes/clk/SM)",
                  "binding_unit_frac": round(alu / alu_peak, 4),
                  "alu_pipe_tops": round(alu, 3), "alu_peak_tops": round(alu_peak, 3),
                  "fma_pipe_tops": round(fma, 3), "fma_peak_tops": round(fma_peak, 3),
                  "issue_budget_frac": round((alu + fma) / (alu_peak + fma_peak), 4),
                  "note": "binding roofline is the integer ALU pipe; the HBM fraction is reported per contract. "
                          "Instruction counts per leaf from profiles/r2_sass_report.txt, peaks from tools/intpeak."})
    return r


def gpu_model_config(pkg, dev, shapes, arch, alg, device, steps, hbm_peak, peak_src, peaks, ref, cores, traffic_db):
    """One ride-along Merkle configuration: GPU time, roofline, and the reference on the same bytes (root asserted)."""
    import torch

    sd = shapes.synthetic_state_dict(arch, device, seed=0)
    plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], BLOCK)
    hasher = dev.MerkleModelHasher(plan, alg)
    step_ms = cuda_time_ms(hasher.run, steps, 3)
    leaf_ms = cuda_time_ms(hasher.run_leaves_only, steps, 2)
    hasher.run()
    root = hasher.out_bytes().hex()
    out = {"workload": f"{arch} (random-init fp32) {alg} Merkle in-place hash, block {BLOCK}", "arch": arch, "alg": alg,
           "bytes": plan.total_bytes, "leaves": plan.leaf_count, "tensors": len(sd),
           "ms_per_step": round(step_ms, 4), "value": round(plan.total_bytes / step_ms / 1e6, 2), "unit": UNIT,
           "root": root,
           "roofline": model_roofline(alg, arch, leaf_ms, plan.leaf_count, plan.total_bytes, step_ms, hbm_peak, peak_src,
                                      peaks, traffic_db.get(f"merkle_fused_kernel<{alg}>:{arch}"))}
    # the public call on the same resident tensors: host wall clock per hash_model(cfg, TensorMap(CUDA tensors))
    api_cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.from_name(alg))
    model_r = pkg.TensorMap([(name, t) for name, t in sd])
    for _ in range(3):
        got_r = pkg.hash_model(api_cfg, model_r).model_digest.data
    assert got_r.hex() == root, f"{arch}/{alg}: hash_model on resident tensors differs from the planned hasher"
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        pkg.hash_model(api_cfg, model_r)
    dt_r = (time.perf_counter() - t0) / steps
    out["api_device_resident"] = {"ms_per_call": round(dt_r * 1e3, 4),
                                  "overhead_vs_value_pct": round((dt_r * 1e3 / step_ms - 1) * 100, 2)}
    del model_r
    if ref is not None:
        host = host_views(sd)
        cfg = reference_cfg(ref, alg)
        dt_all, res = timed_cpu(lambda: ref.hash_model(cfg, reference_model(ref, host), workers=cores))
        assert res.model_digest.data.hex() == root, f"{arch}/{alg}: GPU root differs from the reference package's"
        leaves_ref, n_ref, n_tensors = reference_leaf_digests(ref, alg, host, 64 << 20)
        dl = dev.DIGEST_LEN[alg]
        assert hasher.leaf_bytes()[:n_ref * dl] == leaves_ref, f"{arch}/{alg}: leaf digests differ from the reference's"
        out["cpu_baseline"] = {"value": round(plan.total_bytes / dt_all / 1e9, 4), "unit": UNIT, "cores": cores,
                               "kind": "reference", "ms": round(dt_all * 1e3, 1),
                               "sample": f"sentinel.hash_model(workers={cores}) over the D2H copy of the full state dict, one pass",
                               "parity": f"root identical; first {n_ref} leaf digests ({n_tensors} tensors) identical"}
    del hasher
    plan.close()
    del plan, sd
    torch.cuda.empty_cache()
    return out


def lattice_model_config(pkg, dev, shapes, arch, device, steps, hbm_peak, peak_src, peaks, ref, cores, traffic_db=None):
    """LATTICE in-place model hashing (reference model.py:312-315): every 8 KiB block hashed as
    BLAKE2b-512(LE64(k) || block), the u16 lanes summed into ONE 64-byte digest. GPU time and roofline; with `ref`
    the reference package on the same bytes (digest asserted)."""
    import torch

    sd = shapes.synthetic_state_dict(arch, device, seed=0)
    plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], BLOCK)
    acc = dev.LatticeAccumulator(1)

    def step():
        acc.zero_()
        acc.add_model_leaves(plan, 0, plan.leaf_count)

    step_ms = cuda_time_ms(step, steps, 3)
    step()
    digest, counts, _ = acc.digests()
    assert counts == [plan.leaf_count]
    cfg = pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.BLAKE2B)
    api = pkg.hash_model(cfg, pkg.TensorMap([(name, t) for name, t in sd]))
    assert api.model_digest.data == digest
    achieved = plan.total_bytes / (step_ms * 1e-3) / 1e9
    # BLAKE2b blocks: ceil((8 + leaf bytes) / 128) per leaf -- 65 for a full 8 KiB leaf, fewer for a tensor's ragged tail
    blocks = 0
    for _, t in sd:
        nb = t.numel() * t.element_size()
        full, tail = divmod(nb, BLOCK)
        blocks += full * ((8 + BLOCK + 127) // 128) + (((8 + tail + 127) // 128) if tail else 0)
    roof = {"bound": "hbm", "kernel": "lthash kernel over model blocks (BLAKE2b per block + lane sums)", "achieved": round(achieved, 1),
            "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
            "traffic": (traffic_db or {}).get(f"lthash_chain_kernel:{arch}"), "peak_source": peak_src,
            "kernel_ms": round(step_ms, 4), "algorithmic_bytes": plan.total_bytes}
    if peaks and "error" not in peaks:
        alu_peak = max(peaks["lop3_tops"], peaks["shf_tops"], peaks["iadd3_tops"])
        roof.update({"binding_unit": "integer ALU pipe",
                     # per-block count of the unrolled BLAKE2b compression the chain kernel runs (SASS, as ALU_PER_LEAF)
                     "binding_unit_frac": round(ALU_PER_LEAF["blake2b"] // 64 * blocks / (step_ms * 1e-3) / 1e12 / alu_peak, 4),
                     "blake2b_blocks": blocks})
    out = {"workload": f"{arch} (random-init fp32) LATTICE in-place model hash (LtHash over 8 KiB blocks), block {BLOCK}",
           "arch": arch, "alg": "lthash-blake2b", "bytes": plan.total_bytes, "leaves": plan.leaf_count, "tensors": len(sd),
           "ms_per_step": round(step_ms, 4), "value": round(plan.total_bytes / step_ms / 1e6, 2), "unit": UNIT,
           "digest": digest.hex()[:32], "roofline": roof}
    if ref is not None:
        host = host_views(sd)
        rcfg = ref.HashConfig(ref.Construction.LATTICE, ref.Strategy.IN_PLACE, ref.CompressionAlg.BLAKE2B, BLOCK)
        dt, res = timed_cpu(lambda: ref.hash_model(rcfg, reference_model(ref, host), workers=cores))
        assert res.model_digest.data == digest, f"{arch}: GPU lattice digest differs from the reference package's"
        out["cpu_baseline"] = {"value": round(plan.total_bytes / dt / 1e9, 4), "unit": UNIT, "cores": cores, "kind": "reference",
                               "ms": round(dt * 1e3, 1), "parity": "64-byte lattice digest identical",
                               "sample": f"sentinel.hash_model(LATTICE, IN_PLACE, workers={cores}) over the D2H copy of the full state dict, one pass"}
    plan.close()
    del plan, sd, acc
    torch.cuda.empty_cache()
    return out


def cifar_shaped(np):
    n, ln, n_src = 50_000, 3072, 16
    data = np.random.default_rng(0).integers(0, 256, size=n * ln, dtype=np.uint8)
    r1 = np.random.default_rng(1)
    src = r1.choice(n_src, size=n, p=r1.dirichlet(np.ones(n_src)))
    offs = np.arange(n, dtype=np.uint64) * ln
    return data, offs, np.full(n, ln, dtype=np.uint64), np.arange(n, dtype=np.uint64), src, n_src


def hellaswag_shaped(np):
    n, n_cur, vocab = 40_000, 16, 50257
    lens_tok = np.clip(np.rint(np.random.default_rng(2).lognormal(np.log(90.0), 0.4, n)), 16, 256).astype(np.int64)
    lengths = (lens_tok * 4).astype(np.uint64)
    offsets = np.zeros(n, dtype=np.uint64)
    np.cumsum(lengths[:-1], out=offsets[1:])
    tokens = np.random.default_rng(2).integers(0, vocab, size=int(lens_tok.sum()), dtype=np.int32)
    r3 = np.random.default_rng(3)
    curator = r3.choice(n_cur, size=n, p=r3.dirichlet(np.ones(n_cur)))
    return tokens.view(np.uint8), offsets, lengths, np.arange(n, dtype=np.uint64), curator, n_cur


def reference_dataset_digests(ref, shard, offs, lens, ids, src, n_src, batch=128):
    """The reference's loader loop: SourceAccumulator + process_batch over batches of 128, then finalize."""
    view = memoryview(shard)
    acc = ref.SourceAccumulator()
    acc.declare(range(n_src))
    n = len(ids)
    t0 = time.perf_counter()
    for s in range(0, n, batch):
        recs = [ref.SampleRecord(int(ids[i]), int(src[i]), b"", bytes(view[int(offs[i]):int(offs[i] + lens[i])]))
                for i in range(s, min(n, s + batch))]
        ref.process_batch(ref.Batch(recs), acc)
    out = ref.finalize(acc)
    return time.perf_counter() - t0, out


def dataset_config(name, workload, arrays, np, torch, dsm, dev, dd, world, rank, steps, warmup, barrier, device,
                   hbm_peak, peak_src, peaks, ref, cores, traffic_db=None):
    """A LtHash dataset configuration: device-resident samples/s, end to end from pinned host memory, the
    reference loop on the same samples (per-source digests and counts asserted), roofline of the kernel."""
    import torch.distributed as dist

    shard, offs, lens, ids, src, n_src = arrays
    n = len(ids)
    shard_h = torch.from_numpy(shard).pin_memory()
    dset = dsm.DeviceDataset.from_host(shard_h, offs, lens, ids, src, list(range(n_src)))
    a, b = dd.sample_ranges(n, world)[rank]
    acc = dev.LatticeAccumulator(n_src)

    def ds_step():
        acc.zero_()
        dset.accumulate(acc, a, b)
        if world > 1:
            dd.allreduce_lattice(acc.state)

    for _ in range(max(warmup, 3)):
        ds_step()
    barrier()
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record()
    for _ in range(steps):
        ds_step()
    d1.record()
    barrier()
    ds_ms = d0.elapsed_time(d1) / steps
    kernel_ms = cuda_time_ms(lambda: dset.accumulate(acc, a, b), steps, 2)
    if world > 1:
        t = torch.tensor([ds_ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ds_ms = float(t.item())
    ds_step()
    digests, counts, status = acc.digests()
    assert status == 0
    lo = int(offs[a])
    hi = int(offs[b - 1] + lens[b - 1]) if b > a else lo

    def ds_e2e():       # rows and shard bytes of this rank's range from pinned host memory each step, digests back
        d = dsm.DeviceDataset.from_host(shard_h[lo:hi], offs[a:b] - np.uint64(lo), lens[a:b], ids[a:b], src[a:b],
                                        list(range(n_src)))
        acc2 = dev.LatticeAccumulator(n_src)
        d.accumulate(acc2)
        if world > 1:
            dd.allreduce_lattice(acc2.state)
        return acc2.digests()

    ds_e2e()
    ds_dt = None
    for _ in range(3):          # three rounds of five calls, best round: the page-locked allocator's reuse varies run to run
        barrier()
        t0 = time.perf_counter()
        for _ in range(5):
            ds_e2e()
        barrier()
        dt5 = (time.perf_counter() - t0) / 5
        ds_dt = dt5 if ds_dt is None else min(ds_dt, dt5)
    nbytes = int(lens.sum())
    my_bytes = int(lens[a:b].sum())
    blocks = int(((lens[a:b] + np.uint64(8 + 127)) // np.uint64(128)).sum())
    achieved = my_bytes / (kernel_ms * 1e-3) / 1e9
    kernel_name = ("lthash_kernel (one thread per sample: samples of one length)" if dset.uniform else
                   "lthash_lanes_kernel (persistent lanes: ragged samples, no sort)")
    roof = {"bound": "hbm", "kernel": kernel_name + ", BLAKE2b per sample + per-source lane sums", "achieved": round(achieved, 1),
            "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
            "traffic": (traffic_db or {}).get(("lthash_kernel:" if dset.uniform else "lthash_lanes_kernel:") + name) if world == 1 else None,
            "peak_source": peak_src,
            "kernel_ms": round(kernel_ms, 4), "share_of_step": round(kernel_ms / ds_ms, 4), "algorithmic_bytes": my_bytes}
    if peaks and "error" not in peaks:
        alu_peak = max(peaks["lop3_tops"], peaks["shf_tops"], peaks["iadd3_tops"])
        alu = LT_ALU_PER_BLOCK * blocks / (kernel_ms * 1e-3) / 1e12
        roof.update({"binding_unit": "integer ALU pipe", "binding_unit_frac": round(alu / alu_peak, 4),
                     "alu_pipe_tops": round(alu, 3), "alu_peak_tops": round(alu_peak, 3), "blake2b_blocks": blocks})
    out = {"metric": f"{name}_lthash_samples_per_s", "workload": workload, "value": round(n / (ds_ms * 1e-3), 1),
           "unit": "samples/s", "ms_per_step": round(ds_ms, 4), "samples": n, "sources": n_src, "bytes": nbytes,
           "gbs": round(nbytes / (ds_ms * 1e-3) / 1e9, 2), "roofline": roof,
           "e2e": {"value": round(n / ds_dt, 1), "unit": "samples/s", "ms_per_step": round(ds_dt * 1e3, 3),
                   "h2d_bytes_per_step": int(hi - lo) + 28 * (b - a), "d2h_bytes_per_step": n_src * 72 + 8}}
    if world == 1:
        # the reference-shaped loader loop on this engine: process_batch over batches of 128 host records
        def api_loop():
            view = memoryview(shard)
            sacc = dsm.SourceAccumulator()
            sacc.declare(range(n_src))
            for s in range(0, n, 128):
                recs = [dsm.SampleRecord(int(ids[i]), int(src[i]), b"", bytes(view[int(offs[i]):int(offs[i] + lens[i])]))
                        for i in range(s, min(n, s + 128))]
                dsm.process_batch(dsm.Batch(recs), sacc)
            return dsm.finalize(sacc)

        api_loop()
        dt_api, got_api = timed_cpu(api_loop, 2)
        for i in range(n_src):
            assert (got_api[i][0].data, got_api[i][1]) == (digests[64 * i:64 * i + 64], counts[i]), \
                f"{name}: process_batch loop differs from the one-launch digest for source {i}"
        out["process_batch_api"] = {"value": round(n / dt_api, 1), "unit": "samples/s", "ms": round(dt_api * 1e3, 1),
                                    "api": "SourceAccumulator + process_batch(Batch of 128 host SampleRecords) x "
                                           f"{-(-n // 128)} + finalize, host wall clock incl. building the records"}
        if dset.uniform:
            # the loader-side hook: batches that already live on the GPU, no host round trip
            row = int(lens[0])
            rows_d = dset.shard[:n * row].view(n, row)
            ids_d = torch.from_numpy(np.asarray(ids, dtype=np.uint64).view(np.int64)).to(device)
            src_d = torch.from_numpy(np.asarray(src, dtype=np.int64)).to(device)

            def stream_loop():
                sh = dsm.StreamingDatasetHasher(range(n_src))
                for s in range(0, n, 128):
                    sh.update(rows_d[s:s + 128], ids_d[s:s + 128], src_d[s:s + 128])
                return sh.finalize()

            stream_loop()
            dt_s, got_s = timed_cpu(stream_loop, 2)
            for i in range(n_src):
                assert (got_s[i][0].data, got_s[i][1]) == (digests[64 * i:64 * i + 64], counts[i]), \
                    f"{name}: streaming hasher differs from the one-launch digest for source {i}"
            out["streaming_api"] = {"value": round(n / dt_s, 1), "unit": "samples/s", "ms": round(dt_s * 1e3, 1),
                                    "api": f"StreamingDatasetHasher.update(device batch of 128 rows) x {-(-n // 128)} + finalize, "
                                           "host wall clock (batches resident in HBM, as a GPU data loader holds them)"}
    if world == 1:
        # the manifest-level call (dataset.py:166-195): manifest + shard FILE in, per-source digests out
        import tempfile

        with tempfile.TemporaryDirectory() as tmp:
            rows = [(int(ids[i]), int(src[i]), b"", int(offs[i]), int(lens[i])) for i in range(n)]
            man = dsm.DatasetManifest(rows, Path(tmp) / "shard.bin")
            man.save(Path(tmp) / "manifest.json", memoryview(shard))
            dsm.digest_dataset(man)
            dt_m, got_m = timed_cpu(lambda: dsm.digest_dataset(man), 3)
            for i, sid in enumerate(sorted(got_m)):
                assert (got_m[sid][0].data, got_m[sid][1]) == (digests[64 * sid:64 * sid + 64], counts[sid]), \
                    f"{name}: digest_dataset(manifest) differs from the one-launch digest for source {sid}"
            out["manifest_api"] = {"value": round(n / dt_m, 1), "unit": "samples/s", "ms": round(dt_m * 1e3, 2),
                                   "api": "digest_dataset(DatasetManifest) on a shard file (page cache), host wall clock: "
                                          "file -> pinned ring -> HBM, one launch, digests back"}
            if ref is not None:
                rman = ref.DatasetManifest.load(Path(tmp) / "manifest.json")
                t0 = time.perf_counter()
                want_m = ref.digest_dataset(rman)
                out["manifest_api"]["reference_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
                assert {k: (v[0].data, v[1]) for k, v in want_m.items()} == {k: (v[0].data, v[1]) for k, v in got_m.items()}
                out["manifest_api"]["parity"] = "per-source digests and counts identical to sentinel.digest_dataset on the same files"
    if ref is not None and world == 1:
        dt, want = reference_dataset_digests(ref, shard, offs, lens, ids, src, n_src)
        for i in range(n_src):
            assert (digests[64 * i:64 * i + 64], counts[i]) == (want[i][0].data, want[i][1]), \
                f"{name}: source {i} differs from the reference package's digest"
        out["cpu_baseline"] = {"value": round(n / dt, 1), "unit": "samples/s", "cores": 1, "kind": "reference",
                               "ms": round(dt * 1e3, 1),
                               "sample": "sentinel.SourceAccumulator + process_batch over all samples in batches of 128, "
                                         "finalize (single thread, as the reference runs it)",
                               "parity": f"all {n_src} per-source digests and counts identical"}
    return out, (digests, counts)


# ----------------------------------------------------------------------------- GPU arm

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2510_00554_b200 as pkg
    from paper_2510_00554_b200 import _native, attestation as att, dataset as dsm, device as dev, distributed as dd, shapes
    from paper_2510_00554_b200.model import INDEX_ENCODING

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
    cores = os.cpu_count() or 1
    ref = load_reference() if (rank == 0 and world == 1 and not args.no_cpu_baseline) else None
    traffic_db = {}
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            traffic_db = json.loads(prof.read_text())
        except Exception:
            traffic_db = {}

    # ---- workload: random-init fp32 state dict, every tensor its own allocation
    sd = shapes.synthetic_state_dict(args.arch, device, seed=0)
    n_tensors = len(sd)
    flat = [dev.as_device_bytes(t) for _, t in sd]
    plan = dev.ModelPlan(flat, BLOCK)
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

    # ---- dominant kernel (the persistent leaf-stage launch) alone, CUDA events on the launching stream
    begin, end = sp.leaf_range(rank)
    leaf_hasher = whole if world == 1 else dev.MerkleModelHasher(plan, args.alg, begin, end, sp.levels)
    leaf_ms = cuda_time_ms(leaf_hasher.run_leaves_only, args.steps, 2)
    my_leaves = end - begin
    my_bytes = int(total_bytes * my_leaves / n_leaves)
    peaks = run_intpeak() if (rank == 0 and not args.no_intpeak) else None
    traffic = traffic_db.get(f"merkle_fused_kernel<{args.alg}>:{args.arch}")
    if traffic is not None and world > 1:
        traffic = int(traffic * my_leaves / n_leaves)      # per launch, like `achieved`
    roofline = model_roofline(args.alg, args.arch, leaf_ms, my_leaves, my_bytes, ms_step, hbm_peak, peak_src, peaks, traffic)
    int_pipe = None
    if peaks and "error" not in peaks and args.alg == "sha256":
        ceiling = peaks.get("sha256_fma_regs_gbs") or peaks.get("sha256_regs_gbs")
        int_pipe = {"alu_pipe_utilisation": roofline.get("binding_unit_frac"),
                    "issue_budget_frac": roofline.get("issue_budget_frac"),
                    "model_ops_tops": round(SHA256_OPS_PER_LEAF * my_leaves / (leaf_ms * 1e-3) / 1e12, 3),
                    # the register-only loop of tools/intpeak (same compression, no loads, plain grid): a reference
                    # point, not a bound -- the persistent kernel's scheduling beats it, so no fraction is formed
                    "register_only_loop_gbs": ceiling,
                    "ops_model": "model_ops_tops counts SURVEY.md 8(d)'s 180,600 abstract 32-bit ops per leaf; the kernel "
                                 "issues them as ALU-pipe and FMA-pipe (IMAD) instructions, so utilisation is stated per "
                                 "pipe and against the combined issue budget, never above 1",
                    "microbench": peaks}
    elif peaks:
        int_pipe = {"microbench": peaks}

    # ---- the three schedules of the same hash, for the record (one GPU)
    schedules = None
    if world == 1:
        schedules = {}
        for name, sched in (("fused_single_launch", _native.SCHEDULE_FUSED), ("grid_round1", _native.SCHEDULE_GRID)):
            lib.snt_merkle_schedule(sched)
            l0 = int(lib.snt_debug_launch_count())
            whole.run()
            per_hash = int(lib.snt_debug_launch_count()) - l0
            ms = cuda_time_ms(whole.run, max(5, args.steps // 2), 2)
            assert whole.out_bytes().hex() == root_hex
            schedules[name] = {"ms_per_step": round(ms, 4), "launches_per_hash": per_hash}
        lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT)
        schedules["persistent_default"] = {"ms_per_step": round(ms_step, 4), "launches_per_hash": launches // args.steps}

    # ---- the public call on tensors that already live in HBM: hash_model(cfg, TensorMap(cuda tensors)),
    #      host wall clock per call (cached plan + workspace, launches, 32-byte readback)
    api_resident = None
    cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.from_name(args.alg))
    if world == 1:
        model_r = pkg.TensorMap([(name, t) for name, t in sd])
        for _ in range(2):
            got_r = pkg.hash_model(cfg, model_r).model_digest.data
        assert got_r.hex() == root_hex, "hash_model on resident tensors differs from the planned hasher"
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pkg.hash_model(cfg, model_r)
        dt_r = (time.perf_counter() - t0) / args.steps
        api_resident = {"value": round(total_bytes / dt_r / 1e9, 2), "unit": UNIT, "ms_per_call": round(dt_r * 1e3, 4),
                        "overhead_vs_value_pct": round((dt_r * 1e3 / ms_step - 1) * 100, 2),
                        "api": "hash_model(cfg, TensorMap(CUDA tensors)), host wall clock"}
        del model_r

    # ---- end to end through the public API: pinned host tensors -> hash_model -> root bytes
    e2e = None
    host_pinned = {}
    if not args.no_e2e:
        host_entries = []
        first_leaf = 0
        my_a, my_b = sp.leaf_range(rank)
        for name, t in sd:
            nbytes = t.numel() * 4
            next_leaf = first_leaf + -(-nbytes // BLOCK)
            mine = world == 1 or (first_leaf < my_b and next_leaf > my_a)
            key = (t.data_ptr(), mine)
            if key not in host_pinned:
                if mine:
                    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
                    h.copy_(t.reshape(-1).view(torch.uint8))
                else:
                    h = torch.empty(nbytes, dtype=torch.uint8)   # never read by this rank: not pinned, not touched
                host_pinned[key] = h
            host_entries.append((name, host_pinned[key]))
            first_leaf = next_leaf
        torch.cuda.synchronize()
        model = pkg.TensorMap(host_entries)
        if world == 1:
            def e2e_step():
                return pkg.hash_model(cfg, model).model_digest.data
            h2d = total_bytes
        else:
            def e2e_step():
                return dd.hash_model_sharded(cfg, model, rank, world).model_digest.data
            h2d = dd.staged_bytes(model, BLOCK, *sp.leaf_range(rank))
        got = e2e_step()
        assert got.hex() == root_hex, "e2e digest differs from the device-resident digest"
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        barrier()
        dt = (time.perf_counter() - t0) / args.e2e_steps
        torch.cuda.synchronize()                       # one more, untimed call: the device memory the call itself allocates
        torch.cuda.empty_cache()
        mem_before = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        e2e_step()
        e2e_peak_extra = int(torch.cuda.max_memory_allocated() - mem_before)
        if world > 1:
            t = torch.tensor([dt], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": round(total_bytes / dt / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": 32, "ms_per_step": round(dt * 1e3, 3), "steps": args.e2e_steps,
               "api": "hash_model(HashConfig(MERKLE, IN_PLACE, SHA256, 8192), TensorMap(pinned host tensors))",
               # device memory the call used for the model's bytes: a ring of copy/hash groups, not a copy of the model
               "device_staging_bytes": dict(getattr(sys.modules["paper_2510_00554_b200.model"], "LAST_HOST_STAGING", {})),
               "device_peak_extra_bytes": e2e_peak_extra}
        del model, host_entries

    # ---- the same call on ORDINARY (pageable) host memory -- numpy arrays, what a state dict loaded on the CPU or the
    #      reference's load_model hands over: staged through the pinned ring by copy threads (device.RingWriter)
    e2e_pageable = None
    e2e_file = None
    if host_pinned and world == 1:
        pageable, seen_p = [], {}
        for name, t in sd:
            key = t.data_ptr()
            if key not in seen_p:
                seen_p[key] = np.array(host_pinned[(key, True)].numpy())       # a copy in pageable memory
            pageable.append((name, seen_p[key]))
        model_p = pkg.TensorMap(pageable)
        assert pkg.hash_model(cfg, model_p).model_digest.data.hex() == root_hex, "pageable-host hash_model differs"
        best = None
        for _ in range(2):
            t0 = time.perf_counter()
            pkg.hash_model(cfg, model_p)
            dt_p = time.perf_counter() - t0
            best = dt_p if best is None else min(best, dt_p)
        e2e_pageable = {"value": round(total_bytes / best / 1e9, 3), "unit": UNIT, "ms_per_step": round(best * 1e3, 3),
                        "h2d_bytes_per_step": int(total_bytes), "steps": 2,
                        "api": "hash_model(cfg, TensorMap(numpy arrays in pageable host memory)), host wall clock, best of 2"}
        # ---- and from a checkpoint FILE (the flow of sign-model / verify-model, cli.py:109): load_model(manifest) +
        #      hash_model, the data file in the page cache; the staging threads pread it straight into the pinned ring
        e2e_file = None
        try:
            import shutil
            import tempfile

            shm = "/dev/shm" if os.path.isdir("/dev/shm") and shutil.disk_usage("/dev/shm").free > 3 * total_bytes else None
            with tempfile.TemporaryDirectory(dir=shm) as tmp:
                if shutil.disk_usage(tmp).free > 2 * total_bytes:
                    records, pos = [], 0
                    with open(os.path.join(tmp, "model.bin"), "wb") as f:
                        for name, arr in pageable:
                            f.write(memoryview(arr))
                            records.append({"name": name, "offset": pos, "length": int(arr.nbytes)})
                            pos += int(arr.nbytes)
                    with open(os.path.join(tmp, "model.json"), "w") as f:
                        json.dump({"tensors": records, "data": "model.bin"}, f)
                    best_f = None
                    for _ in range(3):
                        t0 = time.perf_counter()
                        loaded = pkg.load_model(os.path.join(tmp, "model.json"))
                        got_f = pkg.hash_model(cfg, loaded)
                        dt_f = time.perf_counter() - t0
                        del loaded
                        best_f = dt_f if best_f is None else min(best_f, dt_f)
                    assert got_f.model_digest.data.hex() == root_hex, "checkpoint-file hash_model differs"
                    e2e_file = {"value": round(total_bytes / best_f / 1e9, 3), "unit": UNIT, "ms_per_step": round(best_f * 1e3, 3),
                                "steps": 3, "where": "tmpfs" if shm else "temporary directory (page cache)",
                                "api": "load_model(manifest) + hash_model(cfg, model): checkpoint file -> pinned ring -> HBM -> root, "
                                       "host wall clock, best of 3 (reference package, same flow, GPT2-XL: 11.7 s; "
                                       "profiles/r2s4_host_paths.json)"}
        except OSError as exc:
            e2e_file = {"skipped": f"no room for a temporary checkpoint file: {exc}"}
        del model_p, pageable, seen_p

    # ---- CPU baseline on this box's host cores (rank 0, N = 1): the reference package on the SAME bytes,
    #      bit-exactness asserted before anything is printed
    cpu = None
    if ref is not None:
        if host_pinned:                       # the pinned copies made for e2e ARE the D2H copy of the GPU tensors
            host = [(name, host_pinned[(t.data_ptr(), True)].numpy()) for name, t in sd]
        else:
            host = host_views(sd)
        rcfg = reference_cfg(ref, args.alg)
        dt_all, res = timed_cpu(lambda: ref.hash_model(rcfg, reference_model(ref, host), workers=cores))
        assert res.model_digest.data.hex() == root_hex, "GPU root differs from the reference package's root"
        assert res.block_count == n_leaves
        leaves_ref, n_ref, n_ref_tensors = reference_leaf_digests(ref, args.alg, host, 256 << 20)
        dl = dev.DIGEST_LEN[args.alg]
        whole.run()
        assert whole.leaf_bytes()[:n_ref * dl] == leaves_ref, "GPU leaf digests differ from the reference package's"
        # workers = 1 and the sequential (Sigstore/hashlib-style) baseline on a bounded prefix of the same bytes
        prefix, pbytes = [], 0
        for name, arr in host:
            if prefix and pbytes + arr.size > (1 << 30):
                break
            prefix.append((name, arr))
            pbytes += arr.size
        dt_1, _ = timed_cpu(lambda: ref.hash_model(rcfg, reference_model(ref, prefix), workers=1))
        dt_seq, _ = timed_cpu(lambda: ref.sequential_hash(ref.CompressionAlg.from_name(args.alg),
                                                          iter([memoryview(a) for _, a in prefix])))
        cpu = {"value": round(total_bytes / dt_all / 1e9, 4), "unit": UNIT, "cores": cores, "kind": "reference",
               "ms": round(dt_all * 1e3, 1),
               "sample": f"sentinel.hash_model(MERKLE, IN_PLACE, {args.alg}, 8192, workers={cores}) over the D2H copy of "
                         f"the full state dict ({total_bytes / 1e9:.2f} GB), one pass",
               "parity": f"root identical; first {n_ref} leaf digests ({n_ref_tensors} tensors) identical; block_count identical",
               "workers_1_gbs": round(pbytes / dt_1 / 1e9, 4),
               "sequential_hash_gbs": round(pbytes / dt_seq / 1e9, 4),
               "prefix_sample": f"workers=1 and sequential_hash: the first {len(prefix)} tensors ({pbytes / 1e6:.0f} MB)"}
        try:                                   # context: what compiled host code does on the same cores
            from oracle import c_oracle

            tl = c_oracle.TensorList([a for _, a in prefix])
            dt_c, _ = timed_cpu(lambda: c_oracle.inplace_merkle(args.alg, tl, BLOCK, cores), 2)
            cpu["c_port_all_threads_gbs"] = round(pbytes / dt_c / 1e9, 3)
        except Exception:
            pass
        del host, prefix
    host_pinned.clear()

    # ---- the other BASELINE configurations
    configs = None
    if not args.no_configs:
        configs = []
        if world == 1:
            del whole, leaf_hasher, backend
            plan.close()
            del plan, flat, sd
            torch.cuda.empty_cache()
            for arch, alg in (("gpt2", "sha256"), ("gpt2-model", "sha256"), ("bert-large", "blake2b"), ("bert-large", "sha3-256"),
                              ("vgg19", "blake2b"), ("vgg19", "sha3-256")):
                configs.append(gpu_model_config(pkg, dev, shapes, arch, alg, device, args.steps, hbm_peak, peak_src, peaks,
                                                ref, cores, traffic_db))
            configs.append(lattice_model_config(pkg, dev, shapes, "gpt2", device, args.steps, hbm_peak, peak_src, peaks, ref, cores, traffic_db))
            # GPT2-XL: GPU time only (the reference's LATTICE pass over 6.55 GB takes ~20 s; parity at full size is in tests/)
            configs.append(lattice_model_config(pkg, dev, shapes, "gpt2-xl", device, args.steps, hbm_peak, peak_src, peaks, None, cores))
        cifar, _ = dataset_config("cifar10_shaped", "CIFAR10-shaped synthetic dataset (50,000 x 3,072 B uint8, 16 sources) LtHash",
                                  cifar_shaped(np), np, torch, dsm, dev, dd, world, rank, args.steps, args.warmup, barrier,
                                  device, hbm_peak, peak_src, peaks, ref, cores, traffic_db)
        configs.append(cifar)
        pool_arrays = hellaswag_shaped(np)
        pool, (pdig, pcounts) = dataset_config(
            "hellaswag_shaped_pool", "hellaswag-shaped token arrays (40,000 ragged samples, 16 curators) LtHash", pool_arrays,
            np, torch, dsm, dev, dd, world, rank, args.steps, args.warmup, barrier, device, hbm_peak, peak_src, peaks, ref, cores,
            traffic_db)
        if rank == 0:
            # config 5 end to end: one signed bundle per curator + one for the GPT2-XL root, then verification
            n_cur = pool_arrays[5]
            keys = [att.KeyPair.generate() for _ in range(n_cur + 1)]
            t0 = time.perf_counter()
            bundles = []
            for c in range(n_cur):
                stmt = att.Statement([att.Subject(f"pool.json:source:{c}", {"lthash": pdig[64 * c:64 * c + 64].hex()})],
                                     att.DATASET_PREDICATE_TYPE,
                                     {"source_id": c, "sample_count": pcounts[c], "cover_labels": False,
                                      "index_encoding": INDEX_ENCODING})
                bundles.append(att.sign_bundle(stmt, keys[c]))
            bundles.append(att.sign_bundle(att.Statement([att.Subject("gpt2-xl", {"sha256": root_hex})],
                                                         att.MODEL_PREDICATE_TYPE, cfg.predicate()), keys[n_cur]))
            t_sign = time.perf_counter() - t0
            t0 = time.perf_counter()
            verdicts = [att.verify_bundle(bundles[c], {f"pool.json:source:{c}": {"lthash": pdig[64 * c:64 * c + 64].hex()}})
                        for c in range(n_cur)]
            verdicts.append(att.verify_bundle(bundles[n_cur], {"gpt2-xl": {"sha256": root_hex}}))
            t_verify = time.perf_counter() - t0
            assert all(v is att.Verdict.OK for v in verdicts)
            pool["sign_verify"] = {"bundles": n_cur + 1, "ecdsa_sign_ms": round(t_sign * 1e3, 3),
                                   "ecdsa_verify_ms": round(t_verify * 1e3, 3), "all_verified": True,
                                   "model_hash_ms": round(ms_step, 4),
                                   "end_to_end_ms": round(pool["e2e"]["ms_per_step"] + ms_step + (t_sign + t_verify) * 1e3, 3),
                                   "note": "dataset e2e (H2D + LtHash + D2H) + GPT2-XL Merkle root (resident) + host ECDSA P-256"}
        configs.append(pool)

    if rank == 0:
        line = {
            "metric": METRIC if (args.arch, args.alg) == ("gpt2-xl", "sha256")
            else f"{args.arch}_{args.alg}_merkle_inplace_hash_throughput".replace("-", ""),
            "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD if args.arch == "gpt2-xl" and args.alg == "sha256"
                       else f"{args.arch} {args.alg} Merkle in-place hash, block {BLOCK}",
                       "bytes": total_bytes, "leaves": n_leaves, "tensors": n_tensors,
                       "parallelism": f"leaf-range sharding x{world}, shard = 2^{sp.levels} leaves",
                       "l2_policy": "inputs (6.55 GB per pass) larger than the 126 MB L2",
                       "root": root_hex, "root_matches_pinned": PINNED_ROOTS.get((args.arch, args.alg), root_hex) == root_hex},
            **({"debug": "ranks share GPU 0 over gloo; not a measurement"} if same_gpu else {}),
            "e2e": e2e, "e2e_pageable_host": e2e_pageable, "e2e_checkpoint_file": e2e_file, "api_device_resident": api_resident, "gpu_launches": launches, "clocks": clocks.summary(),
            "roofline": roofline, "int_pipe": int_pipe, "cpu_baseline": cpu, "schedules": schedules, "configs": configs,
            # kept for readers of round 1's line: the CIFAR10-shaped entry of `configs`
            "dataset": next((c for c in (configs or []) if c.get("metric", "").startswith("cifar10")), None),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- launch

def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int:
    """`--gpus N` outside torchrun: start N ranks of this script, one per GPU, over NCCL."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "n_gpus": args.gpus, "unavailable":
                          f"--gpus {args.gpus} needs {args.gpus} CUDA devices, this box has {have}"}), flush=True)
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, this box has {have}", file=sys.stderr)
        return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")           # communicator / rank lines on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    else:
        if int(os.environ.get("WORLD_SIZE", "1")) > 1:
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        run_ours(args)


if __name__ == "__main__":
    main()
