"""The multi-rank shard-and-combine path on real CUDA kernels.

* Several ranks share the one GPU of the test box and talk over gloo (NCCL refuses two ranks on one device):
  everything but the NCCL call itself is the product path -- per-rank leaf ranges, shard roots written into the
  all-gather slot, index-compacted receive buffer, top reduce; one all-reduce of the lattice state.
* A one-rank NCCL group runs the exact NCCL calls of that path on the device (uint8 all_gather_into_tensor of
  shard-root slots, int64 all_reduce of the lattice state).
* A two-rank NCCL test runs wherever two devices exist (skipped on the one-GPU box).
"""

import os
import socket

import numpy as np
import pytest

import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, sizes, q, ckpt=None):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_00554_b200 as pkg
        from paper_2510_00554_b200 import dataset as dsm, distributed as dd

        torch.cuda.set_device(0)
        tensors = inputs.model_tensors(91, sizes)
        out = {}
        for alg in ("sha256", "blake2b", "sha3-256"):
            cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.from_name(alg))
            # odd ranks hold the model on the GPU, even ranks as host bytes
            entries = [(f"t{i}", torch.frombuffer(bytearray(t), dtype=torch.uint8).cuda() if (rank % 2 and t) else t)
                       for i, t in enumerate(tensors)]
            out[alg] = dd.hash_model_sharded(cfg, pkg.TensorMap(entries), rank, world).model_digest.data.hex()
        if ckpt is not None:
            # the same model as a checkpoint FILE: every rank preads only the tensors that own leaves of its shard run
            loaded = pkg.load_model(ckpt)
            cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.SHA256)
            out["file"] = dd.hash_model_sharded(cfg, loaded, rank, world).model_digest.data.hex()
            out["file_copied_to_host"] = loaded.entries[0][1].file._whole is not None

        n, declared = 999, [2, 3, 5, 7]
        rng = np.random.default_rng(17)
        data = rng.integers(0, 256, size=(n, 96), dtype=np.uint8)
        ids = np.arange(n, dtype=np.int64) * 3 + 1
        src = np.array(declared)[rng.integers(0, len(declared), size=n)]
        a, b = dd.sample_ranges(n, world)[rank]
        h = dsm.StreamingDatasetHasher(declared)
        for s in range(a, b, 100):
            e = min(b, s + 100)
            h.update(torch.from_numpy(data[s:e]).cuda(), torch.from_numpy(ids[s:e]), torch.from_numpy(src[s:e]))
        h.allreduce()
        out["lattice"] = {k: (v[0].data.hex(), v[1]) for k, v in h.finalize().items()}
        q.put((rank, out))
    except Exception as exc:                     # surface the failure instead of leaving the peers in a collective
        q.put((rank, {"error": repr(exc)}))
        os._exit(1)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_sharing_the_gpu_reproduce_single_gpu_digests(world, porc, tmp_path):
    import torch.multiprocessing as mp

    import paper_2510_00554_b200 as pkg

    sizes = [8192 * 1500 + 77, 100, 0, 8192 * 2100, 31, 8192 * 900 + 4096, 5000]     # 4,501+ leaves: 5 shards of 1024
    tensors = inputs.model_tensors(91, sizes)
    pkg.save_model(pkg.TensorMap([(f"t{i}", t) for i, t in enumerate(tensors)]), tmp_path / "ckpt.json")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sizes, q, str(tmp_path / "ckpt.json"))) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(world):
            rank, out = q.get(timeout=120)
            assert "error" not in out, (rank, out)
            results[rank] = out
        for p in procs:
            p.join(60)
            assert p.exitcode == 0
    finally:
        for p in procs:                      # a failed rank leaves its peers inside a collective: do not wait for them
            if p.is_alive():
                p.kill()

    n, declared = 999, [2, 3, 5, 7]
    rng = np.random.default_rng(17)
    data = rng.integers(0, 256, size=(n, 96), dtype=np.uint8)
    ids = np.arange(n, dtype=np.int64) * 3 + 1
    src = np.array(declared)[rng.integers(0, len(declared), size=n)]
    want_lat = porc.dataset_digests([(int(ids[i]), int(src[i]), b"", data[i].tobytes()) for i in range(n)], declared=declared)
    for rank in range(world):
        got = results[rank]
        for alg in ("sha256", "blake2b", "sha3-256"):
            assert got[alg] == porc.inplace_merkle(alg, tensors, 8192).hex(), (rank, alg)
        assert got["file"] == porc.inplace_merkle("sha256", tensors, 8192).hex(), rank
        assert got["file_copied_to_host"] is False, rank
        assert got["lattice"] == {k: (v[0].hex(), v[1]) for k, v in want_lat.items()}, rank


# ---- NCCL ---------------------------------------------------------------------------------------
# The product's collectives are NCCL calls on device tensors. The test box has one GPU and NCCL refuses
# two ranks on one device, so (a) a ONE-rank NCCL group runs the exact calls of the multi-GPU path
# (all_gather_into_tensor of uint8 shard-root slots, one int64 all_reduce of the lattice state) with
# ``always_gather`` forcing the exchange, and (b) a real two-rank test runs wherever two devices exist.

def _nccl_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        from paper_2510_00554_b200 import device as dev, distributed as dd

        sizes = [8192 * 1500 + 77, 100, 0, 8192 * 2100, 31, 8192 * 900 + 4096, 5000]
        tensors = inputs.model_tensors(91, sizes)
        flat = [torch.frombuffer(bytearray(t), dtype=torch.uint8).cuda() if t else torch.empty(0, dtype=torch.uint8, device="cuda")
                for t in tensors]
        plan = dev.ModelPlan(flat, 8192)
        out = {}
        for alg in ("sha256", "blake2b", "sha3-256"):
            backend = dd.CudaBackend(plan, alg)
            sp = dd.plan_shards(plan.leaf_count, world)
            roots = [dd.sharded_merkle_root(backend, sp, rank, world, always_gather=True) for _ in range(3)]
            torch.cuda.synchronize()
            out[alg] = backend.to_bytes(roots[-1]).hex()
        n, n_src = 4000, 5
        rng = np.random.default_rng(3)
        data = torch.from_numpy(rng.integers(0, 256, size=(n, 200), dtype=np.uint8)).cuda()
        ids = torch.arange(n, dtype=torch.int64)
        src = torch.from_numpy(rng.integers(0, n_src, size=n))
        from paper_2510_00554_b200 import dataset as dsm

        a, b = dd.sample_ranges(n, world)[rank]
        h = dsm.StreamingDatasetHasher(range(n_src))
        h.update(data[a:b], ids[a:b], src[a:b])
        h.allreduce()                                      # one NCCL all_reduce of the int64 state
        out["lattice"] = {k: (v[0].data.hex(), v[1]) for k, v in h.finalize().items()}
        q.put((rank, out))
    except Exception as exc:
        q.put((rank, {"error": repr(exc)}))
        os._exit(1)
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _run_nccl(world, porc):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(world):
            rank, out = q.get(timeout=300)
            assert "error" not in out, (rank, out)
            results[rank] = out
        for p in procs:
            p.join(60)
            assert p.exitcode == 0
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
    sizes = [8192 * 1500 + 77, 100, 0, 8192 * 2100, 31, 8192 * 900 + 4096, 5000]
    tensors = inputs.model_tensors(91, sizes)
    n, n_src = 4000, 5
    rng = np.random.default_rng(3)
    data = rng.integers(0, 256, size=(n, 200), dtype=np.uint8)
    src = rng.integers(0, n_src, size=n)
    want_lat = porc.dataset_digests([(i, int(src[i]), b"", data[i].tobytes()) for i in range(n)], declared=range(n_src))
    for rank in range(world):
        for alg in ("sha256", "blake2b", "sha3-256"):
            assert results[rank][alg] == porc.inplace_merkle(alg, tensors, 8192).hex(), (rank, alg)
        assert results[rank]["lattice"] == {k: (v[0].hex(), v[1]) for k, v in want_lat.items()}, rank


def test_nccl_collectives_of_the_shard_path_one_rank_group(porc):
    _run_nccl(1, porc)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two CUDA devices (the test box has one)")
def test_nccl_two_gpus_reproduce_single_gpu_digests(porc):
    _run_nccl(2, porc)
