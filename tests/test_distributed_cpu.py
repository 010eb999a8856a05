"""World-size-2 and -3 runs of the shard-and-combine layer over gloo (CPU).

The hashing backend is the checker (the Python oracle) -- this exercises the
partitioning, the all-gather of shard roots, the top reduce and the lattice
all-reduce exactly as the NCCL path drives them; the CUDA backend itself is
covered by tests/test_gpu_parity.py::test_shard_roots_recombine_to_whole_root.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleBackend:
    """Same interface as distributed.CudaBackend, hashing with the CPU oracle (tests only)."""

    def __init__(self, alg, leaves: bytes, n: int):
        from oracle import sentinel_oracle as orc

        self.orc, self.alg, self.leaves, self.n = orc, alg, leaves, n
        self.dlen = orc.DIGEST_LEN[alg]
        self.device = torch.device("cpu")

    def shard_roots(self, begin, end, levels):
        dl = self.dlen
        out = self.orc.reduce_levels_forced(self.alg, self.leaves[begin * dl:end * dl], begin, end - begin, self.n, levels)
        return torch.frombuffer(bytearray(out), dtype=torch.uint8)

    def root_of(self, nodes, count):
        return torch.frombuffer(bytearray(self.orc.merkle_root(self.alg, nodes.numpy().tobytes(), count)), dtype=torch.uint8)


def _merkle_worker(rank, world, port, alg, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sentinel_oracle as orc
        from paper_2510_00554_b200 import distributed as dd

        leaves = inputs.seeded_bytes(500 + n, n * orc.DIGEST_LEN[alg])
        backend = OracleBackend(alg, leaves, n)
        for levels in (None, 0, 1, 3):
            if levels is not None and levels > (0 if n <= 1 else (n - 1).bit_length()):
                continue        # a shard may not be deeper than the tree itself
            sp = dd.plan_shards(n, world, levels)
            root = dd.sharded_merkle_root(backend, sp, rank, world).numpy().tobytes()
            q.put((rank, n, levels, root == orc.merkle_root(alg, leaves, n)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_merkle_root_equals_reference_root(world):
    ctx = mp.get_context("spawn")
    for alg, n in (("sha256", 1), ("sha256", 2), ("sha256", 37), ("blake2b", 1000), ("sha3-256", 5000)):
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_merkle_worker, args=(r, world, port, alg, n, q)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        results = []
        while not q.empty():
            results.append(q.get())
        assert results and all(ok for *_, ok in results), (alg, n, results)
        assert {r for r, *_ in results} == set(range(world))


def _lattice_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sentinel_oracle as orc
        from paper_2510_00554_b200 import distributed as dd

        spec = inputs.DATASET_CASES[2]
        samples = inputs.dataset_samples(**spec)
        sources = sorted(spec["declared"])
        a, b = dd.sample_ranges(len(samples), world)[rank]
        # per-rank partial sums in the layout LatticeAccumulator.state has: lanes | counts | status, all u64
        n_src = len(sources)
        state = np.zeros(n_src * 33 + 1, dtype=np.uint64)
        acc, counts = state[:n_src * 32].reshape(n_src, 32), state[n_src * 32:n_src * 33]
        for sid, src, _label, data in samples[a:b]:
            lanes = np.frombuffer(orc.sample_digest(sid, data), dtype="<u2").astype(np.uint64)
            acc[sources.index(src)] += lanes
            counts[sources.index(src)] += 1
        acc[0, 0] += np.uint64(0xFFFFFFFFFFFF0000)  # force a wrap modulo 2^64 in the all-reduce on one lane
        state[-1] = 2 if rank == 1 else 0           # rank 1 skipped two samples of an undeclared source
        t_state = torch.from_numpy(state.view(np.int64).copy())
        dd.allreduce_lattice(t_state)
        summed = t_state.numpy().view(np.uint64)
        assert int(summed[-1]) == 2
        got = (summed[:n_src * 32].reshape(n_src, 32) & np.uint64(0xFFFF)).astype("<u2")
        want = orc.dataset_digests(samples, declared=sources)
        ok = all(got[i].tobytes() == want[s][0] and int(summed[n_src * 32 + i]) == want[s][1]
                 for i, s in enumerate(sources))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_lattice_allreduce_world2_matches_single_pass():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lattice_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    results = [q.get() for _ in range(2)]
    assert all(ok for _, ok in results)
