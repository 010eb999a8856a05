"""Multi-GPU shard-and-combine layer (one process per GPU, torch.distributed).

Merkle: the reference tree (merkle.py:117-165) is node(j, i) = H(node(j-1, 2i) ||
(node(j-1, 2i+1) or zeros)) for i < ceil(N / 2^j). Cutting the leaves into
shards of 2^k leaves and reducing every shard EXACTLY k levels (zero padding on
odd counts, never stopping early at one digest) yields the level-k nodes of that
very tree; the ceil(N / 2^k) shard roots are then reduced by the ordinary rule.
Each rank owns a contiguous run of whole shards; the only exchange is one
all-gather of shard roots (a few KB).

LtHash: lane sums are commutative (dataset.py:67-71), so each rank accumulates a
contiguous sample range into ``n_sources x 32`` widened lanes and one sum all-reduce
combines them (widened to u64 because NCCL has no u16 type and so that lanes, counts and status
share one array; exact modulo 2^16).

The hashing itself is injected as a ``backend`` (CUDA in the product, see
``CudaBackend``); the partition / gather / top-reduce logic here is plain host
code, so the tests drive it over ``gloo`` with a checker backend.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from .errors import InvalidInput
from .workers import chunk_ranges

DEFAULT_SHARD_LEVELS = 10   # 1024 leaves = 8 MiB of tensor bytes per shard


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def choose_shard_levels(n_leaves: int, world: int, max_levels: int = DEFAULT_SHARD_LEVELS) -> int:
    """Largest k <= max_levels with 2^k < N and at least 4 shards per rank (when N allows).

    Small shards balance better: N = 799,954 at k = 10 gives 782 shards, 97 or 98
    per rank on 8 GPUs, whereas rounding ceil(N / G) up to a power of two would
    leave one GPU idle.
    """
    k = max_levels
    while k > 0 and ((1 << k) >= n_leaves or ceil_div(n_leaves, 1 << k) < 4 * world):
        k -= 1
    return k


@dataclass(frozen=True)
class ShardPlan:
    n_leaves: int
    levels: int                              # k: every shard is reduced exactly k levels
    n_shards: int                            # ceil(N / 2^k) = number of level-k nodes
    shard_ranges: Tuple[Tuple[int, int], ...]  # per rank: [first_shard, last_shard)

    def leaf_range(self, rank: int) -> Tuple[int, int]:
        a, b = self.shard_ranges[rank]
        return a << self.levels, min(b << self.levels, self.n_leaves)

    def shard_count(self, rank: int) -> int:
        a, b = self.shard_ranges[rank]
        return b - a


def plan_shards(n_leaves: int, world: int, levels: Optional[int] = None) -> ShardPlan:
    if n_leaves < 1 or world < 1:
        raise InvalidInput("need at least one leaf and one rank")
    k = choose_shard_levels(n_leaves, world) if levels is None else levels
    n_shards = ceil_div(n_leaves, 1 << k)
    ranges = chunk_ranges(n_shards, world)
    ranges += [(n_shards, n_shards)] * (world - len(ranges))      # ranks beyond the shard count idle
    return ShardPlan(n_leaves, k, n_shards, tuple(ranges))


class CudaBackend:
    """Hashing backend of the product: the CUDA kernels through the C ABI."""

    def __init__(self, plan, alg: str):
        from . import device as _dev

        self._dev = _dev
        self.plan = plan
        self.alg = alg
        self.dlen = _dev.DIGEST_LEN[alg]
        self.device = _dev.require_cuda()
        self._hashers = {}

    def shard_roots(self, leaf_begin: int, leaf_end: int, levels: int) -> torch.Tensor:
        """Level-``levels`` nodes of the leaf range, as a flat uint8 device tensor (no sync)."""
        key = (leaf_begin, leaf_end, levels)
        h = self._hashers.get(key)
        if h is None:
            h = self._dev.MerkleModelHasher(self.plan, self.alg, leaf_begin, leaf_end, levels)
            self._hashers[key] = h
        h.run()
        return h.out

    def shard_roots_padded(self, leaf_begin: int, leaf_end: int, levels: int, slots: int) -> torch.Tensor:
        """Same, written at the front of a zero-filled buffer of ``slots`` digests (an all-gather slot)."""
        key = (leaf_begin, leaf_end, levels, slots)
        h = self._hashers.get(key)
        if h is None:
            h = self._dev.MerkleModelHasher(self.plan, self.alg, leaf_begin, leaf_end, levels, out_capacity=slots)
            self._hashers[key] = h
        h.run()
        return h.out_padded

    def gather_buffers(self, shard_plan: "ShardPlan", world: int, widest: int):
        """Persistent buffers of the exchange: the all-gather's receive buffer, the row index that compacts
        its slots (rank r's first ``shard_count(r)`` rows) into shard order, and the compacted node array."""
        key = ("gather", shard_plan.n_shards, world, widest)
        got = self._hashers.get(key)
        if got is None:
            recv = torch.empty(world * widest * self.dlen, dtype=torch.uint8, device=self.device)
            rows = [r * widest + i for r in range(world) for i in range(shard_plan.shard_count(r))]
            nodes = torch.empty(len(rows), self.dlen, dtype=torch.uint8, device=self.device)
            got = (recv, torch.tensor(rows, dtype=torch.int64, device=self.device), nodes)
            self._hashers[key] = got
        return got

    def empty_slot(self, slots: int) -> torch.Tensor:
        """The all-gather contribution of a rank that owns no shard (more ranks than shards)."""
        key = ("empty", slots)
        if key not in self._hashers:
            self._hashers[key] = torch.zeros(slots * self.dlen, dtype=torch.uint8, device=self.device)
        return self._hashers[key]

    def root_of(self, nodes: torch.Tensor, count: int) -> torch.Tensor:
        """Ordinary tree rule over ``count`` level-k nodes; workspace and root buffer are kept per count."""
        key = ("top", count)
        got = self._hashers.get(key)
        if got is None:
            wb = self._dev.merkle_work_bytes(self.alg, count)
            got = (torch.zeros(max(wb, 16), dtype=torch.uint8, device=self.device), wb,
                   torch.empty(self.dlen, dtype=torch.uint8, device=self.device))
            self._hashers[key] = got
        work, wb, root = got
        return self._dev.merkle_root_into(self.alg, nodes, count, work, wb, root)

    def to_bytes(self, t: torch.Tensor) -> bytes:
        return t.cpu().numpy().tobytes()


def _needs_host_staging(t: torch.Tensor, group=None) -> bool:
    """gloo cannot move CUDA tensors for every collective: stage through the host then.

    NCCL (the production backend) takes the device tensors directly; this only matters for
    debugging several ranks on one GPU and for CPU-only test runs.
    """
    return t.device.type == "cuda" and dist.get_backend(group) == "gloo"


def sharded_merkle_root(backend, shard_plan: ShardPlan, rank: int, world: int, group=None,
                        always_gather: bool = False) -> torch.Tensor:
    """This rank's shard roots -> all-gather -> top reduce. Returns the root (flat uint8 tensor).

    Every rank returns the same root. With ``world == 1`` no collective is issued unless
    ``always_gather`` asks for the exchange anyway (a one-rank NCCL group exercises the very calls the
    multi-GPU path makes). Nothing is allocated per call on the product path: send slot, receive
    buffer, compaction index, node array, top-reduce workspace and root live in the backend.
    """
    dlen = backend.dlen
    begin, end = shard_plan.leaf_range(rank)
    mine = shard_plan.shard_count(rank)
    exchange = world > 1 or always_gather
    fused_slot = exchange and hasattr(backend, "shard_roots_padded")
    local = backend.shard_roots(begin, end, shard_plan.levels) if (mine and not fused_slot) else None
    if not exchange:
        if shard_plan.n_shards == 1:
            return local                               # already the single level-k node = the root
        nodes = local
    elif fused_slot:
        # product path (NCCL): the leaf + shard-reduce launches write straight into the all-gather slot,
        # the receive buffer is persistent, one index_select puts the roots in shard order
        widest = max(shard_plan.shard_count(r) for r in range(world))
        send = backend.shard_roots_padded(begin, end, shard_plan.levels, widest) if mine else backend.empty_slot(widest)
        recv, rows, nodes2d = backend.gather_buffers(shard_plan, world, widest)
        if _needs_host_staging(send, group):           # debugging over gloo: same buffers, staged through the host
            host = torch.empty(recv.numel(), dtype=torch.uint8)
            dist.all_gather_into_tensor(host, send.cpu(), group=group)
            recv.copy_(host)
        else:
            dist.all_gather_into_tensor(recv, send, group=group)
        torch.index_select(recv.view(world * widest, dlen), 0, rows, out=nodes2d)
        nodes = nodes2d.view(-1)
        if shard_plan.n_shards == 1:
            return nodes
    else:
        widest = max(shard_plan.shard_count(r) for r in range(world))
        send = torch.zeros(widest * dlen, dtype=torch.uint8, device=backend.device)
        if mine:
            send[:mine * dlen].copy_(local[:mine * dlen])
        if _needs_host_staging(send, group):
            host = torch.empty(world * widest * dlen, dtype=torch.uint8)
            dist.all_gather_into_tensor(host, send.cpu(), group=group)
            recv = host.to(backend.device)
        else:
            recv = torch.empty(world * widest * dlen, dtype=torch.uint8, device=backend.device)
            dist.all_gather_into_tensor(recv, send, group=group)
        parts = [recv[r * widest * dlen:(r * widest + shard_plan.shard_count(r)) * dlen] for r in range(world)]
        nodes = torch.cat(parts)
        if shard_plan.n_shards == 1:
            return nodes
    return backend.root_of(nodes, shard_plan.n_shards)


def _first_leaves(sizes: Sequence[int], block_size: int) -> List[int]:
    first, k = [], 0
    for s in sizes:
        first.append(k)
        k += ceil_div(s, block_size)
    first.append(k)
    return first


def staged_bytes(model, block_size: int, leaf_begin: int, leaf_end: int) -> int:
    """Bytes of the tensors that own at least one leaf of [leaf_begin, leaf_end)."""
    from .model import buffer_nbytes

    sizes = [buffer_nbytes(buf) for _, buf in model.entries]
    first = _first_leaves(sizes, block_size)
    return sum(s for i, s in enumerate(sizes) if first[i] < leaf_end and first[i + 1] > leaf_begin)


def hash_model_sharded(cfg, model, rank: int, world: int, group=None):
    """In-place Merkle hash of one model across ``world`` GPUs (public multi-GPU entry point).

    Every rank passes the same ``TensorMap``; a rank copies to its GPU only the
    tensors that own leaves of its shard run (tensors already on the GPU are used
    in place), hashes them, and all ranks combine the shard roots into the same
    root ``hash_model`` returns on one GPU.
    """
    from . import device as _dev
    from .compression import Digest
    from .model import Construction, ModelDigestResult, Strategy, _require_nonempty, buffer_nbytes

    cfg.validate()
    if cfg.construction is not Construction.MERKLE or cfg.strategy is not Strategy.IN_PLACE:
        raise InvalidInput("hash_model_sharded covers the in-place Merkle configuration")
    _require_nonempty(model)
    dev = _dev.require_cuda()
    bs = cfg.block_size
    sizes = [buffer_nbytes(buf) for _, buf in model.entries]
    first = _first_leaves(sizes, bs)
    sp = plan_shards(first[-1], world)
    a, b = sp.leaf_range(rank)
    # tensors this rank reads (they own leaves of its range) or that already sit on its GPU are described by
    # their real addresses; the host ones among them are staged together (pinned ring + one device arena);
    # every other entry keeps its true size but points at a placeholder that no leaf of this rank touches
    import numpy as np

    placeholder = torch.zeros(16, dtype=torch.uint8, device=dev)
    wanted = [i for i, (_, buf) in enumerate(model.entries)
              if (first[i] < b and first[i + 1] > a) or (isinstance(buf, torch.Tensor) and buf.device.type == "cuda")]
    # file-backed tensors (load_model): this rank reads only the ranges it owns, file -> pinned ring -> its GPU
    from .model import FileTensor

    w_bufs = [model.entries[i][1] for i in wanted]
    lazy = [j for j, buf in enumerate(w_bufs) if isinstance(buf, FileTensor) and buf.file._whole is None]
    by_file = {}
    for j in lazy:
        by_file.setdefault(id(w_bufs[j].file), []).append(j)
    for js in by_file.values():
        got = _dev.file_ranges_to_device(w_bufs[js[0]].file.fd, [(w_bufs[j].offset, w_bufs[j].nbytes) for j in js], dev)
        for j, t in zip(js, got):
            w_bufs[j] = t
    keep, w_ptrs, _ = _dev.device_spans(w_bufs, dev)
    ptrs = np.full(len(sizes), placeholder.data_ptr(), dtype=np.uint64)
    ptrs[np.asarray(wanted, dtype=np.int64)] = w_ptrs[:len(wanted)]
    ptrs[np.asarray(sizes) == 0] = 0
    plan = _dev.ModelPlan.from_spans([keep, placeholder], ptrs, np.asarray(sizes, dtype=np.uint64), bs, count=len(sizes))
    try:
        backend = CudaBackend(plan, cfg.alg.value)
        root = sharded_merkle_root(backend, sp, rank, world, group)
        return ModelDigestResult(Digest(cfg.alg, backend.to_bytes(root)), cfg, first[-1])
    finally:
        plan.close()


def sample_ranges(n_samples: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous sample ranges per rank (empty for ranks beyond the sample count)."""
    ranges = chunk_ranges(n_samples, world)
    return ranges + [(n_samples, n_samples)] * (world - len(ranges))


def allreduce_lattice(state: torch.Tensor, group=None) -> None:
    """Sum the per-rank LtHash accumulators over all ranks, in place, with ONE all-reduce.

    ``state`` is ``LatticeAccumulator.state``: lanes, counts and the status word in one int64 array
    (the bit patterns of u64 sums). A lane sum modulo 2^64 is still exact modulo 2^16, counts add,
    and a summed status word is non-zero exactly when some rank skipped a sample -- so one
    ``all_reduce(SUM)`` of ``n_sources * 33 + 1`` words carries everything and there is nothing to
    pack or unpack around it. The message is a few KB: latency bound, which is why it is one
    collective and not three.
    """
    if _needs_host_staging(state, group):           # debugging over gloo with ranks sharing a GPU
        host = state.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        state.copy_(host)
    else:
        dist.all_reduce(state, op=dist.ReduceOp.SUM, group=group)
