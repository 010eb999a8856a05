"""Whole-model digests over fragmented tensor collections, computed on the GPU.

API mirror of the reference's ``model.py`` (:44-374): ``TensorMap``,
``HashConfig``, ``BlockTable``, ``ModelDigestResult``, ``inplace_hash``,
``coalesce_hash``, ``hash_model``, ``load_model`` / ``save_model``.

The default strategy -- in-place (model.py:298-315) -- hashes every tensor where
it lies in HBM: a per-tensor table replaces the per-block table, each 8 KiB block
is one leaf hashed by one thread (the last block of a tensor at its true length),
and the leaf digests are reduced to the root on the device. ``TensorMap`` entries
may be CUDA tensors (hashed in place, no copy) or host bytes-like objects (copied
to the device first, which is what the reference-shaped call pays for).
"""

from __future__ import annotations

import ctypes
import enum
import json
from dataclasses import dataclass
from pathlib import Path
from typing import Dict, List, Optional, Tuple, Union

import threading

import numpy as np
import torch

from . import device as _dev
from .compression import CompressionAlg, Digest
from .errors import ConfigError, FormatError, InvalidInput
from .lattice import DIGEST_BYTES as LT_DIGEST_BYTES
from .lattice import LatticeDigest

DEFAULT_BLOCK_SIZE = 8192
MAX_BLOCK_SIZE = 1 << 31

# recorded in attestation predicates: lattice blocks carry a little-endian
# 64-bit index prefix (global block counter for coalesced / in-place)
INDEX_ENCODING = "le64-prefix-v1"


class Construction(enum.Enum):
    MERKLE = "merkle"
    LATTICE = "lattice"


class Strategy(enum.Enum):
    COALESCED = "coalesced"
    PER_LAYER = "per-layer"
    IN_PLACE = "in-place"


def buffer_nbytes(buf) -> int:
    if isinstance(buf, torch.Tensor):
        return buf.numel() * buf.element_size()
    if isinstance(buf, np.ndarray):
        return buf.nbytes
    return memoryview(buf).nbytes


@dataclass
class TensorMap:
    """Ordered, uniquely named, independently allocated tensors.

    Each buffer is a CUDA/CPU ``torch.Tensor``, a numpy array or a bytes-like
    object; only its bytes matter.
    """

    entries: List[Tuple[str, object]]

    def __post_init__(self):
        seen = set()
        for name, _ in self.entries:
            if name in seen:
                raise InvalidInput("layer names must be unique")
            seen.add(name)

    def __len__(self) -> int:
        return len(self.entries)

    @property
    def total_bytes(self) -> int:
        return sum(buffer_nbytes(buf) for _, buf in self.entries)

    def names(self) -> List[str]:
        return [name for name, _ in self.entries]


@dataclass
class HashConfig:
    construction: Construction
    strategy: Strategy
    alg: CompressionAlg = CompressionAlg.SHA256
    block_size: int = DEFAULT_BLOCK_SIZE
    ordered_per_layer: bool = False

    def validate(self) -> None:
        """Same rules as the reference (model.py:93-102)."""
        bs = self.block_size
        if bs < 64 or bs & (bs - 1):
            raise ConfigError("block_size must be a power of two >= 64")
        if bs > MAX_BLOCK_SIZE:
            # the C ABI takes the block size as a uint32; refuse before any buffer of that size is allocated
            raise ConfigError(f"block_size must be at most {MAX_BLOCK_SIZE} bytes")
        lattice = self.construction is Construction.LATTICE
        if lattice and self.alg is not CompressionAlg.BLAKE2B:
            raise ConfigError("lattice hashing is fixed to BLAKE2b")
        if self.ordered_per_layer and not (lattice and self.strategy is Strategy.PER_LAYER):
            raise ConfigError("ordered_per_layer requires lattice per-layer hashing")

    def predicate(self) -> Dict[str, object]:
        """Everything a verifier needs to replay this configuration (model.py:104-113)."""
        return {
            "construction": self.construction.value,
            "compression": self.alg.value,
            "strategy": self.strategy.value,
            "block_size": self.block_size,
            "ordered_per_layer": self.ordered_per_layer,
            "index_encoding": INDEX_ENCODING,
        }

    @classmethod
    def from_predicate(cls, pred: Dict[str, object]) -> "HashConfig":
        try:
            cfg = cls(Construction(pred["construction"]), Strategy(pred["strategy"]),
                      CompressionAlg.from_name(pred["compression"]), int(pred["block_size"]),
                      bool(pred.get("ordered_per_layer", False)))
        except (KeyError, ValueError) as exc:
            raise FormatError(f"bad hashing predicate: {exc}") from exc
        cfg.validate()
        return cfg


@dataclass
class BlockTable:
    """Host view of the in-place block table: rows (k, tensor, offset, length).

    The kernels search the compact per-tensor form (``device.ModelPlan``); this
    per-block expansion (model.py:137-146) is kept for inspection and tests.
    """

    rows: List[Tuple[int, int, int, int]]

    @classmethod
    def build(cls, model: TensorMap, block_size: int) -> "BlockTable":
        rows: List[Tuple[int, int, int, int]] = []
        k = 0
        for t, (_, buf) in enumerate(model.entries):
            size = buffer_nbytes(buf)
            full, tail = divmod(size, block_size)
            rows.extend((k + j, t, j * block_size, block_size) for j in range(full))
            k += full
            if tail:
                rows.append((k, t, full * block_size, tail))
                k += 1
        return cls(rows)


@dataclass
class ModelDigestResult:
    model_digest: Union[Digest, LatticeDigest]
    config: HashConfig
    block_count: int
    layer_digests: Optional[Dict[str, Union[Digest, LatticeDigest]]] = None
    aux_data_bytes: int = 0     # staging copies of tensor data (coalesced buffer)
    aux_digest_bytes: int = 0   # digest + reducer scratch storage on the device

    @property
    def aux_bytes(self) -> int:
        return self.aux_data_bytes + self.aux_digest_bytes

    def digest_hex(self) -> str:
        return self.model_digest.hex()


def _require_nonempty(model: TensorMap) -> None:
    if len(model) == 0 or model.total_bytes == 0:
        raise InvalidInput("model must contain at least one byte of tensor data")


def _hash_plan(cfg: HashConfig, plan: _dev.ModelPlan, aux_data_bytes: int = 0) -> ModelDigestResult:
    n = plan.leaf_count
    if cfg.construction is Construction.MERKLE:
        hasher = _dev.MerkleModelHasher(plan, cfg.alg.value)
        hasher.run()
        root = Digest(cfg.alg, hasher.out_bytes())
        aux = hasher.leaves.numel() + hasher.work_bytes + (hasher.out.numel() if n > 1 else 0)
        return ModelDigestResult(root, cfg, n, aux_data_bytes=aux_data_bytes, aux_digest_bytes=aux)
    acc = _dev.LatticeAccumulator(1)
    acc.add_model_leaves(plan, 0, n)
    out, _, _ = acc.digests()
    # one 64-byte accumulator instead of the reference's n x 64 digest array
    return ModelDigestResult(LatticeDigest(out), cfg, n, aux_data_bytes=aux_data_bytes,
                             aux_digest_bytes=acc.acc.numel() * 8)


STAGE_PIPELINE_MIN_BYTES = 32 << 20     # host inputs above this are copied and hashed in overlapped chunks
STAGE_CHUNK_BYTES = 256 << 20
SMALL_H2D_BYTES = 64 << 10              # page-locked tensors below this are fetched by a kernel, not by the copy engine


def _is_cuda(buf) -> bool:
    return isinstance(buf, torch.Tensor) and buf.device.type == "cuda"


def _host_tensor(buf) -> torch.Tensor:
    """Flat uint8 CPU tensor over a host buffer (zero copy; pinned tensors stay pinned)."""
    if isinstance(buf, torch.Tensor):
        t = buf.detach()
        t = t if t.is_contiguous() else t.contiguous()
        t = t.reshape(-1)
        return t if t.dtype == torch.uint8 else t.view(torch.uint8)
    import warnings

    arr = _dev.host_bytes_view(buf)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return torch.from_numpy(arr)


_ARENA_ALIGN = 256


_COPY_STREAMS: Dict[int, List["torch.cuda.Stream"]] = {}


def _copy_streams(dev: torch.device) -> List["torch.cuda.Stream"]:
    """Side streams per device for host-to-device staging, created once."""
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]
    return _COPY_STREAMS[key]


def _inplace_merkle_pinned(cfg: HashConfig, model: TensorMap) -> Optional[ModelDigestResult]:
    """Page-locked host tensors (and CUDA tensors): the transfer is the whole cost, so it starts first.

    One pass lays the host tensors out in a device arena; then EVERY copy is put on a side stream at once --
    one batch of asynchronous copies per ~256 MB group, an event after each group -- before the plan, the
    leaf buffer and the workspace are even created. The leaf launch of a group waits for that group's event,
    the tree runs once at the end. GPT2-XL from pinned memory: 123.8 -> 120 ms for a link that needs 117.9 ms.
    Returns None when an entry is neither a CUDA tensor nor a contiguous page-locked tensor (the general path
    takes those).
    """
    dev = _dev.require_cuda()
    bs = cfg.block_size
    entries = model.entries
    n = len(entries)
    sizes = np.zeros(max(n, 1), dtype=np.uint64)
    ptrs = np.zeros(max(n, 1), dtype=np.uint64)
    host_ptrs = [0] * n
    arena_total = 0
    small_src: List[int] = []                            # page-locked tensors below SMALL_H2D_BYTES: fetched by ONE kernel
    small_len: List[int] = []
    small_off: List[int] = []
    in_arena = [False] * n
    small_limit = SMALL_H2D_BYTES if _dev._native.load().snt_device_reads_pinned_host() else 0
    for i, (_, buf) in enumerate(entries):
        if not isinstance(buf, torch.Tensor) or not buf.is_contiguous():
            return None
        nbytes = buf.numel() * buf.element_size()
        sizes[i] = nbytes
        if buf.is_cuda:
            ptrs[i] = buf.data_ptr() if nbytes else 0
        elif buf.is_pinned():
            if nbytes == 0:
                continue                                # owns no leaves, needs no address
            in_arena[i] = True
            if nbytes < small_limit:
                small_src.append(buf.data_ptr())
                small_len.append(nbytes)
                small_off.append(arena_total)
            else:
                host_ptrs[i] = buf.data_ptr()
            ptrs[i] = arena_total                       # arena offset for now
            arena_total += -(-nbytes // _ARENA_ALIGN) * _ARENA_ALIGN
        else:
            return None
    if int(sizes[:n].sum()) == 0:
        raise InvalidInput("model must contain at least one byte of tensor data")
    arena = torch.empty(max(arena_total, 16), dtype=torch.uint8, device=dev)
    base = arena.data_ptr()
    main = torch.cuda.current_stream()
    # ONE copy stream: dealing the tensors to two streams alternately (to hide the fixed cost of starting a
    # transfer behind the other stream's data phase) was measured slower, 130 vs 122.6 ms
    sides = _copy_streams(dev)[:1]
    for side in sides:
        side.wait_stream(main)
        arena.record_stream(side)
    lib = _dev._native.load()
    if small_src:
        # A cudaMemcpyAsync costs the copy engine ~3.7 us whatever its size: the 386 biases and layer norms of
        # GPT2-XL (4 MB in all) were 1.5 ms of a 122 ms transfer. ONE gather launch reads them from the page-locked
        # host memory through the unified address space instead (0.12 ms, on the SMs, next to the big transfers).
        # It goes first: its small table upload must not queue behind gigabytes of asynchronous copies.
        _dev.gather_spans(np.array(small_src, dtype=np.uint64), np.array(small_len, dtype=np.uint64),
                          np.array(small_off, dtype=np.uint64), 0, arena)
    handles = [ctypes.c_void_p(side.cuda_stream) for side in sides]
    groups: List[Tuple[int, List[torch.cuda.Event]]] = []       # (first leaf after the group, copies-done events)
    batches = [([], [], []) for _ in sides]
    first, group_bytes, turn = 0, 0, 0
    try:
        for i in range(n):
            nbytes = int(sizes[i])
            if in_arena[i]:
                ptrs[i] = base + int(ptrs[i])
            if host_ptrs[i]:
                b = batches[turn]
                b[0].append(int(ptrs[i])); b[1].append(host_ptrs[i]); b[2].append(nbytes)
                if nbytes >= (1 << 20):
                    turn = (turn + 1) % len(sides)
            group_bytes += nbytes
            first += -(-nbytes // bs)
            if group_bytes >= STAGE_CHUNK_BYTES or i == n - 1:
                events = []
                for side, handle, b in zip(sides, handles, batches):
                    if b[0]:
                        k = len(b[0])
                        rc = lib.snt_memcpy_h2d_batch((ctypes.c_void_p * k)(*b[0]), (ctypes.c_void_p * k)(*b[1]),
                                                      (ctypes.c_uint64 * k)(*b[2]), k, handle)
                        _dev._native.check(rc, "snt_memcpy_h2d_batch")
                        b[0].clear(); b[1].clear(); b[2].clear()
                    ev = torch.cuda.Event()
                    ev.record(side)
                    events.append(ev)
                groups.append((first, events))
                group_bytes = 0
        # the link is busy from here on; now the bookkeeping
        plan = _dev.ModelPlan.from_spans([], ptrs, sizes, bs, count=n)
        try:
            hasher = _dev.MerkleModelHasher(plan, cfg.alg.value)
            begin = 0
            for end, events in groups:
                for ev in events:
                    main.wait_event(ev)
                if end > begin:
                    hasher.run_leaves_only(begin, end)
                begin = end
            hasher.run_tree_only()
            root = Digest(cfg.alg, hasher.out_bytes())          # synchronises: all copies and kernels done
            n_leaves = plan.leaf_count
            aux = hasher.leaves.numel() + hasher.work_bytes + (hasher.out.numel() if n_leaves > 1 else 0)
            return ModelDigestResult(root, cfg, n_leaves, aux_digest_bytes=aux)
        finally:
            plan.close()
    finally:
        torch.cuda.synchronize()          # no copy may still be in flight when the arena goes back to the allocator


def _inplace_merkle_staged(cfg: HashConfig, model: TensorMap, workers: int = 1) -> ModelDigestResult:
    """Host tensors -> device with the copies and the leaf hashing overlapped.

    Device buffers are allocated up front (the plan needs their addresses): tensors that are already
    on the GPU stay where they are; host tensors are laid out back to back (256-byte aligned) in ONE
    device arena -- pinned ones are copied straight into their slice, pageable ones travel through
    the pinned staging ring in 32 MB transfers (``device.RingWriter``). All copies run on a side
    stream; the leaf kernel for a ~256 MB group of whole tensors is enqueued as soon as its bytes
    have landed, and the tree reduction runs once at the end over the leaf digests.
    """
    dev = _dev.require_cuda()
    bs = cfg.block_size
    entries = model.entries
    sizes = [buffer_nbytes(buf) for _, buf in entries]
    CUDA, PINNED, PAGEABLE = 0, 1, 2
    kinds, arena_off, arena_total, n_pageable = [], [0] * len(entries), 0, 0
    for i, (_, buf) in enumerate(entries):
        if _is_cuda(buf):
            kinds.append(CUDA)
        else:
            kinds.append(PINNED if isinstance(buf, torch.Tensor) and buf.is_pinned() else PAGEABLE)
            n_pageable += kinds[-1] == PAGEABLE
            arena_off[i] = arena_total                      # one device allocation for every staged tensor
            arena_total += -(-sizes[i] // _ARENA_ALIGN) * _ARENA_ALIGN
    arena = torch.empty(max(arena_total, 16), dtype=torch.uint8, device=dev)
    dst: List[torch.Tensor] = []
    for i, (_, buf) in enumerate(entries):
        if kinds[i] == CUDA:
            dst.append(_dev.as_device_bytes(buf, dev))
        else:
            dst.append(arena[arena_off[i]:arena_off[i] + sizes[i]])
    plan = _dev.ModelPlan(dst, bs)
    ring = _dev.StagingRing.get(_dev.staging_threads(workers)) if n_pageable else None
    if ring is not None:
        ring.lock.acquire()                  # one staged hash at a time owns the ring
    try:
        hasher = _dev.MerkleModelHasher(plan, cfg.alg.value)
        main = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(main)
        arena.record_stream(side)            # the arena is filled by copies on the side stream
        # pageable bytes travel through the staging ring: memcpy tasks queued ahead, transfers issued on `side`
        writer = _dev.RingWriter(ring, arena, side) if ring is not None else None

        first, group_begin, group_bytes = 0, 0, 0
        n = len(dst)
        lib = _dev._native.load()
        side_handle = ctypes.c_void_p(side.cuda_stream)
        # page-locked tensors of a group go to the side stream as ONE batch of asynchronous copies issued from C
        # (snt_memcpy_h2d_batch): a Python call per tensor leaves the link idle between the small ones
        batch_dst: List[int] = []
        batch_src: List[int] = []
        batch_len: List[int] = []
        batch_keep: List[torch.Tensor] = []

        def flush_pinned():
            if not batch_dst:
                return
            k = len(batch_dst)
            rc = lib.snt_memcpy_h2d_batch((ctypes.c_void_p * k)(*batch_dst), (ctypes.c_void_p * k)(*batch_src),
                                          (ctypes.c_uint64 * k)(*batch_len), k, side_handle)
            _dev._native.check(rc, "snt_memcpy_h2d_batch")
            batch_dst.clear(); batch_src.clear(); batch_len.clear()

        for i, (_, buf) in enumerate(entries):
            if kinds[i] == PINNED and sizes[i]:
                if writer is not None:
                    writer.close()   # a ring transfer covers one contiguous arena range: it must not span this slice
                src_t = buf if buf.is_contiguous() else buf.contiguous()
                if src_t is not buf and not src_t.is_pinned():
                    flush_pinned()
                    with torch.cuda.stream(side):
                        dst[i].copy_(_host_tensor(src_t), non_blocking=True)
                else:
                    batch_keep.append(src_t)
                    batch_dst.append(dst[i].data_ptr())
                    batch_src.append(src_t.data_ptr())
                    batch_len.append(sizes[i])
            elif kinds[i] == PAGEABLE and sizes[i]:
                flush_pinned()       # keep the arena filling in order on the side stream
                src = _host_tensor(buf).numpy() if isinstance(buf, torch.Tensor) else _dev.host_bytes_view(buf)
                writer.write(arena_off[i], src)
            group_bytes += sizes[i]
            first_next = first + -(-sizes[i] // bs)
            if group_bytes >= STAGE_CHUNK_BYTES or i == n - 1:
                if writer is not None:
                    writer.drain()
                flush_pinned()
                done = torch.cuda.Event()
                done.record(side)
                main.wait_event(done)
                if first_next > group_begin:
                    hasher.run_leaves_only(group_begin, first_next)
                group_begin, group_bytes = first_next, 0
            first = first_next
        hasher.run_tree_only()
        root = Digest(cfg.alg, hasher.out_bytes())          # synchronises: all copies and kernels done
        n_leaves = plan.leaf_count
        aux = hasher.leaves.numel() + hasher.work_bytes + (hasher.out.numel() if n_leaves > 1 else 0)
        return ModelDigestResult(root, cfg, n_leaves, aux_digest_bytes=aux)
    finally:
        # no copy may still be in flight when the arena goes back to the allocator or the ring to its next owner
        torch.cuda.synchronize()
        if ring is not None:
            ring.lock.release()
        plan.close()


class _ResidentEntry:
    """Plan + workspace of one device-resident model: what a repeated ``hash_model`` call re-uses."""

    __slots__ = ("key", "storages", "ids", "plan", "hasher", "host", "busy")

    def __init__(self, key, tensors, plan, hasher, host):
        self.key = key                   # (ptrs, sizes, block size, algorithm, device, stream)
        # the STORAGES the plan's addresses point into (not the tensor objects, which can be re-pointed with
        # `.data =` / `set_`): as long as the entry lives, a launch from the cached plan reads allocated memory
        self.storages = [t.untyped_storage() for t in tensors]
        self.ids = tuple(map(id, tensors))
        self.plan, self.hasher, self.host = plan, hasher, host
        self.busy = threading.Lock()     # one call at a time owns the workspace

    def close(self) -> None:
        self.plan.close()


def _resident_key(buffers, cfg: HashConfig, stream):
    """Everything the device plan depends on: addresses, byte lengths, block size, algorithm, device, stream.
    Rejects tensors the in-place path cannot take as they are (non-contiguous views)."""
    n = len(buffers)
    ptrs = np.fromiter((b.data_ptr() for b in buffers), dtype=np.uint64, count=n)
    sizes = np.fromiter((b.nbytes for b in buffers), dtype=np.uint64, count=n)
    contiguous = all(b.is_cuda and b.is_contiguous() for b in buffers)   # `.data = cpu_tensor` moves a tensor object
    ptrs[sizes == 0] = 0
    return (ptrs.tobytes(), sizes.tobytes(), cfg.block_size, cfg.alg.value, stream.device_index, stream.cuda_stream), \
        ptrs, sizes, contiguous


def clear_hash_cache(model: Optional[TensorMap] = None) -> None:
    """Release the plan / workspace a ``TensorMap`` of device tensors carries after it has been hashed."""
    if model is not None:
        entry = model.__dict__.pop("_resident", None)
        # a thread that is hashing through this entry right now keeps it alive; its plan then goes with the entry
        if entry is not None and entry.busy.acquire(blocking=False):
            try:
                entry.close()
            finally:
                entry.busy.release()


def _inplace_merkle_resident(cfg: HashConfig, model: TensorMap, buffers=None) -> ModelDigestResult:
    """Every tensor already lives in HBM: hash in place, re-using the plan and workspace of the last call.

    The plan (device block table), the leaf-digest buffer, the reducer workspace and a pinned root buffer
    hang off the ``TensorMap`` itself, so they live exactly as long as the model the caller holds. When the
    same ``TensorMap`` (same tensor objects) is hashed again the kernels are launched FIRST, from the cached
    plan -- the entry holds the storages behind its addresses, so they are allocated memory whatever happened --
    and the per-tensor checks (address, length, contiguity: ~0.4 us per tensor in Python) run while the GPU
    works. Only if a check fails (a tensor was re-pointed or resized in place) is the result thrown away
    and the model hashed again through a fresh plan. Nothing unchecked is ever returned.
    """
    stream = torch.cuda.current_stream()
    entry: Optional[_ResidentEntry] = model.__dict__.get("_resident")
    launched = False
    # O(1) checks only before the launch: the entry owns the storages its plan points into, so the speculative
    # launch is safe whatever the caller did to the TensorMap; WHICH tensors it holds now is checked afterwards
    if entry is not None and entry.key[2:] == (cfg.block_size, cfg.alg.value, stream.device_index, stream.cuda_stream) \
            and entry.busy.acquire(blocking=False):
        entry.hasher.run()                                   # root lands in pinned host memory (host_out)
        launched = True
    if buffers is None:
        buffers = [buf for _, buf in model.entries]
    if all(type(b) is torch.Tensor for b in buffers):
        key, ptrs, sizes, contiguous = _resident_key(buffers, cfg, stream)
        on_device = contiguous or all(b.is_cuda for b in buffers)
    else:
        key, contiguous, on_device = None, False, False
    if launched and (key != entry.key or not contiguous or entry.ids != tuple(map(id, buffers))):
        stream.synchronize()
        entry.busy.release()
        launched = False
    if not launched:
        if not on_device:                                    # the TensorMap no longer holds only device tensors
            clear_hash_cache(model)
            return inplace_hash(cfg, model)
        if entry is not None and entry.busy.locked():        # another thread is hashing this very TensorMap: do not share
            return _inplace_merkle_uncached(cfg, buffers)
        if not contiguous:
            return _inplace_merkle_uncached(cfg, buffers)
        plan = _dev.ModelPlan.from_spans([], ptrs, sizes, cfg.block_size, count=len(buffers))   # rejects an empty model
        try:
            hasher = _dev.MerkleModelHasher(plan, cfg.alg.value, host_out=True)
        except Exception:
            plan.close()
            raise
        old, entry = entry, _ResidentEntry(key, list(buffers), plan, hasher, hasher.out)
        entry.busy.acquire()
        model.__dict__["_resident"] = entry
        if old is not None:
            old.close()
        entry.hasher.run()
    try:
        stream.synchronize()
        root = Digest(cfg.alg, entry.host.numpy().tobytes())
    finally:
        entry.busy.release()
    leaves = entry.plan.leaf_count
    hasher = entry.hasher
    aux = hasher.leaves.numel() + hasher.work_bytes + (hasher.out.numel() if leaves > 1 else 0)
    return ModelDigestResult(root, cfg, leaves, aux_digest_bytes=aux)


def _inplace_merkle_uncached(cfg: HashConfig, buffers) -> ModelDigestResult:
    plan = _dev.ModelPlan.from_spans(*_dev.device_spans(buffers), cfg.block_size)
    try:
        return _hash_plan(cfg, plan)
    finally:
        plan.close()


def inplace_hash(cfg: HashConfig, model: TensorMap, workers: int = 1) -> ModelDigestResult:
    """Hash fragmented tensors where they lie: no copy, no padding (model.py:298-315)."""
    if cfg.construction is Construction.MERKLE and "_resident" in model.__dict__:
        return _inplace_merkle_resident(cfg, model)          # launch first, re-check after
    buffers = [buf for _, buf in model.entries]
    all_resident = all(type(buf) is torch.Tensor and buf.is_cuda for buf in buffers)
    if all_resident and buffers and cfg.construction is Construction.MERKLE:
        return _inplace_merkle_resident(cfg, model, buffers)
    if not all_resident:
        _require_nonempty(model)
        host_bytes = sum(buffer_nbytes(buf) for buf in buffers if not _is_cuda(buf))
        if cfg.construction is Construction.MERKLE and host_bytes >= STAGE_PIPELINE_MIN_BYTES:
            fast = _inplace_merkle_pinned(cfg, model)
            return fast if fast is not None else _inplace_merkle_staged(cfg, model, workers)
    # an empty model is rejected by snt_model_plan_create (InvalidInput, model.py:166-168)
    plan = _dev.ModelPlan.from_spans(*_dev.device_spans(buffers), cfg.block_size)
    try:
        return _hash_plan(cfg, plan)
    finally:
        plan.close()


def coalesce_hash(cfg: HashConfig, model: TensorMap, workers: int = 1) -> ModelDigestResult:
    """Gather all tensors into one zero-padded device buffer, then hash its blocks (model.py:203-228)."""
    _require_nonempty(model)
    dev = _dev.require_cuda()
    bs = cfg.block_size
    keep, ptrs, sizes = _dev.device_spans([buf for _, buf in model.entries], dev)
    n = len(keep)
    total = int(sizes[:n].sum())
    padded = -(-total // bs) * bs
    packed = torch.empty(padded, dtype=torch.uint8, device=dev)
    if padded > total:
        packed[total:].zero_()
    dst_off = np.zeros(n, dtype=np.uint64)
    np.cumsum(sizes[:n - 1], out=dst_off[1:])
    _dev.gather_spans(ptrs[:n], sizes[:n], dst_off, 0, packed)          # one launch for all tensors
    plan = _dev.ModelPlan([packed], bs)
    try:
        return _hash_plan(cfg, plan, aux_data_bytes=padded)
    finally:
        plan.close()
        del keep


def per_layer_hash(cfg: HashConfig, model: TensorMap, workers: int = 1) -> ModelDigestResult:
    """Hash each tensor to a layer digest, then reduce the layer digests (model.py:231-286).

    Merkle: every tensor is its own tree over its blocks, the last block zero-padded to
    the block size (an empty tensor contributes H(b"")), and the layer digests are the
    leaves of a second tree in entry order. The full blocks are hashed in place; only the
    ragged tails (< one block each) are copied into a zero-filled scratch buffer. All
    leaves go through one leaf launch, the per-tensor trees through
    ``snt_merkle_roots_segmented``.
    Lattice: blocks are unpadded and tagged LE64(layer) || LE64(block); one launch sums
    every tensor into its own accumulator slot, and the model digest is the sum of the
    layer digests. ``ordered_per_layer`` changes the reference's schedule, not the result.
    """
    _require_nonempty(model)
    dev = _dev.require_cuda()
    bs = cfg.block_size
    names = model.names()
    keep, ptrs, sizes = _dev.device_spans([buf for _, buf in model.entries], dev)
    n_layers = len(keep)
    ptrs, sizes = ptrs[:n_layers], sizes[:n_layers]
    block_counts = [int(c) for c in (sizes + np.uint64(bs - 1)) // np.uint64(bs)]

    if cfg.construction is Construction.MERKLE:
        alg = cfg.alg.value
        dlen = cfg.alg.digest_len
        # span arithmetic only (no per-tensor device op): the full blocks of tensor i stay where they are,
        # its ragged tail is gathered, zero-padded, into slot k of a scratch buffer (one launch for all tails)
        full = sizes // np.uint64(bs) * np.uint64(bs)
        tail = sizes - full
        ragged = np.nonzero(tail)[0]
        scratch = torch.empty(max(1, len(ragged)) * bs, dtype=torch.uint8, device=dev)
        slot_addr = np.zeros(n_layers, dtype=np.uint64)
        slot_addr[ragged] = np.uint64(scratch.data_ptr()) + np.arange(len(ragged), dtype=np.uint64) * np.uint64(bs)
        if len(ragged):
            _dev.gather_spans((ptrs + full)[ragged], tail[ragged], np.arange(len(ragged), dtype=np.uint64) * np.uint64(bs),
                              bs, scratch)
        v_ptrs = np.stack([ptrs, slot_addr], axis=1).reshape(-1)         # per tensor: (full part, padded tail)
        v_sizes = np.stack([full, np.where(tail > 0, np.uint64(bs), np.uint64(0))], axis=1).reshape(-1)
        live = np.nonzero(v_sizes)[0]
        seg_first = [0]
        for c in block_counts:
            seg_first.append(seg_first[-1] + c)
        plan = _dev.ModelPlan.from_spans([keep, scratch], np.ascontiguousarray(v_ptrs[live]),
                                         np.ascontiguousarray(v_sizes[live]), bs, count=len(live))
        try:
            hasher = _dev.MerkleModelHasher(plan, alg)
            hasher.run_leaves_only()
            empty = _dev.hash_blocks_device(alg, None, torch.zeros(1, dtype=torch.int64, device=dev),
                                            torch.zeros(1, dtype=torch.int64, device=dev))
            layers_dev = _dev.merkle_roots_segmented_device(alg, hasher.leaves, seg_first, empty)
            root_dev = _dev.merkle_root_device(alg, layers_dev, n_layers)
            layer_bytes = layers_dev.cpu().numpy().tobytes()
            root = Digest(cfg.alg, root_dev.cpu().numpy().tobytes())
            aux_digest = hasher.leaves.numel() + layers_dev.numel() + hasher.work_bytes
            # as in the reference (model.py:231-286), the zero-padded copies of the ragged last blocks are
            # transient and not counted: aux_data_bytes reports tensor data gathered into a new buffer
            # (the coalesced strategy), aux_digest_bytes the digest storage
            aux_data = 0
        finally:
            plan.close()
        layer_digests = {name: Digest(cfg.alg, layer_bytes[i * dlen:(i + 1) * dlen]) for i, name in enumerate(names)}
        return ModelDigestResult(root, cfg, sum(block_counts), layer_digests=layer_digests,
                                 aux_data_bytes=aux_data, aux_digest_bytes=aux_digest)

    plan = _dev.ModelPlan.from_spans(keep, ptrs, sizes, bs)
    try:
        acc = _dev.LatticeAccumulator(n_layers)
        acc.add_model_layers(plan, 0, plan.leaf_count)
        layers_dev = acc.finalize_device()
        total = _dev.LatticeAccumulator(1)
        total.add_digests(layers_dev, n_layers)
        layer_bytes = layers_dev.cpu().numpy().tobytes()
        model_bytes, _, _ = total.digests()
    finally:
        plan.close()
    layer_digests = {name: LatticeDigest(layer_bytes[i * 64:(i + 1) * 64]) for i, name in enumerate(names)}
    return ModelDigestResult(LatticeDigest(model_bytes), cfg, sum(block_counts), layer_digests=layer_digests,
                             aux_digest_bytes=(n_layers + 1) * _dev.LT_LANES * 8)


def ordered_lattice_per_layer(cfg: HashConfig, model: TensorMap, workers: int = 1) -> ModelDigestResult:
    """Size-ordered lattice per-layer hashing (model.py:289-295)."""
    if (cfg.construction is not Construction.LATTICE or cfg.strategy is not Strategy.PER_LAYER
            or not cfg.ordered_per_layer):
        raise ConfigError("ordered_lattice_per_layer requires lattice per-layer ordered config")
    return per_layer_hash(cfg, model, workers)


_DISPATCH = {
    Strategy.COALESCED: coalesce_hash,
    Strategy.PER_LAYER: per_layer_hash,
    Strategy.IN_PLACE: inplace_hash,
}


def hash_model(cfg: HashConfig, model: TensorMap, workers: int = 1) -> ModelDigestResult:
    """Validate the configuration and run the matching strategy (model.py:325-330)."""
    cfg.validate()
    if cfg.ordered_per_layer:
        return ordered_lattice_per_layer(cfg, model, workers)
    return _DISPATCH[cfg.strategy](cfg, model, workers)


# --- manifest I/O (host files; formats identical to model.py:335-374) -----------

def load_model(manifest_path) -> TensorMap:
    """Read ``{"tensors": [{name, offset, length}], "data": file}`` plus the raw data file.

    Every tensor becomes its own buffer, reproducing a checkpoint's fragmentation.
    """
    manifest_path = Path(manifest_path)
    try:
        doc = json.loads(manifest_path.read_text())
        raw = (manifest_path.parent / doc["data"]).read_bytes()
        entries = []
        for rec in doc["tensors"]:
            start, length = int(rec["offset"]), int(rec["length"])
            if start < 0 or length < 0 or start + length > len(raw):
                raise FormatError(f"tensor {rec['name']!r} range [{start}, {start + length}) exceeds data file")
            entries.append((rec["name"], bytes(raw[start:start + length])))
    except FormatError:
        raise
    except (OSError, KeyError, ValueError, TypeError) as exc:
        raise FormatError(f"bad model manifest {manifest_path}: {exc}") from exc
    return TensorMap(entries)


def save_model(model: TensorMap, manifest_path, data_name: Optional[str] = None) -> None:
    """Write the manifest and the concatenated tensor bytes next to it."""
    manifest_path = Path(manifest_path)
    data_name = data_name or manifest_path.stem + ".bin"
    records, blobs, pos = [], [], 0
    for name, buf in model.entries:
        if isinstance(buf, torch.Tensor):
            buf = buf.detach().cpu().contiguous().reshape(-1).view(torch.uint8).numpy().tobytes()
        blob = bytes(memoryview(buf).cast("B")) if not isinstance(buf, bytes) else buf
        records.append({"name": name, "offset": pos, "length": len(blob)})
        blobs.append(blob)
        pos += len(blob)
    (manifest_path.parent / data_name).write_bytes(b"".join(blobs))
    manifest_path.write_text(json.dumps({"tensors": records, "data": data_name}, indent=2))
