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


class _OpenFile:
    """A data file kept open for the tensors that view it (closed when the last of them is gone)."""

    def __init__(self, path):
        import os

        self.path = path
        self.fd = os.open(path, os.O_RDONLY)
        self.size = os.fstat(self.fd).st_size
        self._whole: Optional[memoryview] = None

    def whole(self) -> memoryview:
        """The file's bytes in host memory, read ONCE (in parallel, ``device.read_file_host``) when a consumer other
        than the in-place GPU path first asks for any tensor's bytes."""
        if self._whole is None:
            self._whole = memoryview(_dev.read_file_host(self.path)).toreadonly()
            if len(self._whole) < self.size:
                raise FormatError(f"data file {self.path} shrank while it was open")
        return self._whole

    def __del__(self, _close=__import__("os").close):      # (bound now: at interpreter shutdown imports no longer work)
        try:
            _close(self.fd)
        except OSError:
            pass


class FileTensor:
    """Bytes [offset, offset + nbytes) of a checkpoint's data file, read only when somebody needs them.

    ``load_model`` hands these out: ``hash_model`` on the in-place path has the staging threads ``pread`` each
    piece straight into the pinned ring (file -> page-locked memory -> HBM, no copy of the checkpoint in host
    memory at all). Everything else sees an ordinary read-only bytes-like object: it exports the buffer protocol
    (PEP 688; the first use reads the whole file once, in parallel, and every tensor is then a view of that) and
    compares equal to the ``bytes`` the reference builds (model.py:335-352).
    """

    __slots__ = ("file", "offset", "nbytes")
    __hash__ = None

    def __init__(self, file: _OpenFile, offset: int, nbytes: int):
        self.file, self.offset, self.nbytes = file, offset, nbytes

    def view(self) -> memoryview:
        return self.file.whole()[self.offset:self.offset + self.nbytes]

    def __buffer__(self, flags):                            # np.frombuffer / memoryview / bytes() all work
        return self.view()

    def tobytes(self) -> bytes:
        return bytes(self.view())

    __bytes__ = tobytes

    def __len__(self) -> int:
        return self.nbytes

    def __eq__(self, other):
        try:
            return self.view() == memoryview(other)
        except TypeError:
            return NotImplemented

    def __repr__(self) -> str:
        return f"FileTensor(offset={self.offset}, nbytes={self.nbytes})"


def buffer_nbytes(buf) -> int:
    if isinstance(buf, FileTensor):
        return buf.nbytes
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


LAST_HOST_STAGING: Dict[str, int] = {}   # layout of the most recent _inplace_merkle_host call (diagnostics)
STAGE_PIECE_BYTES = 64 << 20             # a host tensor travels in pieces of at most this (a multiple of the block size)
STAGE_RING_GROUPS = 3                    # copy/hash groups the transfers may run ahead of the hashing


def _inplace_merkle_host(cfg: HashConfig, model: TensorMap, workers: int = 1) -> ModelDigestResult:
    """Host tensors (page-locked or pageable, CUDA tensors mixed in) hashed while they arrive, in BOUNDED device memory
    (both constructions: Merkle leaves + tree, or LATTICE block sums).

    Every host tensor is cut into pieces of at most 64 MB at block boundaries -- the leaf sequence of the pieces
    is the leaf sequence of the tensor -- and the pieces are laid out in a RING of device memory that holds a few
    copy/hash groups (~256 MB each): a 6.55 GB state dict needs 1.3 GB of HBM, not a copy of itself, and a model
    larger than the GPU's memory can be hashed at all. The plan (one row per piece) is built once, up front: ring
    addresses are known before a byte has moved. Then, group by group:

      * the transfers of group g are put on a side stream -- page-locked pieces as ONE batch of asynchronous
        copies issued from C (``snt_memcpy_h2d_batch``), pageable ones through the pinned staging ring and its
        copy threads (``device.RingWriter``) -- after the stream has been told to wait for the leaf launch that
        last read the ring memory they overwrite (group g - 3);
      * the leaf launch of group g waits for the group's transfers and hashes its leaf range; the tree runs once at
        the end over the leaf digests.

    When every host tensor is page-locked the first three groups of transfers are on the stream before the plan
    and the workspace are even created: the link is the whole cost (GPT2-XL: 121 ms for 117.9 ms of link). A
    ``cudaMemcpyAsync`` costs the copy engine ~3.7 us whatever its size, so page-locked tensors below 64 KB (the
    386 biases and layer norms of GPT2-XL: 4 MB, 1.5 ms of copy engine) live in a small arena of their own and are
    fetched by ONE gather launch that reads the host memory through the unified address space.
    """
    dev = _dev.require_cuda()
    lib = _dev._native.load()
    bs = cfg.block_size
    entries = model.entries
    CUDA, PINNED, PAGEABLE, SMALL, FILE = 0, 1, 2, 3, 4
    piece = max(bs, STAGE_PIECE_BYTES // bs * bs)
    small_limit = SMALL_H2D_BYTES if lib.snt_device_reads_pinned_host() else 0

    # ---- spans: (kind, source, source offset, bytes); a host tensor contributes one span per piece
    spans: List[Tuple[int, object, int, int]] = []
    keep: List[object] = []
    n_pageable = 0
    for _, buf in entries:
        is_tensor = isinstance(buf, torch.Tensor)
        nbytes = buf.nbytes if is_tensor else buffer_nbytes(buf)
        if nbytes == 0:
            spans.append((CUDA, None, 0, 0))
        elif is_tensor and buf.is_cuda:
            t = _dev.as_device_bytes(buf, dev)
            keep.append(t)
            spans.append((CUDA, t, 0, nbytes))
        elif isinstance(buf, FileTensor):
            keep.append(buf)                               # pread by the staging threads straight into the pinned ring
            spans.extend((FILE, buf, o, min(piece, nbytes - o)) for o in range(0, nbytes, piece))
            n_pageable += 1
        elif is_tensor and buf.is_pinned() and buf.is_contiguous():
            if nbytes < small_limit:
                spans.append((SMALL, buf, 0, nbytes))
            else:
                spans.extend((PINNED, buf, o, min(piece, nbytes - o)) for o in range(0, nbytes, piece))
        else:
            src = _host_tensor(buf).numpy() if isinstance(buf, torch.Tensor) else _dev.host_bytes_view(buf)
            keep.append(src)
            spans.extend((PAGEABLE, src, o, min(piece, nbytes - o)) for o in range(0, nbytes, piece))
            n_pageable += 1
    n = len(spans)
    if sum(sp[3] for sp in spans) == 0:
        raise InvalidInput("model must contain at least one byte of tensor data")

    # ---- layout: ring offsets of the pieces, groups of >= STAGE_CHUNK_BYTES, the small tensors' own arena
    def aligned(x: int) -> int:
        return -(-x // _ARENA_ALIGN) * _ARENA_ALIGN

    ring_need = sum(aligned(sp[3]) for sp in spans if sp[0] in (PINNED, PAGEABLE, FILE))
    ring_bytes = min(ring_need, (STAGE_RING_GROUPS + 1) * (STAGE_CHUNK_BYTES + aligned(piece)))
    small_bytes = sum(aligned(sp[3]) for sp in spans if sp[0] == SMALL)
    ring = torch.empty(max(ring_bytes, 16), dtype=torch.uint8, device=dev)
    small_arena = torch.empty(max(small_bytes, 16), dtype=torch.uint8, device=dev)
    ring_base, small_base = ring.data_ptr(), small_arena.data_ptr()
    ptrs = np.zeros(n, dtype=np.uint64)
    sizes = np.fromiter((sp[3] for sp in spans), dtype=np.uint64, count=n)
    offs = [0] * n                                         # ring offset of a PINNED / PAGEABLE span
    groups: List[Tuple[int, int, int]] = []               # (first span, end span, first leaf after the group)
    pos, small_pos, leaf, g_begin, g_bytes = 0, 0, 0, 0, 0
    left = ring_need                                       # host bytes not yet assigned to a group
    small_src: List[int] = []
    small_len: List[int] = []
    small_off: List[int] = []
    for i, (kind, src, off, nbytes) in enumerate(spans):
        if kind == CUDA:
            ptrs[i] = src.data_ptr() if nbytes else 0
        elif kind == SMALL:
            ptrs[i] = small_base + small_pos
            small_src.append(src.data_ptr())
            small_len.append(nbytes)
            small_off.append(small_pos)
            small_pos += aligned(nbytes)
        else:
            if pos + aligned(nbytes) > ring_bytes:
                pos = 0                                    # a piece is contiguous: wrap before it, not inside it
            offs[i] = pos
            ptrs[i] = ring_base + pos
            pos += aligned(nbytes)
            g_bytes += aligned(nbytes)                     # the group's footprint in the ring, padding included
            left -= aligned(nbytes)
        leaf += -(-nbytes // bs)
        # groups shrink towards the end (half of what is left, at least 1/16 of a full group): the hashing of the
        # LAST group is the only one no transfer hides
        if g_bytes >= min(STAGE_CHUNK_BYTES, max(STAGE_CHUNK_BYTES >> 4, left >> 1)) or i == n - 1:
            groups.append((g_begin, i + 1, leaf))
            g_begin, g_bytes = i + 1, 0

    global LAST_HOST_STAGING                               # (diagnostics: tests and bench read it)
    LAST_HOST_STAGING = {"ring_bytes": int(ring_bytes), "host_bytes": int(ring_need), "small_arena_bytes": int(small_bytes),
                         "pieces": n, "groups": len(groups)}
    main = torch.cuda.current_stream()
    side = _copy_streams(dev)[0]
    side.wait_stream(main)
    ring.record_stream(side)
    side_handle = ctypes.c_void_p(side.cuda_stream)
    staging = _dev.StagingRing.get(_dev.staging_threads(workers)) if n_pageable else None
    if staging is not None:
        staging.lock.acquire()                             # one staged hash at a time owns the pinned staging ring
    plan = None
    writer = None
    try:
        writer = _dev.RingWriter(staging, ring, side) if staging is not None else None
        copied: List[Optional[torch.cuda.Event]] = [None] * len(groups)
        hashed: List[Optional[torch.cuda.Event]] = [None] * len(groups)

        def issue(g: int) -> None:
            """Put the transfers of group g on the side stream (ring memory: after the leaf launch of group g - R)."""
            if g >= STAGE_RING_GROUPS and ring_bytes < ring_need:
                side.wait_event(hashed[g - STAGE_RING_GROUPS])
            b_dst: List[int] = []
            b_src: List[int] = []
            b_len: List[int] = []

            def flush_pinned() -> None:
                if b_dst:
                    k = len(b_dst)
                    rc = lib.snt_memcpy_h2d_batch((ctypes.c_void_p * k)(*b_dst), (ctypes.c_void_p * k)(*b_src),
                                                  (ctypes.c_uint64 * k)(*b_len), k, side_handle)
                    _dev._native.check(rc, "snt_memcpy_h2d_batch")
                    b_dst.clear(); b_src.clear(); b_len.clear()

            first, end, _ = groups[g]
            for i in range(first, end):
                kind, src, off, nbytes = spans[i]
                if kind == PINNED:
                    if writer is not None:
                        writer.close()                     # a staging transfer covers ONE contiguous ring range
                    b_dst.append(int(ptrs[i])); b_src.append(src.data_ptr() + off); b_len.append(nbytes)
                elif kind == PAGEABLE:
                    flush_pinned()
                    writer.write(offs[i], src[off:off + nbytes])
                elif kind == FILE:
                    flush_pinned()
                    writer.write_file(offs[i], src.file.fd, src.offset + off, nbytes)
            if writer is not None:
                writer.drain()
            flush_pinned()
            ev = torch.cuda.Event()
            ev.record(side)
            copied[g] = ev

        ahead = min(len(groups), STAGE_RING_GROUPS)
        if n_pageable == 0:
            for g in range(ahead):                         # page-locked sources: the link is busy from here on
                issue(g)
        if small_src:                                      # on the main stream, ahead of every leaf launch
            _dev.gather_spans(np.array(small_src, dtype=np.uint64), np.array(small_len, dtype=np.uint64),
                              np.array(small_off, dtype=np.uint64), 0, small_arena)
        plan = _dev.ModelPlan.from_spans(keep, ptrs, sizes, bs, count=n)
        merkle = cfg.construction is Construction.MERKLE
        hasher = _dev.MerkleModelHasher(plan, cfg.alg.value) if merkle else None
        acc = None if merkle else _dev.LatticeAccumulator(1)     # LATTICE: leaves tagged LE64(k), summed (model.py:312-315)
        if n_pageable:
            for g in range(ahead):
                issue(g)
        begin = 0
        for g, (_, _, leaf_end) in enumerate(groups):
            main.wait_event(copied[g])
            if leaf_end > begin:
                if merkle:
                    hasher.run_leaves_only(begin, leaf_end)
                else:
                    acc.add_model_leaves(plan, begin, leaf_end)
            begin = leaf_end
            done = torch.cuda.Event()
            done.record(main)
            hashed[g] = done
            if g + ahead < len(groups):
                issue(g + ahead)
        n_leaves = plan.leaf_count
        if not merkle:
            out, _, _ = acc.digests()                       # synchronises
            return ModelDigestResult(LatticeDigest(out), cfg, n_leaves, aux_digest_bytes=acc.acc.numel() * 8)
        hasher.run_tree_only()
        root = Digest(cfg.alg, hasher.out_bytes())          # synchronises: all copies and kernels done
        aux = hasher.leaves.numel() + hasher.work_bytes + (hasher.out.numel() if n_leaves > 1 else 0)
        return ModelDigestResult(root, cfg, n_leaves, aux_digest_bytes=aux)
    finally:
        # no copy may still be in flight when the ring goes back to the allocator or the staging ring to its next owner
        if writer is not None:
            writer.abandon()                                # (a no-op unless an exception left staged copies behind)
        torch.cuda.synchronize()
        if staging is not None:
            staging.lock.release()
        if plan is not None:
            plan.close()


class _ResidentEntry:
    """Plan + workspace of one device-resident model: what a repeated ``hash_model`` call re-uses."""

    __slots__ = ("key", "storages", "ids", "plan", "hasher", "host", "busy", "acc")

    def __init__(self, key, tensors, plan, hasher, host, acc=None):
        self.key = key                   # (ptrs, sizes, block size, algorithm, device, stream)
        # the STORAGES the plan's addresses point into (not the tensor objects, which can be re-pointed with
        # `.data =` / `set_`): as long as the entry lives, a launch from the cached plan reads allocated memory
        self.storages = [t.untyped_storage() for t in tensors]
        self.ids = tuple(map(id, tensors))
        self.plan, self.hasher, self.host = plan, hasher, host
        self.acc = acc                   # LATTICE construction: the accumulator instead of a Merkle hasher
        self.busy = threading.Lock()     # one call at a time owns the workspace

    def launch(self) -> None:
        """Enqueue the whole hash from the cached plan; the result lands in page-locked host memory."""
        if self.hasher is not None:
            self.hasher.run()
        else:
            self.acc.zero_()
            self.acc.add_model_leaves(self.plan, 0, self.plan.leaf_count)
            self.acc.finalize_to_host()

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
    return (ptrs.tobytes(), sizes.tobytes(), cfg.block_size, cfg.alg.value, cfg.construction.value, stream.device_index,
            stream.cuda_stream), ptrs, sizes, contiguous


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
    if entry is not None and entry.key[2:] == (cfg.block_size, cfg.alg.value, cfg.construction.value, stream.device_index,
                                               stream.cuda_stream) and entry.busy.acquire(blocking=False):
        entry.launch()                                       # the result lands in pinned host memory
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
            if cfg.construction is Construction.MERKLE:
                hasher, acc = _dev.MerkleModelHasher(plan, cfg.alg.value, host_out=True), None
            else:
                hasher, acc = None, _dev.LatticeAccumulator(1)
        except Exception:
            plan.close()
            raise
        old, entry = entry, _ResidentEntry(key, list(buffers), plan, hasher, hasher.out if hasher is not None else None, acc)
        entry.busy.acquire()
        model.__dict__["_resident"] = entry
        if old is not None:
            old.close()
        entry.launch()
    leaves = entry.plan.leaf_count
    try:
        stream.synchronize()
        if entry.hasher is None:
            out, _, _ = entry.acc.host_result()
            # one 64-byte accumulator instead of the reference's n x 64 digest array
            return ModelDigestResult(LatticeDigest(out), cfg, leaves, aux_digest_bytes=entry.acc.acc.numel() * 8)
        root = Digest(cfg.alg, entry.host.numpy().tobytes())
    finally:
        entry.busy.release()
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
    if "_resident" in model.__dict__:
        return _inplace_merkle_resident(cfg, model)          # launch first, re-check after
    buffers = [buf for _, buf in model.entries]
    all_resident = all(type(buf) is torch.Tensor and buf.is_cuda for buf in buffers)
    if all_resident and buffers:
        return _inplace_merkle_resident(cfg, model, buffers)
    if not all_resident:
        _require_nonempty(model)
        host_bytes = sum(buffer_nbytes(buf) for buf in buffers if not _is_cuda(buf))
        if host_bytes >= STAGE_PIPELINE_MIN_BYTES:
            return _inplace_merkle_host(cfg, model, workers)
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
        # the data file stays open; every tensor is a lazy read-only view of its byte range (see FileTensor)
        data = _OpenFile(manifest_path.parent / doc["data"])
        entries = []
        for rec in doc["tensors"]:
            start, length = int(rec["offset"]), int(rec["length"])
            if start < 0 or length < 0 or start + length > data.size:
                raise FormatError(f"tensor {rec['name']!r} range [{start}, {start + length}) exceeds data file")
            entries.append((rec["name"], FileTensor(data, start, length)))
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
