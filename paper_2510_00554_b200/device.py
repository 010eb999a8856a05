"""Device plumbing: torch supplies HBM buffers and streams, the C ABI does the work.

Everything that touches the GPU goes through this module: staging host bytes
into device tensors, building model plans, and calling the ``snt_*`` entry
points on torch's current stream. There is no CPU implementation behind these
functions -- without a CUDA device they raise ``ResourceError``.
"""

from __future__ import annotations

import collections
import ctypes
import threading
import warnings
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native
from .errors import InvalidInput, ResourceError

try:                                    # CPython helper built next to the CUDA library (build.build_hostpack)
    from . import _hostpack
except ImportError:                     # only the packing gets slower; hashing never runs on the host either way
    _hostpack = None

ALG_IDS = {"sha256": 0, "blake2b": 1, "sha3-256": 2}
DIGEST_LEN = {"sha256": 32, "blake2b": 64, "sha3-256": 32}
LT_LANES = 32


def require_cuda() -> torch.device:
    """The current CUDA device, or ``ResourceError`` (no CPU fallback exists)."""
    if not torch.cuda.is_available():
        raise ResourceError("a CUDA device is required: the hashing engine has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: Optional[torch.Tensor]) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def host_bytes_view(buf) -> np.ndarray:
    """Zero-copy uint8 view of a host bytes-like object."""
    if isinstance(buf, np.ndarray):
        return np.ascontiguousarray(buf).reshape(-1).view(np.uint8)
    return np.frombuffer(buf, dtype=np.uint8)


def as_device_bytes(buf, device: Optional[torch.device] = None) -> torch.Tensor:
    """A flat uint8 CUDA tensor holding the bytes of ``buf``.

    CUDA tensors are reinterpreted in place (hashed where they lie); host
    tensors, numpy arrays and bytes-like objects are copied to the device.
    """
    device = device or require_cuda()
    if isinstance(buf, torch.Tensor):
        t = buf.detach()
        if not t.is_contiguous():
            t = t.contiguous()
        t = t.reshape(-1)
        if t.dtype != torch.uint8:
            t = t.view(torch.uint8)
        if t.device.type != "cuda":
            if t.numel() >= STAGE_DIRECT_MAX_BYTES and not t.is_pinned():
                out = torch.empty(t.numel(), dtype=torch.uint8, device=device)
                pageable_to_device(t.numpy(), out)
                return out
            t = t.to(device, non_blocking=True)
        return t
    arr = host_bytes_view(buf)
    if arr.size == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    if arr.size >= STAGE_DIRECT_MAX_BYTES:
        out = torch.empty(arr.size, dtype=torch.uint8, device=device)
        pageable_to_device(arr, out)
        return out
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")          # read-only buffers are only read
        host = torch.from_numpy(arr)
    return host.to(device, non_blocking=True)


class PinnedPack:
    """One reused page-locked block that sequences of host blocks are gathered into (``_hostpack.gather``),
    then copied to the device with one asynchronous transfer. The block is reused once the transfer that
    last read it has completed."""

    MAX_BYTES = 2 << 30                 # larger packs take the staging ring (bounded pinned memory)
    _local = threading.local()

    @classmethod
    def get(cls) -> "PinnedPack":
        inst = getattr(cls._local, "inst", None)
        if inst is None:
            inst = cls._local.inst = cls()
        return inst

    def __init__(self):
        self.block: Optional[torch.Tensor] = None
        self.done: Optional[torch.cuda.Event] = None

    def to_device(self, blocks: Sequence, device: torch.device) -> Optional[Tuple[torch.Tensor, np.ndarray]]:
        """(device bytes, u64 lengths) of the blocks laid back to back, or None when the helper cannot take
        them (not built, an item without a contiguous buffer, a pack above ``MAX_BYTES``)."""
        if _hostpack is None:
            return None
        lens = np.empty(len(blocks), dtype=np.uint64)
        try:
            total = _hostpack.gather(blocks, 0, 0, lens.ctypes.data)
        except (TypeError, BufferError, ValueError):
            return None
        if total > self.MAX_BYTES:
            return None
        if total == 0:
            return torch.zeros(16, dtype=torch.uint8, device=device), lens
        if self.done is not None:
            self.done.synchronize()
        if self.block is None or self.block.numel() < total:
            self.block = torch.empty(max(total, 1 << 20), dtype=torch.uint8, pin_memory=True)
        _hostpack.gather(blocks, self.block.data_ptr(), total, 0)
        out = torch.empty(total, dtype=torch.uint8, device=device)
        out.copy_(self.block[:total], non_blocking=True)
        self.done = torch.cuda.Event()
        self.done.record()
        return out, lens


STAGE_RING_SLOTS = 4
STAGE_SLOT_BYTES = 32 << 20            # one pinned staging buffer = one H2D transfer
STAGE_PIECE_BYTES = 4 << 20            # memcpy granularity handed to the staging threads


class StagingRing:
    """Pinned bounce buffers + memcpy threads for host memory that is not page-locked.

    ``bytes`` / numpy / ordinary CPU tensors cannot be the source of an asynchronous DMA: a plain
    ``cudaMemcpy`` from them runs at ~10 GB/s through the driver's own small bounce buffer. Here a few
    threads copy the pageable bytes into a ring of pinned 32 MB buffers (numpy releases the GIL for
    the memcpy) and every full buffer goes to the device as ONE asynchronous transfer while the next
    buffer is being filled. The ring is created once per process.
    """

    _instance: Optional["StagingRing"] = None

    def __init__(self, threads: int):
        from concurrent.futures import ThreadPoolExecutor

        self.bufs = [torch.empty(STAGE_SLOT_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(STAGE_RING_SLOTS)]
        self.views = [b.numpy() for b in self.bufs]
        self.events: List[Optional[torch.cuda.Event]] = [None] * STAGE_RING_SLOTS
        self.threads = threads
        self.lock = threading.Lock()         # one staged hash at a time owns the ring (hash_model stays thread-safe)
        self.pool = ThreadPoolExecutor(max_workers=threads, thread_name_prefix="snt-stage")
        self.slot = 0

    @classmethod
    def get(cls, threads: int) -> "StagingRing":
        old = cls._instance
        if old is None or old.threads < threads or \
                old.bufs[0].numel() != STAGE_SLOT_BYTES or len(old.bufs) != STAGE_RING_SLOTS:
            cls._instance = cls(threads)
            if old is not None:
                with old.lock:                       # wait for a hash that still owns the old ring
                    old.pool.shutdown(wait=True)
        return cls._instance

    def acquire(self) -> int:
        """Next slot, once the transfer that last used it has completed."""
        slot = self.slot
        self.slot = (slot + 1) % len(self.bufs)
        if self.events[slot] is not None:
            self.events[slot].synchronize()
        return slot


def staging_threads(workers: int = 1) -> int:
    import os

    # Python pool (no helper): 12 copy threads on a 16-core box -- tools/hostcopy_probe.py measures 48 / 54 / 59 GB/s for
    # 8 / 12 / 16 threads. C pool with streaming stores: 8 threads already copy 74 GB/s (tools/ring_probe.py), more only
    # compete with the copy engine for memory bandwidth (GPT2-XL from pageable memory: 139 / 136 / 133 / 139 / 141 ms with
    # 6 / 8 / 10 / 12 / 16 threads); the calling thread and the driver need cores too
    cpus = os.cpu_count() or 1
    forced = os.environ.get("SNT_STAGE_THREADS")           # probes only (tools/host_small_probe.py)
    if forced:
        return max(1, min(16, int(forced)))
    return max(1, min(16, max(int(workers), min(10 if _hostpack is not None else 12, max(1, cpus - 4)))))


STAGE_DIRECT_MAX_BYTES = 8 << 20       # smaller pageable buffers take the plain (synchronous) copy
STAGE_INLINE_MAX_BYTES = 256 << 10     # pieces below this are copied by the calling thread, not the pool


import os as _os

_copy_pool = _hostpack if not _os.environ.get("SNT_NO_COPY_POOL") else None      # A/B switch for tools/host_small_probe.py


class RingWriter:
    """Streams host bytes into a device buffer through the staging ring, keeping the copy threads busy.

    A staging buffer mirrors one contiguous range of the destination: ``[base, base + fill)``. Its memcpy tasks
    are queued on the ring's pool and the buffer is *closed*; the transfer itself is issued later, when the
    tasks have finished -- up to ``MAX_PENDING`` closed buffers wait like that while the caller already queues
    the tasks of the next one, so the pool never drains while the caller waits (the first version waited for
    every buffer before touching the next: 23-30 GB/s from pageable memory on a box whose threads copy 54 GB/s).
    With the C helper the copy threads live in C (``_hostpack.copy_submit`` / ``copy_wait``: 1 MB jobs, no GIL, no
    task objects, **streaming stores** -- the copy engine reads the staging buffer next, and lines left dirty in a
    dozen L2 caches by ordinary stores have to be snooped out by every DMA read: 64 MB through the ring 3.8 -> 1.8 ms,
    a GPT-2-small-sized state dict 19.3 -> 15.5 ms); the Python pool is the path without the helper.
    The caller must hold ``ring.lock``.
    """

    def __init__(self, ring: StagingRing, dst: torch.Tensor, stream: "torch.cuda.Stream"):
        self.ring, self.dst, self.stream = ring, dst, stream
        self.MAX_PENDING = max(0, min(2, len(ring.bufs) - 2))   # the slot being acquired is never one that still waits
        self.slot, self.base, self.fill, self.tasks = -1, 0, 0, []
        self.pending: "collections.deque" = collections.deque()
        self.fd = -1                         # >= 0: the pieces of this writer are file offsets (write_file)
        self.keep: list = []                 # source arrays of the pieces not copied yet

    def write(self, off: int, src: np.ndarray) -> None:
        """Queue the copy of flat uint8 ``src`` to ``dst[off : off + len(src)]``."""
        if _copy_pool is not None:
            if self.fd != -1 and self.tasks:
                self.close()                                # a batch of the C pool reads memory OR one file
            self.fd = -1
            self.keep.append(src)
            self._write(off, int(src.shape[0]), None, src.__array_interface__["data"][0])
        else:
            self._write(off, int(src.shape[0]), lambda view, p0, p1: np.copyto(view, src[p0:p1]), 0)

    def write_file(self, off: int, fd: int, file_off: int, n: int) -> None:
        """Queue ``n`` bytes of the open file ``fd`` from ``file_off`` to ``dst[off : off + n]``: the staging threads
        ``pread`` straight into the pinned buffers (one copy out of the page cache, none through a ``bytes`` object).
        """
        if _copy_pool is not None:
            if self.fd != fd and self.tasks:
                self.close()
            self.fd = fd
            self._write(off, n, None, file_off)
        else:
            self._write(off, n, lambda view, p0, p1: _pread_exact(fd, view, file_off + p0), 0)

    def _write(self, off: int, n: int, copy, src_base: int) -> None:
        """With the C helper the pieces ``(pinned address, source address or file offset, length)`` of a staging
        buffer are collected and copied by its thread pool when the buffer is closed (``copy_many``: no GIL, no
        task objects). Without it ``copy(view, p0, p1)`` fills the pinned ``view`` with source bytes [p0, p1) on the
        Python pool for large pieces."""
        pos = 0
        ring = self.ring
        while pos < n:
            if self.slot < 0:
                self.slot, self.base = ring.acquire(), off + pos
            so = off + pos - self.base
            if so >= STAGE_SLOT_BYTES or so < self.fill:
                self.close()
                continue
            take = min(n - pos, STAGE_SLOT_BYTES - so)
            view = ring.views[self.slot]
            if so > self.fill:
                view[self.fill:so] = 0                      # alignment gap between two buffers: defined bytes
            if copy is None:
                self.tasks += (ring.bufs[self.slot].data_ptr() + so, src_base + pos, take)
            elif take < STAGE_INLINE_MAX_BYTES:             # a task costs more than a small memcpy
                copy(view[so:so + take], pos, pos + take)
            else:
                for p0 in range(0, take, STAGE_PIECE_BYTES):
                    p1 = min(take, p0 + STAGE_PIECE_BYTES)
                    self.tasks.append(ring.pool.submit(copy, view[so + p0:so + p1], pos + p0, pos + p1))
            self.fill = so + take
            pos += take
            if self.fill >= STAGE_SLOT_BYTES:
                self.close()

    def close(self) -> None:
        """End the current staging buffer (the next write starts a new one, at any destination offset)."""
        if self.slot >= 0 and self.fill:
            if _copy_pool is not None:
                # the C pool starts filling the buffer now; the transfer is issued when a later buffer is closed (or at
                # drain), so the threads copy while the caller queues more and the copy engine moves the older buffers
                handle = _copy_pool.copy_submit(self.tasks, self.fd, self.ring.threads)
                self.pending.append((self.slot, self.base, self.fill, (handle, self.keep)))
                self.keep = []
            else:
                self.pending.append((self.slot, self.base, self.fill, self.tasks))
            while len(self.pending) > self.MAX_PENDING:
                self._issue(self.pending.popleft())
        elif self.slot >= 0:
            self.ring.slot = self.slot                      # nothing written: hand the slot back
        self.slot, self.fill, self.tasks = -1, 0, []

    def _issue(self, item) -> None:
        slot, base, fill, tasks = item
        if isinstance(tasks, tuple):
            _copy_pool.copy_wait(tasks[0])                  # (handle, source arrays kept alive until here)
        else:
            for t in tasks:
                t.result()
        with torch.cuda.stream(self.stream):
            self.dst[base:base + fill].copy_(self.ring.bufs[slot][:fill], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.stream)
        self.ring.events[slot] = ev

    def abandon(self) -> None:
        """Wait for every copy still queued without issuing its transfer (error paths: the sources are about to go away)."""
        while self.pending:
            tasks = self.pending.popleft()[3]
            try:
                if isinstance(tasks, tuple):
                    _copy_pool.copy_wait(tasks[0])
                else:
                    for t in tasks:
                        t.exception()
            except OSError:
                pass
        for t in self.tasks:
            if hasattr(t, "exception"):
                t.exception()
        self.slot, self.fill, self.tasks, self.keep = -1, 0, [], []

    def drain(self) -> None:
        """Issue every transfer queued so far (they are then ordered on ``stream``)."""
        self.close()
        while self.pending:
            self._issue(self.pending.popleft())


def pageable_to_device(src: np.ndarray, dst: torch.Tensor, workers: int = 1) -> None:
    """Copy a flat uint8 host array into ``dst`` (flat uint8 CUDA tensor) through the pinned ring.

    The transfers go to the current stream; the call returns after the last one has completed
    (the staging buffers are handed back to the ring only when nothing reads them any more).
    """
    ring = StagingRing.get(staging_threads(workers))
    stream = torch.cuda.current_stream()
    with ring.lock:
        w = RingWriter(ring, dst, stream)
        try:
            w.write(0, src)
            w.drain()
        finally:
            w.abandon()
            stream.synchronize()  # the ring may be handed to another caller / stream after the lock is released


def _pread_exact(fd: int, view: np.ndarray, file_off: int) -> None:
    import os

    mv, got = memoryview(view), 0
    while got < len(mv):
        r = os.preadv(fd, [mv[got:]], file_off + got)
        if r <= 0:
            raise OSError(f"short read at byte {file_off + got}")
        got += r


def read_file_host(path, workers: int = 1) -> np.ndarray:
    """The bytes of a file as one uint8 array in (pageable) host memory. Large files are read by the C pool's
    threads in parallel (``pread`` of 1 MB jobs straight into the array, whose pages the threads also fault in):
    ``Path.read_bytes`` moves 2.5 GB/s on one thread. Raises ``OSError`` like ``open``/``read``."""
    import os

    with open(path, "rb", buffering=0) as f:
        size = os.fstat(f.fileno()).st_size
        if _hostpack is None or size < STAGE_DIRECT_MAX_BYTES:
            return np.frombuffer(f.read(), dtype=np.uint8)
        out = np.empty(size, dtype=np.uint8)
        _hostpack.copy_many([out.ctypes.data, 0, size], f.fileno(), staging_threads(workers))
    return out


def file_to_device(path, device: Optional[torch.device] = None, workers: int = 1) -> torch.Tensor:
    """The bytes of a file as a flat uint8 CUDA tensor. Large files are read by the staging threads straight into
    the pinned ring and transferred buffer by buffer while the next one is being read (``read_bytes`` + copy of a
    150 MB shard: 59 + 7 ms; this: one pass at the speed of the page cache). Raises ``OSError`` like ``open``/``read``."""
    import os

    device = device or require_cuda()
    with open(path, "rb", buffering=0) as f:
        size = os.fstat(f.fileno()).st_size
        if size < STAGE_DIRECT_MAX_BYTES:
            return as_device_bytes(f.read(), device)
        out = torch.empty(size, dtype=torch.uint8, device=device)
        ring = StagingRing.get(staging_threads(workers))
        stream = torch.cuda.current_stream()
        with ring.lock:
            w = RingWriter(ring, out, stream)
            try:
                w.write_file(0, f.fileno(), 0, size)
                w.drain()
            finally:
                w.abandon()                                              # no copy may outlive the file descriptor
                stream.synchronize()
    return out


ARENA_ALIGN = 256


def file_ranges_to_device(fd: int, ranges: Sequence[Tuple[int, int]], device: Optional[torch.device] = None,
                          workers: int = 1) -> List[torch.Tensor]:
    """Byte ranges ``(offset, nbytes)`` of the open file ``fd`` as flat uint8 CUDA tensors (views of ONE arena), read
    by the staging threads straight into the pinned ring: a rank of a sharded hash reads only the tensors it owns."""
    device = device or require_cuda()
    offs, pos = [], 0
    for _, n in ranges:
        offs.append(pos)
        pos += -(-n // ARENA_ALIGN) * ARENA_ALIGN
    arena = torch.empty(max(pos, 16), dtype=torch.uint8, device=device)
    ring = StagingRing.get(staging_threads(workers))
    stream = torch.cuda.current_stream()
    with ring.lock:
        w = RingWriter(ring, arena, stream)
        try:
            for (file_off, n), off in zip(ranges, offs):
                if n:
                    w.write_file(off, fd, file_off, n)
            w.drain()
        finally:
            w.abandon()
            stream.synchronize()
    return [arena[off:off + n] for (_, n), off in zip(ranges, offs)]


def _host_array(buf) -> np.ndarray:
    """Flat uint8 numpy view of a host buffer (bytes-like, numpy array or CPU tensor); zero copy when contiguous."""
    if isinstance(buf, torch.Tensor):
        t = buf.detach()
        t = t if t.is_contiguous() else t.contiguous()
        t = t.reshape(-1)
        return (t if t.dtype == torch.uint8 else t.view(torch.uint8)).numpy()
    return host_bytes_view(buf)


def pageable_arena(arrays: Sequence[np.ndarray], device: torch.device, workers: int = 1):
    """Lay host arrays back to back (256-byte aligned) in ONE device buffer, filled through the pinned ring.

    Returns (arena tensor, byte offset of every array). Transfers are enqueued on the current stream.
    """
    offs, total = [], 0
    for a in arrays:
        offs.append(total)
        total += -(-int(a.shape[0]) // ARENA_ALIGN) * ARENA_ALIGN
    arena = torch.empty(max(total, 16), dtype=torch.uint8, device=device)
    ring = StagingRing.get(staging_threads(workers))
    stream = torch.cuda.current_stream()
    with ring.lock:
        w = RingWriter(ring, arena, stream)
        try:
            for a, off in zip(arrays, offs):
                w.write(off, a)
            w.drain()
        finally:
            w.abandon()
            stream.synchronize()      # the ring goes back to the pool only when no transfer still reads it
    return arena, offs


def device_spans(buffers: Sequence[object], device: Optional[torch.device] = None, workers: int = 1):
    """(keep-alive list, addresses, byte lengths) of the buffers' bytes in HBM, in order.

    The fast path of the drop-in API: a contiguous CUDA tensor is described by its
    ``data_ptr()`` and ``nbytes`` alone -- no detach / reshape / view per tensor, which for a
    581-tensor state dict costs more host time than a GPT-2 small hash takes on the GPU.
    Host memory is staged: pinned tensors and small buffers by a direct copy each; when the
    pageable buffers add up to more than a few MB they are packed into one device arena
    through the pinned staging ring (``pageable_arena``) instead of one slow copy per buffer.
    """
    device = device or require_cuda()
    n = len(buffers)
    keep: List[object] = [None] * n
    ptrs = np.zeros(max(n, 1), dtype=np.uint64)
    sizes = np.zeros(max(n, 1), dtype=np.uint64)
    pageable: List[int] = []
    for i, buf in enumerate(buffers):
        if type(buf) is torch.Tensor and buf.is_cuda and buf.is_contiguous():
            pass
        elif isinstance(buf, torch.Tensor) and (buf.is_cuda or buf.is_pinned()):
            buf = as_device_bytes(buf, device)
        else:
            pageable.append(i)
            continue
        nbytes = buf.nbytes
        keep[i] = buf
        sizes[i] = nbytes
        if nbytes:
            ptrs[i] = buf.data_ptr()
    if pageable:
        arrays = [_host_array(buffers[i]) for i in pageable]
        if sum(int(a.shape[0]) for a in arrays) >= STAGE_DIRECT_MAX_BYTES:
            arena, offs = pageable_arena(arrays, device, workers)
            base = arena.data_ptr()
            for i, a, off in zip(pageable, arrays, offs):
                keep[i] = arena
                sizes[i] = int(a.shape[0])
                if sizes[i]:
                    ptrs[i] = base + off
        else:
            for i in pageable:
                t = as_device_bytes(buffers[i], device)
                keep[i], sizes[i] = t, t.nbytes
                if t.nbytes:
                    ptrs[i] = t.data_ptr()
    return keep, ptrs, sizes


def gather_spans(src_addr: np.ndarray, lengths: np.ndarray, dst_off: np.ndarray, pad_block: int,
                 dst: torch.Tensor) -> None:
    """``snt_gather_spans``: copy span i (``lengths[i]`` bytes at device address ``src_addr[i]``) to
    ``dst[dst_off[i]:]``, zero-padded to a multiple of ``pad_block`` when that is non-zero. One launch."""
    lib = _native.load()
    n = int(lengths.shape[0])
    if n == 0:
        return
    lengths = lengths.astype(np.uint64, copy=False)
    padded = lengths if not pad_block else (lengths + np.uint64(pad_block - 1)) // np.uint64(pad_block) * np.uint64(pad_block)
    chunk = int(lib.snt_gather_chunk_bytes())
    chunk_first = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum((padded + np.uint64(chunk - 1)) // np.uint64(chunk), out=chunk_first[1:])
    n_chunks = int(chunk_first[-1])
    if n_chunks == 0:
        return
    table = np.concatenate([src_addr.astype(np.uint64, copy=False), lengths, dst_off.astype(np.uint64, copy=False),
                            chunk_first])
    d_table = torch.from_numpy(table.view(np.int64)).to(dst.device, non_blocking=False)
    base = d_table.data_ptr()
    rc = lib.snt_gather_spans(ctypes.c_void_p(base), ctypes.c_void_p(base + 8 * n), ctypes.c_void_p(base + 16 * n),
                              ctypes.c_void_p(base + 24 * n), n, n_chunks, pad_block, _ptr(dst), _stream())
    _native.check(rc, "snt_gather_spans")
    d_table.record_stream(torch.cuda.current_stream())


class ModelPlan:
    """Device-side block table over fragmented tensors (``snt_model_plan``).

    Replaces ``BlockTable.build`` (reference model.py:137-146) for the kernels:
    one row per tensor instead of one row per block. Keeps the tensors alive.
    """

    def __init__(self, tensors: Sequence[torch.Tensor], block_size: int,
                 sizes_override: Optional[Sequence[int]] = None):
        """``sizes_override[i]`` gives tensor i's true byte length when ``tensors[i]`` is only a
        placeholder (a tensor this rank never reads because its leaves belong to other ranks)."""
        self._handle = ctypes.c_void_p()
        lib = _native.load()
        require_cuda()
        self.tensors = list(tensors)
        n = len(self.tensors)
        ptrs = (ctypes.c_void_p * max(n, 1))()
        sizes = (ctypes.c_uint64 * max(n, 1))()
        for i, t in enumerate(self.tensors):
            if t.device.type != "cuda" or t.dtype != torch.uint8 or t.dim() != 1:
                raise InvalidInput("ModelPlan needs flat uint8 CUDA tensors")
            nbytes = t.numel() if sizes_override is None else int(sizes_override[i])
            ptrs[i] = t.data_ptr() if nbytes else None
            sizes[i] = nbytes
        rc = lib.snt_model_plan_create(ptrs, sizes, n, block_size, _stream(), ctypes.byref(self._handle))
        _native.check(rc, "snt_model_plan_create")
        self.block_size = block_size
        self.leaf_count = int(lib.snt_model_plan_leaf_count(self._handle))
        self.total_bytes = int(lib.snt_model_plan_total_bytes(self._handle))

    @classmethod
    def from_spans(cls, keep: Sequence[object], ptrs: np.ndarray, sizes: np.ndarray, block_size: int,
                   count: Optional[int] = None) -> "ModelPlan":
        """Plan over ``device_spans`` output (addresses + byte lengths; ``keep`` holds the owners alive).
        ``count`` = number of spans when ``keep`` is not one object per span."""
        self = cls.__new__(cls)
        self._handle = ctypes.c_void_p()
        lib = _native.load()
        require_cuda()
        self.tensors = list(keep)
        rc = lib.snt_model_plan_create(ptrs.ctypes.data_as(ctypes.POINTER(ctypes.c_void_p)),
                                       sizes.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                       len(keep) if count is None else count, block_size,
                                       _stream(), ctypes.byref(self._handle))
        _native.check(rc, "snt_model_plan_create")
        self.block_size = block_size
        self.leaf_count = int(lib.snt_model_plan_leaf_count(self._handle))
        self.total_bytes = int(lib.snt_model_plan_total_bytes(self._handle))
        return self

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._handle

    def close(self) -> None:
        if self._handle:
            _native.load().snt_model_plan_destroy(self._handle)
            self._handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def merkle_work_bytes(alg: str, count: int) -> int:
    return int(_native.load().snt_merkle_work_bytes(ALG_IDS[alg], count))


def ceil_log2(n: int) -> int:
    return 0 if n <= 1 else (n - 1).bit_length()


class MerkleModelHasher:
    """Reusable launch state for in-place Merkle hashing of one model.

    Holds the plan and the device buffers (leaf digests, reducer scratch,
    output nodes) so that ``run`` only enqueues kernels -- no allocation, no
    synchronisation. ``leaf_begin``/``leaf_end``/``levels`` select a shard
    (multi-GPU); the defaults hash the whole model down to the root.
    """

    def __init__(self, plan: ModelPlan, alg: str, leaf_begin: int = 0, leaf_end: Optional[int] = None,
                 levels: Optional[int] = None, out_capacity: Optional[int] = None, host_out: bool = False):
        """``out_capacity`` (in digests) over-allocates the zero-filled output buffer so that a rank's
        shard roots can be handed to an all-gather of fixed-size slots without a staging copy.
        ``host_out`` puts the output nodes in page-locked HOST memory: the last kernel of the hash stores the
        root through the unified address space, so reading it needs a stream synchronisation and no copy."""
        self.plan = plan
        self.alg = alg
        self.dlen = DIGEST_LEN[alg]
        n = plan.leaf_count
        self.leaf_begin = leaf_begin
        self.leaf_end = n if leaf_end is None else leaf_end
        if not (0 <= self.leaf_begin < self.leaf_end <= n):
            raise InvalidInput("empty or out-of-range leaf range")
        self.levels = levels
        count = self.leaf_end - self.leaf_begin
        dev = require_cuda()
        self.n_out = 1 if levels is None else -(-count // (1 << levels))
        self.leaves = torch.empty(count * self.dlen, dtype=torch.uint8, device=dev)
        self.work_bytes = merkle_work_bytes(alg, count)
        # zeroed once: the fused kernel keeps its completion counters at zero between launches
        self.work = torch.zeros(max(self.work_bytes, 16), dtype=torch.uint8, device=dev)
        n_out_bytes = max(self.n_out, out_capacity or 0) * self.dlen
        if host_out:
            self.out_padded = torch.zeros(n_out_bytes, dtype=torch.uint8, pin_memory=True)
        else:
            self.out_padded = torch.zeros(n_out_bytes, dtype=torch.uint8, device=dev)
        self.out = self.out_padded[:self.n_out * self.dlen]

    def run(self) -> None:
        lib = _native.load()
        levels = _native.SNT_LEVELS_TO_ROOT if self.levels is None else self.levels
        rc = lib.snt_merkle_inplace(self.plan.handle, ALG_IDS[self.alg], self.leaf_begin, self.leaf_end,
                                    levels, _ptr(self.leaves), _ptr(self.work), self.work_bytes,
                                    _ptr(self.out), _stream())
        _native.check(rc, "snt_merkle_inplace")

    def capture(self) -> "torch.cuda.CUDAGraph":
        """Record ``run`` (leaf launch + level-reducer launches) into a CUDA graph.

        ``graph.replay()`` then re-hashes whatever bytes the tensors hold at replay time into
        ``self.out`` with one submission instead of three launches -- for callers that re-hash
        the same model every few steps (small models are launch-latency sensitive: GPT-2 small
        is one wave of CTAs). The first ``run`` happens outside the capture so that one-time
        function-attribute calls are not recorded.
        """
        self.run()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self.run()
        return graph

    def run_leaves_only(self, begin: Optional[int] = None, end: Optional[int] = None) -> None:
        """The leaf stage alone (``snt_merkle_leaves``) over [begin, end) of this hasher's range."""
        lib = _native.load()
        begin = self.leaf_begin if begin is None else begin
        end = self.leaf_end if end is None else end
        out = self.leaves[(begin - self.leaf_begin) * self.dlen:]
        rc = lib.snt_merkle_leaves(self.plan.handle, ALG_IDS[self.alg], begin, end, _ptr(out), _stream())
        _native.check(rc, "snt_merkle_leaves")

    def run_tree_only(self) -> None:
        """Reduce the leaf digests already in ``self.leaves`` to the root (whole-model hashers only)."""
        if self.levels is not None or self.leaf_begin != 0 or self.leaf_end != self.plan.leaf_count:
            raise InvalidInput("run_tree_only needs a whole-model hasher")
        lib = _native.load()
        rc = lib.snt_merkle_root(ALG_IDS[self.alg], _ptr(self.leaves), self.plan.leaf_count, _ptr(self.work),
                                 self.work_bytes, _ptr(self.out), _stream())
        _native.check(rc, "snt_merkle_root")

    def out_bytes(self) -> bytes:
        return self.out.cpu().numpy().tobytes()

    def leaf_bytes(self) -> bytes:
        return self.leaves.cpu().numpy().tobytes()


def hash_blocks_device(alg: str, base: Optional[torch.Tensor], offsets: torch.Tensor, lengths: torch.Tensor,
                       out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """``snt_hash_blocks``: digests of blocks ``base[off[i] : off[i] + len[i]]`` (device arrays)."""
    lib = _native.load()
    dev = require_cuda()
    n = int(offsets.numel())
    dlen = DIGEST_LEN[alg]
    if out is None:
        out = torch.empty(n * dlen, dtype=torch.uint8, device=dev)
    rc = lib.snt_hash_blocks(ALG_IDS[alg], _ptr(base), _ptr(offsets), _ptr(lengths), n, _ptr(out), _stream())
    _native.check(rc, "snt_hash_blocks")
    return out


def merkle_root_device(alg: str, nodes: torch.Tensor, count: int) -> torch.Tensor:
    """``snt_merkle_root`` over ``count`` digests held in a flat uint8 CUDA tensor."""
    lib = _native.load()
    dev = require_cuda()
    dlen = DIGEST_LEN[alg]
    wb = merkle_work_bytes(alg, count)
    work = torch.empty(max(wb, 16), dtype=torch.uint8, device=dev)
    root = torch.empty(dlen, dtype=torch.uint8, device=dev)
    rc = lib.snt_merkle_root(ALG_IDS[alg], _ptr(nodes), count, _ptr(work), wb, _ptr(root), _stream())
    _native.check(rc, "snt_merkle_root")
    return root


def merkle_root_into(alg: str, nodes: torch.Tensor, count: int, work: torch.Tensor, work_bytes: int,
                     root: torch.Tensor) -> torch.Tensor:
    """``snt_merkle_root`` with caller-owned workspace and root buffer (no allocation, no synchronisation)."""
    rc = _native.load().snt_merkle_root(ALG_IDS[alg], _ptr(nodes), count, _ptr(work), work_bytes, _ptr(root), _stream())
    _native.check(rc, "snt_merkle_root")
    return root


def merkle_reduce_levels_device(alg: str, nodes: torch.Tensor, first: int, n_in: int, level_count: int,
                                levels: int) -> torch.Tensor:
    """``snt_merkle_reduce_levels``: apply ``levels`` tree levels to a node range."""
    lib = _native.load()
    dev = require_cuda()
    dlen = DIGEST_LEN[alg]
    n_out = -(-n_in // (1 << levels))
    wb = merkle_work_bytes(alg, n_in)
    work = torch.empty(max(wb, 16), dtype=torch.uint8, device=dev)
    out = torch.empty(n_out * dlen, dtype=torch.uint8, device=dev)
    rc = lib.snt_merkle_reduce_levels(ALG_IDS[alg], _ptr(nodes), first, n_in, level_count, levels,
                                      _ptr(work), wb, _ptr(out), _stream())
    _native.check(rc, "snt_merkle_reduce_levels")
    return out


def merkle_roots_segmented_device(alg: str, digests: torch.Tensor, seg_first: Sequence[int],
                                  empty_digest: torch.Tensor) -> torch.Tensor:
    """``snt_merkle_roots_segmented``: one tree per segment of a digest array (per-layer Merkle)."""
    lib = _native.load()
    dev = require_cuda()
    dlen = DIGEST_LEN[alg]
    n_seg = len(seg_first) - 1
    counts = [b - a for a, b in zip(seg_first[:-1], seg_first[1:])]
    widest = max(counts)
    # workspace: the reducer chain's buffers for the widest tree, or one node per 512 leaf digests of every large
    # tree (the first launch of the segmented reducer leaves its level-9/10 nodes there), whichever is more
    wb = max(merkle_work_bytes(alg, max(widest, 1)), sum(-(-c // 512) for c in counts if c > 512) * dlen)
    work = torch.empty(max(wb, 16), dtype=torch.uint8, device=dev)
    out = torch.empty(n_seg * dlen, dtype=torch.uint8, device=dev)
    first = (ctypes.c_uint64 * (n_seg + 1))(*seg_first)
    rc = lib.snt_merkle_roots_segmented(ALG_IDS[alg], _ptr(digests), first, n_seg, _ptr(empty_digest), _ptr(work),
                                        wb, _ptr(out), _stream())
    _native.check(rc, "snt_merkle_roots_segmented")
    return out


class LatticeAccumulator:
    """Device-resident per-source LtHash sums: ``n_sources x 32`` u64 lanes, u64 counts, a status word.

    The running state of ``SourceAccumulator`` (reference dataset.py:52-71) kept
    in HBM as ONE int64 array ``state = [lanes | counts | status]`` (``acc``, ``counts`` and
    ``status`` are views of it), so the partial accumulators of several GPUs combine with a
    single sum all-reduce of ``state`` and nothing is packed or unpacked. Lanes are summed
    modulo 2^64 and masked to 16 bits by ``digests``: exact modulo 2^16 for any number of
    samples. ``status`` counts the samples that named an undeclared source.
    """

    def __init__(self, n_sources: int):
        dev = require_cuda()
        if n_sources < 1:
            raise InvalidInput("at least one source slot is required")
        self.n_sources = n_sources
        self.state = torch.zeros(n_sources * (LT_LANES + 1) + 1, dtype=torch.int64, device=dev)
        self.acc = self.state[:n_sources * LT_LANES]
        self.counts = self.state[n_sources * LT_LANES:n_sources * (LT_LANES + 1)]
        self.status = self.state[n_sources * (LT_LANES + 1):]
        self._out_host: Optional[torch.Tensor] = None

    def zero_(self) -> None:
        self.state.zero_()

    def add_samples(self, shard: torch.Tensor, offsets: torch.Tensor, lengths: torch.Tensor,
                    ids: torch.Tensor, slots: torch.Tensor, digests: Optional[torch.Tensor] = None,
                    uniform: Optional[bool] = None) -> None:
        """``uniform``: what the caller knows about ``lengths`` (True = all equal, False = ragged, None =
        unknown); it only selects the launch (``snt_lthash_samples_shaped``), never the result."""
        lib = _native.load()
        n = int(offsets.numel())
        shape = _native.SAMPLES_UNKNOWN if uniform is None else (_native.SAMPLES_UNIFORM if uniform else _native.SAMPLES_RAGGED)
        rc = lib.snt_lthash_samples_shaped(_ptr(shard), _ptr(offsets), _ptr(lengths), _ptr(ids), _ptr(slots), n,
                                           self.n_sources, _ptr(self.acc), _ptr(self.counts), _ptr(digests),
                                           _ptr(self.status), shape, _stream())
        _native.check(rc, "snt_lthash_samples_shaped")

    def add_packed(self, block: torch.Tensor, n: int, header: int, uniform: Optional[bool] = None) -> None:
        """A batch in the one-block layout ``offsets[n] u64 | lengths[n] u64 | ids[n] u64 | slots[n] i32 | pad |
        sample bytes (from byte ``header``)`` -- what ``process_batch`` ships per batch; addresses by arithmetic,
        no tensor views."""
        lib = _native.load()
        base = block.data_ptr()
        shape = _native.SAMPLES_UNKNOWN if uniform is None else (_native.SAMPLES_UNIFORM if uniform else _native.SAMPLES_RAGGED)
        vp = ctypes.c_void_p
        rc = lib.snt_lthash_samples_shaped(vp(base + header), vp(base), vp(base + 8 * n), vp(base + 16 * n), vp(base + 24 * n),
                                           n, self.n_sources, _ptr(self.acc), _ptr(self.counts), None,
                                           _ptr(self.status), shape, _stream())
        _native.check(rc, "snt_lthash_samples_shaped")

    def add_rows(self, rows: torch.Tensor, row_bytes: int, n: int, ids: torch.Tensor, source_ids: torch.Tensor,
                 table: torch.Tensor, digests: Optional[torch.Tensor] = None) -> None:
        """``snt_lthash_rows``: n rows of ``row_bytes`` bytes in one flat device tensor, raw source ids (int64) looked up
        in ``table`` (the declared ids, sorted, int64, on the device) inside the kernel. One launch."""
        lib = _native.load()
        rc = lib.snt_lthash_rows(_ptr(rows), row_bytes, n, _ptr(ids), _ptr(source_ids), _ptr(table), self.n_sources,
                                 _ptr(self.acc), _ptr(self.counts), _ptr(digests), _ptr(self.status), _stream())
        _native.check(rc, "snt_lthash_rows")

    def add_model_leaves(self, plan: ModelPlan, leaf_begin: int, leaf_end: int,
                         digests: Optional[torch.Tensor] = None) -> None:
        lib = _native.load()
        rc = lib.snt_lthash_model(plan.handle, leaf_begin, leaf_end, _ptr(self.acc), _ptr(self.counts),
                                  _ptr(digests), _stream())
        _native.check(rc, "snt_lthash_model")

    def add_digests(self, digests: torch.Tensor, n: int) -> None:
        lib = _native.load()
        rc = lib.snt_lt_reduce(_ptr(digests), n, _ptr(self.acc), _stream())
        _native.check(rc, "snt_lt_reduce")

    def add_model_layers(self, plan: ModelPlan, leaf_begin: int, leaf_end: int) -> None:
        """Per-layer lattice: block j of tensor i tagged LE64(i) || LE64(j), summed into slot i."""
        lib = _native.load()
        rc = lib.snt_lthash_model_layers(plan.handle, leaf_begin, leaf_end, _ptr(self.acc), _ptr(self.counts),
                                         None, _stream())
        _native.check(rc, "snt_lthash_model_layers")

    def finalize_device(self) -> torch.Tensor:
        """``n_sources x 64`` digest bytes as a device tensor (no synchronisation)."""
        lib = _native.load()
        out = torch.empty(self.n_sources * 64, dtype=torch.uint8, device=self.acc.device)
        rc = lib.snt_lt_finalize(_ptr(self.acc), self.n_sources, _ptr(out), _stream())
        _native.check(rc, "snt_lt_finalize")
        return out

    def finalize_to_host(self) -> None:
        """Enqueue the read-out (no synchronisation): the finalize kernel stores the ``n_sources x 64`` digest bytes
        straight into page-locked host memory through the unified address space, counts and status follow as one
        asynchronous copy into the same block. ``host_result`` reads it after the stream has been synchronised."""
        lib = _native.load()
        n = self.n_sources
        if self._out_host is None:
            self._out_host = torch.empty(n * 64 + (n + 1) * 8, dtype=torch.uint8, pin_memory=True)
        if lib.snt_device_reads_pinned_host():
            rc = lib.snt_lt_finalize(_ptr(self.acc), n, _ptr(self._out_host), _stream())
            _native.check(rc, "snt_lt_finalize")
        else:
            self._out_host[:n * 64].copy_(self.finalize_device(), non_blocking=True)
        self._out_host[n * 64:].view(torch.int64).copy_(self.state[n * LT_LANES:], non_blocking=True)

    def host_result(self) -> Tuple[bytes, List[int], int]:
        n = self.n_sources
        host = self._out_host.numpy()
        tail = host[n * 64:].view(np.int64).tolist()
        return host[:n * 64].tobytes(), [int(c) for c in tail[:-1]], int(tail[-1])

    def digests(self) -> Tuple[bytes, List[int], int]:
        """(n_sources x 64 digest bytes, counts, status bits); synchronises (once)."""
        self.finalize_to_host()
        torch.cuda.current_stream().synchronize()
        return self.host_result()
