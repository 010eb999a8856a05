"""Two-stage Merkle construction on the GPU: block hashing, then level reduction.

Same names, arguments and results as the reference's ``merkle.py`` (:20-171):

* ``hash_blocks``  -> ``snt_hash_blocks``  (one thread per block)
* ``reduce_level`` -> ``snt_merkle_reduce_levels`` with ``levels=1``
* ``merkle_root``  -> ``snt_merkle_root``  (all levels in a few launches)

The tree rule is the reference's (merkle.py:117-149): parent = H(left || right),
an odd level pairs its last node with ``digest_len`` zero bytes, a single leaf
is its own root. ``workers`` is accepted and ignored (the grid is the pool).

These functions take and return host buffers like the reference does; the
device-resident model path is ``model.inplace_hash`` / ``device.MerkleModelHasher``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import device as _dev
from .compression import CompressionAlg, Digest
from .errors import InvalidInput, InvalidState


@dataclass
class DigestBuffer:
    """``count`` digests of one algorithm, back to back in a host ``bytearray``."""

    alg: CompressionAlg
    data: bytearray
    count: int

    @classmethod
    def allocate(cls, alg: CompressionAlg, capacity: int) -> "DigestBuffer":
        return cls(alg, bytearray(capacity * alg.digest_len), 0)

    @classmethod
    def from_digests(cls, alg: CompressionAlg, digests: Sequence[Digest]) -> "DigestBuffer":
        return cls(alg, bytearray(b"".join(d.data for d in digests)), len(digests))

    @property
    def digest_len(self) -> int:
        return self.alg.digest_len

    @property
    def nbytes(self) -> int:
        return len(self.data)

    def entry(self, i: int) -> bytes:
        n = self.digest_len
        return bytes(self.data[i * n:(i + 1) * n])

    def entries(self) -> list:
        return [self.entry(i) for i in range(self.count)]


@dataclass
class ReductionState:
    """Two digest buffers whose input/output roles swap after every level (merkle.py:57-90)."""

    buffer_a: DigestBuffer
    buffer_b: DigestBuffer
    active: int = 0

    @classmethod
    def from_leaves(cls, leaves: DigestBuffer) -> "ReductionState":
        # buffer_a is the leaf buffer itself; only buffer_b is new storage
        return cls(leaves, DigestBuffer.allocate(leaves.alg, max(1, (leaves.count + 1) // 2)))

    @property
    def input_buffer(self) -> DigestBuffer:
        return self.buffer_b if self.active else self.buffer_a

    @property
    def output_buffer(self) -> DigestBuffer:
        return self.buffer_a if self.active else self.buffer_b

    @property
    def aux_bytes(self) -> int:
        return self.buffer_b.nbytes


def _stage_blocks(blocks: Sequence):
    """Pack host blocks into one device buffer; returns (base, offsets, lengths).

    Blocks that already live on the GPU are addressed where they lie.
    """
    dev = _dev.require_cuda()
    n = len(blocks)
    if all(isinstance(b, torch.Tensor) and b.device.type == "cuda" for b in blocks):
        keep = [_dev.as_device_bytes(b) for b in blocks]
        offs = np.array([t.data_ptr() if t.numel() else 0 for t in keep], dtype=np.uint64)
        lens = np.array([t.numel() for t in keep], dtype=np.uint64)
        base = None
    else:
        host = [b.cpu().numpy() if isinstance(b, torch.Tensor) else b for b in blocks] \
            if any(isinstance(b, torch.Tensor) for b in blocks) else blocks
        packed = _dev.PinnedPack.get().to_device(host, dev)      # one C pass over the buffers into pinned memory
        if packed is not None:
            base, lens = packed
        else:
            views = [_dev.host_bytes_view(b) for b in host]
            lens = np.fromiter((v.size for v in views), dtype=np.uint64, count=n)
            total = int(lens.sum())
            flat = np.concatenate(views) if total else np.zeros(0, dtype=np.uint8)
            # (large packs travel through the pinned staging ring: ~50 GB/s instead of a pageable cudaMemcpy's ~10)
            base = _dev.as_device_bytes(flat, dev) if total else torch.zeros(16, dtype=torch.uint8, device=dev)
        offs = np.zeros(n, dtype=np.uint64)
        if n > 1:
            np.cumsum(lens[:-1], out=offs[1:])
        keep = [base]
    d_off = torch.from_numpy(offs.view(np.int64)).to(dev)
    d_len = torch.from_numpy(lens.view(np.int64)).to(dev)
    return base, d_off, d_len, keep


def hash_blocks(alg: CompressionAlg, blocks: Sequence, workers: int = 1) -> DigestBuffer:
    """Entry i is the digest of block i (merkle.py:93-114); zero blocks -> ``InvalidInput``."""
    n = len(blocks)
    if n == 0:
        raise InvalidInput("hash_blocks requires at least one block")
    base, d_off, d_len, _keep = _stage_blocks(blocks)
    out = _dev.hash_blocks_device(alg.value, base, d_off, d_len)
    return DigestBuffer(alg, bytearray(out.cpu().numpy().tobytes()), n)


def reduce_level(state: ReductionState, workers: int = 1) -> int:
    """One tree level on the GPU, then swap the buffers; returns ceil(count / 2) (merkle.py:117-149)."""
    inp, out = state.input_buffer, state.output_buffer
    count = inp.count
    if count < 2:
        raise InvalidState("reduce_level requires at least two digests")
    dlen = inp.digest_len
    dev = _dev.require_cuda()
    nodes = _dev.as_device_bytes(np.frombuffer(inp.data, dtype=np.uint8, count=count * dlen), dev)
    res = _dev.merkle_reduce_levels_device(inp.alg.value, nodes, 0, count, count, 1)
    pairs = (count + 1) // 2
    out.data[:pairs * dlen] = res.cpu().numpy().tobytes()
    out.count = pairs
    state.active ^= 1
    return pairs


def merkle_root(alg: CompressionAlg, leaves: DigestBuffer, workers: int = 1) -> Digest:
    """Root of the tree over ``leaves``; one leaf is returned unchanged (merkle.py:152-165)."""
    if leaves.count == 0:
        raise InvalidInput("merkle_root requires at least one leaf")
    dlen = alg.digest_len
    dev = _dev.require_cuda()
    nodes = _dev.as_device_bytes(np.frombuffer(leaves.data, dtype=np.uint8, count=leaves.count * dlen), dev)
    root = _dev.merkle_root_device(alg.value, nodes, leaves.count)
    return Digest(alg, root.cpu().numpy().tobytes())


def merkle_root_of_digests(alg: CompressionAlg, digests: Sequence[Digest], workers: int = 1) -> Digest:
    """Build a leaf buffer from ``digests`` and reduce it (merkle.py:168-171)."""
    return merkle_root(alg, DigestBuffer.from_digests(alg, digests), workers)
