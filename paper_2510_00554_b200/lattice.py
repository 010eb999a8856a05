"""LtHash: order-invariant lattice hashing over BLAKE2b-512 digests.

API mirror of the reference's ``lattice.py`` (:22-134). A lattice digest is 64
bytes = 32 little-endian u16 lanes combined by per-lane addition modulo 2^16.

* hashing (``lt_hash_block`` / ``lt_hash_tagged``) and bulk summation
  (``lt_reduce``) run on the GPU (``snt_lthash_samples``, ``snt_lt_reduce``);
* ``lt_add`` / ``lt_sub`` on two 64-byte host values are plain integer
  arithmetic on the host, like the ECDSA step: they combine final digests,
  they are not the accumulation path (that is ``device.LatticeAccumulator``).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np
import torch

from . import device as _dev

DIGEST_BYTES = 64
WORDS = 8
PARTITIONS = 32
PARTITION_BITS = 16
PARTITION_MOD = 1 << PARTITION_BITS

_LANES = struct.Struct("<32H")
_WORDS = struct.Struct("<8Q")


@dataclass(frozen=True)
class LatticeDigest:
    """64 bytes: 8 x 64-bit words, each packing four 16-bit lanes."""

    data: bytes

    def __post_init__(self):
        if len(self.data) != DIGEST_BYTES:
            raise ValueError(f"lattice digest must be {DIGEST_BYTES} bytes, got {len(self.data)}")

    def words(self) -> tuple:
        return _WORDS.unpack(self.data)

    def partitions(self) -> tuple:
        return _LANES.unpack(self.data)

    def hex(self) -> str:
        return self.data.hex()

    @classmethod
    def from_hex(cls, s: str) -> "LatticeDigest":
        return cls(bytes.fromhex(s))


_ZERO = LatticeDigest(bytes(DIGEST_BYTES))


def lt_zero() -> LatticeDigest:
    """The additive identity."""
    return _ZERO


def lt_add(a: LatticeDigest, b: LatticeDigest) -> LatticeDigest:
    """Lane-wise sum modulo 2^16 (lattice.py:69-82)."""
    return LatticeDigest(_LANES.pack(*((x + y) & 0xFFFF for x, y in zip(a.partitions(), b.partitions()))))


def lt_sub(a: LatticeDigest, b: LatticeDigest) -> LatticeDigest:
    """Lane-wise difference modulo 2^16; undoes ``lt_add`` (lattice.py:85-89)."""
    return LatticeDigest(_LANES.pack(*((x - y) & 0xFFFF for x, y in zip(a.partitions(), b.partitions()))))


def _hash_one(tag: bytes, data) -> LatticeDigest:
    """BLAKE2b-512(tag || data) on the GPU for one item.

    An 8-byte tag takes the tagged LtHash kernel (the tag becomes message word
    0); any other tag length hashes the concatenation as a plain block.
    """
    dev = _dev.require_cuda()
    if len(tag) == 8:
        acc = _dev.LatticeAccumulator(1)
        payload = _dev.as_device_bytes(data, dev)
        shard = payload if payload.numel() else torch.zeros(16, dtype=torch.uint8, device=dev)
        off = torch.zeros(1, dtype=torch.int64, device=dev)
        ln = torch.tensor([payload.numel()], dtype=torch.int64, device=dev)
        ids = torch.from_numpy(np.frombuffer(tag, dtype=np.int64).copy()).to(dev)
        slot = torch.zeros(1, dtype=torch.int32, device=dev)
        out = torch.empty(64, dtype=torch.uint8, device=dev)
        acc.add_samples(shard, off, ln, ids, slot, digests=out, uniform=True)
        return LatticeDigest(out.cpu().numpy().tobytes())
    from .compression import CompressionAlg
    from .merkle import hash_blocks

    host = bytes(tag) + bytes(_dev.host_bytes_view(data.cpu().numpy() if isinstance(data, torch.Tensor) else data))
    return LatticeDigest(hash_blocks(CompressionAlg.BLAKE2B, [host]).entry(0))


def lt_hash_block(index: int, data) -> LatticeDigest:
    """BLAKE2b over LE64(index) || data (lattice.py:92-94)."""
    return _hash_one(struct.pack("<Q", index), data)


def lt_hash_tagged(tag: bytes, data) -> LatticeDigest:
    """BLAKE2b over an arbitrary tag followed by the block bytes (lattice.py:97-101)."""
    return _hash_one(bytes(tag), data)


def lt_reduce(digests: Iterable[LatticeDigest]) -> LatticeDigest:
    """Sum of a collection on the GPU; empty -> zero, one -> itself (lattice.py:104-119)."""
    items = list(digests)
    if not items:
        return lt_zero()
    if len(items) == 1:
        return items[0]
    dev = _dev.require_cuda()
    raw = torch.from_numpy(np.frombuffer(b"".join(d.data for d in items), dtype=np.uint8).copy()).to(dev)
    acc = _dev.LatticeAccumulator(1)
    acc.add_digests(raw, len(items))
    out, _, _ = acc.digests()
    return LatticeDigest(out)


def lt_reduce_pairwise(digests: Sequence[LatticeDigest]) -> LatticeDigest:
    """Binary-tree order of ``lt_add``; equal to ``lt_reduce`` by associativity (lattice.py:122-134)."""
    level = list(digests)
    if not level:
        return lt_zero()
    while len(level) > 1:
        nxt = [lt_add(level[i], level[i + 1]) for i in range(0, len(level) - 1, 2)]
        if len(level) & 1:
            nxt.append(level[-1])
        level = nxt
    return level[0]
