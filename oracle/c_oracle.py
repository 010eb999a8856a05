"""ctypes wrapper around oracle/_build/liboracle.so (TEST INFRASTRUCTURE; see oracle.c)."""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"
ALG = {"sha256": 0, "blake2b": 1, "sha3-256": 2}
DLEN = {"sha256": 32, "blake2b": 64, "sha3-256": 32}

_lib = None


def build() -> Path:
    src = HERE / "oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        LIB.parent.mkdir(exist_ok=True)
        subprocess.run(["gcc", "-O3", "-std=c11", "-fPIC", "-shared", "-pthread", str(src), "-o", str(LIB)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(str(LIB))
        _lib.orc_leaf_count.restype = ctypes.c_uint64
    return _lib


def threads_default() -> int:
    return os.cpu_count() or 1


def _u8(buf) -> np.ndarray:
    if isinstance(buf, np.ndarray):
        return np.ascontiguousarray(buf).reshape(-1).view(np.uint8)
    return np.frombuffer(buf, dtype=np.uint8)


def hash_one(alg: str, data) -> bytes:
    arr = _u8(data)
    out = (ctypes.c_uint8 * 64)()
    lib().orc_hash(ALG[alg], ctypes.c_void_p(arr.ctypes.data), ctypes.c_uint64(arr.size), out)
    return bytes(out)[:DLEN[alg]]


def lt_hash_tagged(tag: bytes, data) -> bytes:
    arr = _u8(data)
    out = (ctypes.c_uint8 * 64)()
    lib().orc_lt_hash_tagged(tag, ctypes.c_uint64(len(tag)), ctypes.c_void_p(arr.ctypes.data),
                             ctypes.c_uint64(arr.size), out)
    return bytes(out)


def merkle_root(alg: str, leaves: bytes, count: int, threads: int = 1) -> bytes:
    out = (ctypes.c_uint8 * 64)()
    arr = _u8(leaves)
    rc = lib().orc_merkle_root(ALG[alg], ctypes.c_void_p(arr.ctypes.data), ctypes.c_uint64(count), out, threads)
    assert rc == 0
    return bytes(out)[:DLEN[alg]]


class TensorList:
    """Host tensors as the (pointer, length) arrays the C oracle takes; keeps them alive."""

    def __init__(self, tensors: Sequence):
        self.arrays = [_u8(t) for t in tensors]
        n = len(self.arrays)
        self.ptrs = (ctypes.c_void_p * max(1, n))(*[a.ctypes.data if a.size else None for a in self.arrays])
        self.sizes = (ctypes.c_uint64 * max(1, n))(*[a.size for a in self.arrays])
        self.n = n

    def leaf_count(self, block_size: int) -> int:
        return int(lib().orc_leaf_count(self.sizes, self.n, block_size))


def inplace_leaves(alg: str, tensors: TensorList, block_size: int, threads: int = 1) -> bytes:
    n = tensors.leaf_count(block_size)
    out = np.empty(n * DLEN[alg], dtype=np.uint8)
    rc = lib().orc_inplace_leaves(ALG[alg], tensors.ptrs, tensors.sizes, tensors.n, block_size,
                                  ctypes.c_void_p(out.ctypes.data), threads)
    assert rc == 0
    return out.tobytes()


def inplace_merkle(alg: str, tensors: TensorList, block_size: int, threads: int = 1) -> bytes:
    out = (ctypes.c_uint8 * 64)()
    rc = lib().orc_inplace_merkle(ALG[alg], tensors.ptrs, tensors.sizes, tensors.n, block_size, out, threads)
    assert rc == 0
    return bytes(out)[:DLEN[alg]]


def inplace_lattice(tensors: TensorList, block_size: int, threads: int = 1) -> bytes:
    out = (ctypes.c_uint8 * 64)()
    rc = lib().orc_inplace_lattice(tensors.ptrs, tensors.sizes, tensors.n, block_size, out, threads)
    assert rc == 0
    return bytes(out)


def lthash_samples(shard, offsets, lengths, ids, slots, n_sources: int, threads: int = 1,
                   want_digests: bool = False):
    """Returns (n_sources x 64 digest bytes, counts list[, n x 64 sample digests])."""
    sh = _u8(shard)
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    ln = np.ascontiguousarray(lengths, dtype=np.uint64)
    idv = np.ascontiguousarray(ids, dtype=np.uint64)
    sl = np.ascontiguousarray(slots, dtype=np.uint32)
    n = off.size
    sums = np.zeros(n_sources * 32, dtype="<u2")
    counts = np.zeros(n_sources, dtype=np.uint64)
    dig = np.empty(n * 64, dtype=np.uint8) if want_digests else None
    rc = lib().orc_lthash_samples(ctypes.c_void_p(sh.ctypes.data), ctypes.c_void_p(off.ctypes.data),
                                  ctypes.c_void_p(ln.ctypes.data), ctypes.c_void_p(idv.ctypes.data),
                                  ctypes.c_void_p(sl.ctypes.data), ctypes.c_uint64(n), n_sources,
                                  ctypes.c_void_p(sums.ctypes.data), ctypes.c_void_p(counts.ctypes.data),
                                  ctypes.c_void_p(dig.ctypes.data if dig is not None else 0), threads)
    assert rc == 0, rc
    res = (sums.tobytes(), [int(c) for c in counts])
    return res + (dig.tobytes(),) if want_digests else res
