"""The CPython packing helper (csrc/hostpack.c): layout and checks, no GPU needed.

It only moves bytes: sequences of host blocks (hash_blocks, merkle.py:93-114) and batches of sample
records (process_batch, dataset.py:74-86) into one block. The layout it writes must be the one
``_BatchEngine.add`` writes in Python, byte for byte.
"""

import random

import numpy as np
import pytest

from paper_2510_00554_b200 import _hostpack
from paper_2510_00554_b200.dataset import SampleRecord


def _python_layout(samples, cover_labels, slot_of):
    n = len(samples)
    payloads = [s.label + bytes(s.data) for s in samples] if cover_labels else [bytes(s.data) for s in samples]
    lengths = np.array([len(p) for p in payloads], dtype=np.uint64)
    header = -(-28 * n // 16) * 16
    total = int(lengths.sum())
    out = np.zeros(header + max(total, 16), dtype=np.uint8)
    offs = out[0:8 * n].view(np.uint64)
    offs[0] = 0
    np.cumsum(lengths[:-1], out=offs[1:])
    out[8 * n:16 * n].view(np.uint64)[:] = lengths
    out[16 * n:24 * n].view(np.uint64)[:] = np.array([s.sample_id for s in samples], dtype=np.uint64)
    out[24 * n:28 * n].view(np.int32)[:] = [slot_of[s.source_id] for s in samples]
    out[header:header + total] = np.frombuffer(b"".join(payloads), dtype=np.uint8)
    return out, header, total


def test_gather_lengths_and_bytes():
    rng = random.Random(1)
    blocks = [rng.randbytes(rng.choice([0, 1, 63, 64, 4097])) for _ in range(300)]
    blocks[7] = bytearray(blocks[7])
    blocks[9] = memoryview(blocks[9])[: len(blocks[9]) // 2]
    blocks[11] = np.frombuffer(blocks[11], dtype=np.uint8)
    lens = np.zeros(len(blocks), dtype=np.uint64)
    total = _hostpack.gather(blocks, 0, 0, lens.ctypes.data)            # measure only
    assert total == sum(len(bytes(b)) for b in blocks)
    assert lens.tolist() == [len(bytes(b)) for b in blocks]
    dst = np.full(total + 8, 0xEE, dtype=np.uint8)
    assert _hostpack.gather(blocks, dst.ctypes.data, total, 0) == total
    assert dst[:total].tobytes() == b"".join(bytes(b) for b in blocks)
    assert (dst[total:] == 0xEE).all()                                  # nothing past the end


def test_gather_large_pack_uses_threads_and_matches():
    rng = np.random.default_rng(2)
    big = rng.integers(0, 256, size=48 << 20, dtype=np.uint8)
    view = memoryview(big)
    blocks = [view[i:i + 8192] for i in range(0, big.size, 8192)]
    dst = np.empty(big.size, dtype=np.uint8)
    assert _hostpack.gather(blocks, dst.ctypes.data, dst.size, 0, 8) == big.size
    assert np.array_equal(dst, big)


def test_gather_too_small_copies_nothing_and_bad_items_raise():
    dst = np.zeros(4, dtype=np.uint8)
    assert _hostpack.gather([b"abcdef"], dst.ctypes.data, 4, 0) == 6
    assert not dst.any()
    with pytest.raises(TypeError):
        _hostpack.gather(["text"], 0, 0, 0)
    with pytest.raises((BufferError, ValueError)):
        _hostpack.gather([np.arange(10, dtype=np.uint8)[::2]], 0, 0, 0)  # not contiguous


@pytest.mark.parametrize("cover_labels", [False, True])
def test_pack_records_matches_python_layout(cover_labels):
    rng = random.Random(3)
    slot_of = {5: 0, 2: 1, 9: 2}
    samples = [SampleRecord(rng.randrange(1 << 64), rng.choice([5, 2, 9]), rng.randbytes(rng.randrange(4)),
                            rng.randbytes(rng.choice([0, 1, 100, 3072]))) for _ in range(129)]
    samples[3] = SampleRecord((1 << 64) - 1, 2, b"x", bytearray(b"mutable payload"))
    want, header, total = _python_layout(samples, cover_labels, slot_of)
    dst = np.zeros(want.size + 64, dtype=np.uint8)
    code, a, b = _hostpack.pack_records(samples, cover_labels, slot_of, None, dst.ctypes.data, dst.size)
    assert (code, a, b) == (0, total, header)
    assert np.array_equal(dst[:want.size], want)


def test_pack_records_status_codes():
    slot_of = {1: 0}
    ok = SampleRecord(1, 1, b"", b"abc")
    dst = np.zeros(256, dtype=np.uint8)
    args = (dst.ctypes.data, dst.size)
    assert _hostpack.pack_records([ok, SampleRecord(2, 7, b"", b"z")], False, slot_of, frozenset({1}), *args)[:2] == (2, 1)
    assert _hostpack.pack_records([ok, SampleRecord(-1, 1, b"", b"z")], False, slot_of, None, *args)[:2] == (3, 1)
    assert _hostpack.pack_records([ok, SampleRecord(1 << 64, 1, b"", b"z")], False, slot_of, None, *args)[:2] == (3, 1)
    assert _hostpack.pack_records([ok, SampleRecord(2, 7, b"", b"z")], False, slot_of, None, *args)[:2] == (4, 1)
    # undeclared source is reported before a bad id, a bad id before a missing slot (the order process_batch checks in)
    assert _hostpack.pack_records([SampleRecord(-1, 1, b"", b""), SampleRecord(2, 7, b"", b"")], False, slot_of,
                                  frozenset({1}), *args)[:2] == (2, 1)
    code, needed, _ = _hostpack.pack_records([ok], False, slot_of, None, dst.ctypes.data, 8)
    assert (code, needed) == (1, 32 + 16)
    assert not dst.any()
    assert _hostpack.pack_records([], False, slot_of, None, *args) == (0, 0, 0)


def test_manifest_columns():
    rows = [(5, 1, b"a", 0, 10), ((1 << 64) - 1, -3, b"", 7, 0), (0, 2, b"zz", 1 << 40, 3)]
    ids = np.zeros(3, dtype=np.uint64)
    src, off, ln = (np.zeros(3, dtype=np.int64) for _ in range(3))
    ptrs = (ids.ctypes.data, src.ctypes.data, off.ctypes.data, ln.ctypes.data)
    assert _hostpack.manifest_columns(rows, *ptrs) == (0, 3)
    assert ids.tolist() == [5, (1 << 64) - 1, 0] and src.tolist() == [1, -3, 2]
    assert off.tolist() == [0, 7, 1 << 40] and ln.tolist() == [10, 0, 3]
    assert _hostpack.manifest_columns([(1, 1, b"", 0, 1), (-1, 1, b"", 0, 1)], *ptrs) == (3, 1)
    assert _hostpack.manifest_columns([(1 << 64, 1, b"", 0, 1)], *ptrs) == (3, 0)
    assert _hostpack.manifest_columns([(1, 1, b"", 1 << 70, 1)], *ptrs) == (5, 0)      # caller's Python path decides
    assert _hostpack.manifest_columns([[1, 1, b"", 0, 1]], *ptrs) == (5, 0)            # not a tuple
    assert _hostpack.manifest_columns([], *ptrs) == (0, 0)


def test_copy_many_memory_and_file(tmp_path):
    rng = np.random.default_rng(4)
    src = rng.integers(0, 256, size=(9 << 20) + 123, dtype=np.uint8)
    dst = np.zeros(src.size + 64, dtype=np.uint8)
    pieces = []
    for o in range(0, src.size, (2 << 20) + 77):                      # pieces at odd offsets, cut into 1 MB jobs inside
        ln = min((2 << 20) + 77, src.size - o)
        pieces += [dst.ctypes.data + 32 + o, src.ctypes.data + o, ln]
    for threads in (1, 3, 12):
        dst[:] = 0
        assert _hostpack.copy_many(pieces, -1, threads) == src.size
        assert np.array_equal(dst[32:32 + src.size], src) and not dst[:32].any() and not dst[32 + src.size:].any()
    path = tmp_path / "shard.bin"
    path.write_bytes(src.tobytes())
    import os

    fd = os.open(path, os.O_RDONLY)
    try:
        dst[:] = 0
        assert _hostpack.copy_many([dst.ctypes.data, 7, src.size - 7], fd, 4) == src.size - 7
        assert np.array_equal(dst[:src.size - 7], src[7:])
        with pytest.raises(OSError):
            _hostpack.copy_many([dst.ctypes.data, src.size - 10, 100], fd, 2)     # runs past the end of the file
    finally:
        os.close(fd)
    assert _hostpack.copy_many([]) == 0
    with pytest.raises(ValueError):
        _hostpack.copy_many([1, 2])
