"""The kernels' per-thread code, compiled for the host, against hashlib and the block-table rule.

paper_2510_00554_b200/csrc/*.cuh is written __host__ __device__; tests/hostcheck
builds the same functions for the CPU so that padding, unaligned loads, the
tagged BLAKE2b message layout, the SHA-256 aligned fast path and the leaf locator
are verified before any GPU time is spent. (GPU parity proper: test_gpu_parity.py.)
"""

import ctypes
import hashlib
import random
import struct

import numpy as np
import pytest

import inputs

ALG = {"sha256": (0, hashlib.sha256, 32), "blake2b": (1, hashlib.blake2b, 64), "sha3-256": (2, hashlib.sha3_256, 32)}


@pytest.fixture(scope="module")
def hc():
    from paper_2510_00554_b200 import build

    return ctypes.CDLL(str(build.build_hostcheck()))


def _aligned(data: bytes, shift: int):
    buf = np.frombuffer(bytearray(len(data) + 64), dtype=np.uint8)
    start = (-buf.ctypes.data) % 16 + shift
    buf[start:start + len(data)] = np.frombuffer(data, dtype=np.uint8)
    return buf, buf.ctypes.data + start


def test_golden_kats(hc, golden):
    for rec in golden["kats"]:
        data = rec["msg"].encode() if "msg" in rec else inputs.seeded_bytes(rec["seed"], rec["len"])
        aid, _, dl = ALG[rec["alg"]]
        keep, p = _aligned(data, 0)
        out = (ctypes.c_uint8 * dl)()
        assert hc.hc_leaf(aid, ctypes.c_void_p(p), ctypes.c_uint64(len(data)), out) == 0
        assert bytes(out).hex() == rec["digest"], rec


def test_every_alignment_and_ragged_length(hc):
    rng = random.Random(1)
    for name, (aid, fn, dl) in ALG.items():
        for _ in range(250):
            n = rng.choice([0, 1, 55, 56, 63, 64, 65, 127, 128, 129, 135, 136, 137, rng.randint(0, 5000), 8192])
            shift = rng.randint(0, 15)
            data = rng.randbytes(n)
            keep, p = _aligned(data, shift)
            out = (ctypes.c_uint8 * dl)()
            hc.hc_leaf(aid, ctypes.c_void_p(p), ctypes.c_uint64(n), out)
            assert bytes(out) == fn(data).digest(), (name, n, shift)


def test_node_hash_and_zero_padding(hc):
    rng = random.Random(2)
    for name, (aid, fn, dl) in ALG.items():
        for small in (0, 1):                 # unrolled and rolled formulations of the node hash
            left, right = rng.randbytes(dl), rng.randbytes(dl)
            out = (ctypes.c_uint8 * dl)()
            hc.hc_pair(aid, left, right, out, small)
            assert bytes(out) == fn(left + right).digest()
            hc.hc_pair(aid, left, bytes(dl), out, small)
            assert bytes(out) == fn(left + bytes(dl)).digest()


def test_sha256_aligned_path_sliced_and_ragged(hc):
    """The aligned block loop resumed mid-leaf, the constant padding block, and the closing blocks of a ragged leaf."""
    rng = random.Random(3)
    for n in (64, 128, 1024, 8192, 65536, 1, 55, 56, 63, 65, 100, 119, 120, 127, 6400, 8191, 3072 + 57):
        data = rng.randbytes(n)
        keep, p = _aligned(data, 0)
        for split in (0, 1, 7, (n >> 6) // 2, n >> 6):
            out = (ctypes.c_uint8 * 32)()
            hc.hc_sha256_aligned(ctypes.c_void_p(p), ctypes.c_uint64(n), ctypes.c_uint32(split), out)
            assert bytes(out) == hashlib.sha256(data).digest(), (n, split)


def test_sliced_blake2b_and_sha3_carry_nothing_but_the_state(hc):
    """hash_blocks / absorb_blocks in slices (what a parked chain resumes from) == the one-shot digest."""
    rng = random.Random(8)
    lengths = [0, 1, 127, 128, 129, 135, 136, 137, 255, 256, 257, 271, 272, 273, 1000, 3072, 8191, 8192, 8193]
    for n in lengths + [rng.randint(0, 9000) for _ in range(40)]:
        for shift in (0, 8, rng.randint(1, 15)):
            data = rng.randbytes(n)
            keep, p = _aligned(data, shift)
            for slice_blocks in (1, 3, 16, 1000):
                out = (ctypes.c_uint8 * 32)()
                hc.hc_sha3_sliced(ctypes.c_void_p(p), ctypes.c_uint64(n), ctypes.c_uint32(slice_blocks), out)
                assert bytes(out) == hashlib.sha3_256(data).digest(), (n, shift, slice_blocks)
                for t in (0, 1, 2):
                    t0, t1 = rng.getrandbits(64), rng.getrandbits(64)
                    out = (ctypes.c_uint8 * 64)()
                    hc.hc_blake2b_sliced(t, ctypes.c_uint64(t0), ctypes.c_uint64(t1), ctypes.c_void_p(p),
                                         ctypes.c_uint64(n), ctypes.c_uint32(slice_blocks), out)
                    tag = [b"", struct.pack("<Q", t0), struct.pack("<QQ", t0, t1)][t]
                    assert bytes(out) == hashlib.blake2b(tag + data).digest(), (t, n, shift, slice_blocks)


def test_tagged_blake2b_layouts(hc, golden):
    rng = random.Random(4)
    for _ in range(400):
        t = rng.randint(0, 2)
        n = rng.choice([0, 1, 7, 8, 111, 112, 113, 119, 120, 121, 127, 128, 129, 247, 248, 249, 256, 3072,
                        rng.randint(0, 4000)])
        shift = rng.randint(0, 15)
        data = rng.randbytes(n)
        keep, p = _aligned(data, shift)
        t0, t1 = rng.getrandbits(64), rng.getrandbits(64)
        out = (ctypes.c_uint8 * 64)()
        hc.hc_blake2b_tagged(t, ctypes.c_uint64(t0), ctypes.c_uint64(t1), ctypes.c_void_p(p), ctypes.c_uint64(n), out)
        tag = [b"", struct.pack("<Q", t0), struct.pack("<QQ", t0, t1)][t]
        assert bytes(out) == hashlib.blake2b(tag + data).digest(), (t, n, shift)
    for rec in golden["lattice"]["hash_block"]:
        data = inputs.seeded_bytes(rec["seed"], rec["len"])
        keep, p = _aligned(data, 0)
        out = (ctypes.c_uint8 * 64)()
        hc.hc_blake2b_tagged(1, ctypes.c_uint64(rec["index"]), ctypes.c_uint64(0), ctypes.c_void_p(p),
                             ctypes.c_uint64(len(data)), out)
        assert bytes(out).hex() == rec["digest"]


def test_staged_blake2b_block_tail_and_carry_logic(hc):
    """blake2b_staged.cuh: chunk staging, sliding tag window, tails, every alignment (host stager)."""
    rng = random.Random(6)
    lengths = [0, 1, 7, 8, 9, 104, 111, 112, 113, 119, 120, 121, 127, 128, 129, 240, 247, 248, 249, 255, 256, 257,
               383, 384, 3072, 8192]
    for t in (0, 1, 2):
        for n in lengths + [rng.randint(0, 5000) for _ in range(60)]:
            for shift in (0, 8, rng.randint(1, 7), rng.randint(9, 15)):
                data = rng.randbytes(n)
                keep, p = _aligned(data, shift)
                t0, t1 = rng.getrandbits(64), rng.getrandbits(64)
                out = (ctypes.c_uint8 * 64)()
                assert hc.hc_blake2b_staged(t, ctypes.c_uint64(t0), ctypes.c_uint64(t1), ctypes.c_void_p(p),
                                            ctypes.c_uint64(n), out) == 0
                tag = [b"", struct.pack("<Q", t0), struct.pack("<QQ", t0, t1)][t]
                assert bytes(out) == hashlib.blake2b(tag + data).digest(), (t, n, shift)


def test_leaf_locator_equals_block_table(hc):
    """locate_leaf (per-tensor table + binary search) == the reference's per-block rows (model.py:137-146)."""
    from paper_2510_00554_b200.model import BlockTable, TensorMap

    rng = random.Random(5)
    for _ in range(30):
        sizes = [rng.choice([0, 0, 1, 63, 64, 65, 1000, 8192, 8193, rng.randint(0, 50000)]) for _ in range(rng.randint(1, 12))]
        if sum(sizes) == 0:
            sizes[0] = 5
        bs = rng.choice([64, 1024, 8192])
        table = BlockTable.build(TensorMap([(f"t{i}", bytes(s)) for i, s in enumerate(sizes)]), bs)
        arr = (ctypes.c_uint64 * len(sizes))(*sizes)
        for k, t, off, ln in table.rows:
            gt, goff, glen = ctypes.c_uint32(), ctypes.c_uint64(), ctypes.c_uint64()
            rc = hc.hc_locate(arr, len(sizes), bs, ctypes.c_uint64(k), ctypes.byref(gt), ctypes.byref(goff), ctypes.byref(glen))
            assert rc == 0 and (gt.value, goff.value, glen.value) == (t, off, ln), (sizes, bs, k)
        assert hc.hc_locate(arr, len(sizes), bs, ctypes.c_uint64(len(table.rows)), ctypes.byref(gt),
                            ctypes.byref(goff), ctypes.byref(glen)) == -1
