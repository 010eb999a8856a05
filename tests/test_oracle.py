"""Pin both CPU oracles (Python/hashlib and plain C) against the golden vectors.

The golden vectors come from the unmodified reference package
(tests/golden/make_golden.py) and include the reference suite's own known
answers and golden digest. An oracle that passes here is what the GPU parity
tests compare against.
"""

import hashlib
import struct

import numpy as np
import pytest

import inputs

ALGS = ["sha256", "blake2b", "sha3-256"]


def test_known_answers_both_oracles(golden, porc, corc):
    for rec in golden["kats"]:
        data = rec["msg"].encode() if "msg" in rec else inputs.seeded_bytes(rec["seed"], rec["len"])
        want = bytes.fromhex(rec["digest"])
        assert porc.h(rec["alg"], data) == want
        assert corc.hash_one(rec["alg"], data) == want


def test_c_oracle_matches_hashlib_on_unaligned_and_large(corc):
    big = inputs.seeded_bytes(99, 1 << 20)
    for alg, fn in (("sha256", hashlib.sha256), ("blake2b", hashlib.blake2b), ("sha3-256", hashlib.sha3_256)):
        for start in (0, 1, 3, 7):
            view = memoryview(big)[start:start + 700_001]
            assert corc.hash_one(alg, view) == fn(view).digest()


def test_merkle_roots(golden, porc, corc):
    for rec in golden["merkle"]:
        alg, n = rec["alg"], rec["n"]
        leaves = inputs.seeded_bytes(rec["seed"], n * porc.DIGEST_LEN[alg])
        want = bytes.fromhex(rec["root"])
        assert porc.merkle_root(alg, leaves, n) == want
        assert porc.merkle_root(alg, leaves, n, workers=3) == want
        assert corc.merkle_root(alg, leaves, n, threads=1) == want
        assert corc.merkle_root(alg, leaves, n, threads=4) == want


def test_hand_built_small_trees(porc):
    # the reference suite's hand-built cases (tests/test_merkle.py:51-67, :87-104)
    for alg in ALGS:
        dl = porc.DIGEST_LEN[alg]
        d = [porc.h(alg, bytes([i])) for i in range(4)]
        assert porc.merkle_root(alg, d[0], 1) == d[0]
        assert porc.merkle_root(alg, d[0] + d[1], 2) == porc.h(alg, d[0] + d[1])
        three = porc.h(alg, porc.h(alg, d[0] + d[1]) + porc.h(alg, d[2] + bytes(dl)))
        assert porc.merkle_root(alg, d[0] + d[1] + d[2], 3) == three
        four = porc.h(alg, porc.h(alg, d[0] + d[1]) + porc.h(alg, d[2] + d[3]))
        assert porc.merkle_root(alg, b"".join(d), 4) == four


def test_reference_suite_golden_inplace_digest(golden, porc, corc):
    rec = next(m for m in golden["models"] if m["kind"] == "reference-suite-golden")
    tensors = inputs.model_tensors(rec["rng_seed"], rec["sizes"])
    want = bytes.fromhex("5d70823521307e19d8a9451a8c264c8cd156ee99a9d7f46e9406867d712c9a7e")
    assert bytes.fromhex(rec["merkle_inplace"]) == want
    assert porc.inplace_merkle("sha256", tensors, 8192) == want
    tl = corc.TensorList(tensors)
    assert tl.leaf_count(8192) == rec["n_blocks"] == 6
    assert corc.inplace_merkle("sha256", tl, 8192, threads=3) == want


def test_seeded_models(golden, porc, corc):
    for rec in golden["models"]:
        if rec["kind"] != "seeded":
            continue
        tensors = inputs.model_tensors(rec["seed"], rec["sizes"])
        bs = rec["block_size"]
        tl = corc.TensorList(tensors)
        assert tl.leaf_count(bs) == rec["n_blocks"]
        for alg in ALGS:
            want = bytes.fromhex(rec[f"merkle_inplace_{alg}"])
            leaves, n = porc.inplace_leaves(alg, tensors, bs, workers=2)
            assert n == rec["n_blocks"]
            assert hashlib.sha256(bytes(leaves)).hexdigest() == rec[f"leaves_sha256_{alg}"]
            assert porc.merkle_root(alg, leaves, n) == want
            c_leaves = corc.inplace_leaves(alg, tl, bs, threads=3)
            assert c_leaves == bytes(leaves)
            assert corc.inplace_merkle(alg, tl, bs, threads=2) == want
            assert porc.coalesced_merkle(alg, tensors, bs).hex() == rec[f"merkle_coalesced_{alg}"]
            root, layers = porc.per_layer_merkle(alg, tensors, bs)
            assert root.hex() == rec[f"merkle_per_layer_{alg}"]
            assert hashlib.sha256(b"".join(layers)).hexdigest() == rec[f"merkle_layers_sha256_{alg}"]
        root, layers = porc.per_layer_lattice(tensors, bs)
        assert root.hex() == rec["lattice_per_layer"]
        assert hashlib.sha256(b"".join(layers)).hexdigest() == rec["lattice_layers_sha256"]
        assert porc.inplace_lattice(tensors, bs, workers=3).hex() == rec["lattice_inplace"]
        assert corc.inplace_lattice(tl, bs, threads=3).hex() == rec["lattice_inplace"]
        assert porc.coalesced_lattice(tensors, bs).hex() == rec["lattice_coalesced"]


def test_lattice_vectors(golden, porc, corc):
    lat = golden["lattice"]
    for rec in lat["hash_block"]:
        data = inputs.seeded_bytes(rec["seed"], rec["len"])
        tag = struct.pack("<Q", rec["index"])
        assert porc.lt_hash_tagged(tag, data).hex() == rec["digest"]
        assert corc.lt_hash_tagged(tag, data).hex() == rec["digest"]
    for rec in lat["tagged"]:
        tag = inputs.seeded_bytes(rec["tag_seed"], rec["tag_len"])
        data = inputs.seeded_bytes(rec["seed"], rec["len"])
        assert porc.lt_hash_tagged(tag, data).hex() == rec["digest"]
        assert corc.lt_hash_tagged(tag, data).hex() == rec["digest"]
    for rec in lat["add"]:
        assert porc.lt_add(bytes.fromhex(rec["a"]), bytes.fromhex(rec["b"])).hex() == rec["sum"]
    for rec in lat["reduce"]:
        ds = [inputs.seeded_bytes(rec["seed_base"] + i, 64) for i in range(rec["n"])]
        assert porc.lt_sum(ds).hex() == rec["sum"]


def test_dataset_digests(golden, porc, corc):
    for rec in golden["datasets"]:
        spec = inputs.DATASET_CASES[rec["case"]]
        samples = inputs.dataset_samples(**spec)
        got = porc.dataset_digests(samples, declared=spec["declared"], cover_labels=rec["cover_labels"])
        want = {int(k): (bytes.fromhex(v[0]), v[1]) for k, v in rec["digests"].items()}
        assert got == want
        # batch size does not matter
        assert porc.dataset_digests(samples, declared=spec["declared"], cover_labels=rec["cover_labels"],
                                    batch_size=7) == want
        if not rec["cover_labels"]:
            shard, off, ln, ids, src = inputs.pack_samples(samples)
            sources = sorted(spec["declared"])
            slots = np.array([sources.index(int(s)) for s in src], dtype=np.uint32)
            sums, counts = corc.lthash_samples(shard, off, ln, ids, slots, len(sources), threads=3)
            for i, sid in enumerate(sources):
                assert (sums[64 * i:64 * i + 64], counts[i]) == want[sid]


def test_shard_rule_equals_plain_root(porc):
    # reduce each 2^k-leaf shard exactly k levels, then the shard roots
    for alg in ALGS:
        dl = porc.DIGEST_LEN[alg]
        for n in (1, 2, 3, 5, 8, 9, 31, 32, 33, 100, 257):
            leaves = inputs.seeded_bytes(7000 + n, n * dl)
            want = porc.merkle_root(alg, leaves, n)
            for k in range(0, 7):
                if k > (0 if n <= 1 else (n - 1).bit_length()):
                    continue        # more forced levels than the tree has: not a valid shard size
                assert porc.subtree_sharded_root(alg, leaves, n, k) == want, (alg, n, k)
