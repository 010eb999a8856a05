"""Generate tests/golden/golden.json by running the UNMODIFIED reference package.

Run in the build container only (the reference does not travel to the GPU box):

    python tests/golden/make_golden.py

It imports ``sentinel`` from /root/reference/pkg/src, feeds it seeded inputs and
records the outputs. Inputs are never stored: every test regenerates them from the
recorded seeds with ``random.Random(seed).randbytes`` (helpers in tests/inputs.py).
The known-answer vectors and the golden in-place digest are the ones the
reference's own suite pins (tests/test_compression.py:11-26, tests/test_model.py:269-277);
they are recomputed here through the reference and asserted to match.
"""

from __future__ import annotations

import base64
import hashlib
import json
import random
import struct
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))            # tests/inputs.py
sys.path.insert(0, "/root/reference/pkg/src")

import sentinel  # noqa: E402  (the reference)
from sentinel import attestation as ratt  # noqa: E402
from sentinel.compression import CompressionAlg, compress_block  # noqa: E402
from sentinel.dataset import Batch, SampleRecord, SourceAccumulator, finalize, process_batch  # noqa: E402
from sentinel.lattice import LatticeDigest, lt_add, lt_hash_block, lt_hash_tagged, lt_reduce, lt_sub  # noqa: E402
from sentinel.merkle import DigestBuffer, hash_blocks, merkle_root  # noqa: E402
from sentinel.model import Construction, HashConfig, Strategy, TensorMap, hash_model  # noqa: E402

import inputs  # noqa: E402

ALGS = {"sha256": CompressionAlg.SHA256, "blake2b": CompressionAlg.BLAKE2B, "sha3-256": CompressionAlg.SHA3_256}


def kats():
    published = {
        ("sha256", ""): "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855",
        ("sha256", "abc"): "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad",
        ("sha3-256", ""): "a7ffc6f8bf1ed76651c14756a061d662f580ff4de43b49fa82d80a4b80f8434a",
        ("sha3-256", "abc"): "3a985da74fe225b2045c172d6bd390bd855f086e3e9d525b46bfe24511431532",
        ("blake2b", ""): "786a02f742015903c6c6fd852552d272912f4740e15847618a86e217f71f5419"
                         "d25e1031afee585313896444934eb04b903a685b1448b755d56f701afe9be2ce",
        ("blake2b", "abc"): "ba80a53f981c4d0d6a2797b69f12f6e94c212f14685ac4b74b12bb6fdbffa2d1"
                            "7d87c5392aab792dc252d5de4533cc9518d38aa8dbf1925ab92386edd4009923",
    }
    out = []
    for (alg, msg), want in published.items():
        got = compress_block(ALGS[alg], msg.encode()).hex()
        assert got == want, (alg, msg)
        out.append({"alg": alg, "msg": msg, "digest": got})
    # message lengths around every padding boundary of the three algorithms
    for alg in ALGS:
        for n in inputs.BOUNDARY_LENGTHS:
            data = inputs.seeded_bytes(1000 + n, n)
            out.append({"alg": alg, "seed": 1000 + n, "len": n, "digest": compress_block(ALGS[alg], data).hex()})
    return out


def merkle_cases():
    out = []
    for alg in ALGS:
        dlen = ALGS[alg].digest_len
        for n in (1, 2, 3, 4, 5, 7, 16, 31, 33, 100, 1023, 1025, 2500):
            leaves = inputs.seeded_bytes(2000 + n, n * dlen)
            buf = DigestBuffer(ALGS[alg], bytearray(leaves), n)
            out.append({"alg": alg, "n": n, "seed": 2000 + n, "root": merkle_root(ALGS[alg], buf).hex()})
    return out


def model_cases():
    out = []
    golden_sizes = [100, 8192, 5000, 0, 20000]
    rng = random.Random(2024)
    model = TensorMap([(f"t{i}", rng.randbytes(s)) for i, s in enumerate(golden_sizes)])
    res = hash_model(HashConfig(Construction.MERKLE, Strategy.IN_PLACE), model)
    assert res.digest_hex() == "5d70823521307e19d8a9451a8c264c8cd156ee99a9d7f46e9406867d712c9a7e"
    out.append({"kind": "reference-suite-golden", "rng_seed": 2024, "sizes": golden_sizes, "block_size": 8192,
                "alg": "sha256", "merkle_inplace": res.digest_hex(), "n_blocks": res.block_count})
    for case_id, (seed, sizes) in enumerate(inputs.MODEL_CASES):
        tensors = inputs.model_tensors(seed, sizes)
        tm = TensorMap([(f"t{i}", t) for i, t in enumerate(tensors)])
        for bs in inputs.MODEL_BLOCK_SIZES:
            rec = {"kind": "seeded", "case": case_id, "seed": seed, "sizes": sizes, "block_size": bs}
            for alg in ALGS:
                cfg = HashConfig(Construction.MERKLE, Strategy.IN_PLACE, ALGS[alg], bs)
                r = hash_model(cfg, tm)
                blocks = []
                for t in tensors:
                    blocks += [t[o:o + bs] for o in range(0, len(t), bs)]
                leaves = hash_blocks(ALGS[alg], blocks)
                rec[f"merkle_inplace_{alg}"] = r.digest_hex()
                rec[f"leaves_sha256_{alg}"] = hashlib.sha256(bytes(leaves.data)).hexdigest()
                rec["n_blocks"] = r.block_count
                rec[f"merkle_coalesced_{alg}"] = hash_model(
                    HashConfig(Construction.MERKLE, Strategy.COALESCED, ALGS[alg], bs), tm).digest_hex()
                pl = hash_model(HashConfig(Construction.MERKLE, Strategy.PER_LAYER, ALGS[alg], bs), tm)
                rec[f"merkle_per_layer_{alg}"] = pl.digest_hex()
                rec[f"merkle_layers_sha256_{alg}"] = hashlib.sha256(
                    b"".join(d.data for d in pl.layer_digests.values())).hexdigest()
                rec["per_layer_block_count"] = pl.block_count
            pl = hash_model(HashConfig(Construction.LATTICE, Strategy.PER_LAYER, CompressionAlg.BLAKE2B, bs), tm)
            rec["lattice_per_layer"] = pl.digest_hex()
            rec["lattice_layers_sha256"] = hashlib.sha256(b"".join(d.data for d in pl.layer_digests.values())).hexdigest()
            po = hash_model(HashConfig(Construction.LATTICE, Strategy.PER_LAYER, CompressionAlg.BLAKE2B, bs,
                                       ordered_per_layer=True), tm)
            assert po.digest_hex() == pl.digest_hex()
            rec["lattice_inplace"] = hash_model(
                HashConfig(Construction.LATTICE, Strategy.IN_PLACE, CompressionAlg.BLAKE2B, bs), tm).digest_hex()
            rec["lattice_coalesced"] = hash_model(
                HashConfig(Construction.LATTICE, Strategy.COALESCED, CompressionAlg.BLAKE2B, bs), tm).digest_hex()
            out.append(rec)
    return out


def lattice_cases():
    out = {"hash_block": [], "add": [], "reduce": []}
    for idx, n in [(0, 0), (1, 1), (7, 119), (8, 120), (9, 121), (2**40 + 5, 128), (12345, 3072), (2**64 - 1, 1000)]:
        data = inputs.seeded_bytes(3000 + n, n)
        out["hash_block"].append({"index": idx, "seed": 3000 + n, "len": n, "digest": lt_hash_block(idx, data).hex()})
    assert lt_hash_block(0, b"").data == hashlib.blake2b(bytes(8)).digest()      # tests/test_lattice.py:92-94
    out["tagged"] = []
    for tag_len, n in [(16, 500), (11, 64), (8, 0), (20, 3000)]:
        tag = inputs.seeded_bytes(3500 + tag_len, tag_len)
        data = inputs.seeded_bytes(3600 + n, n)
        out["tagged"].append({"tag_seed": 3500 + tag_len, "tag_len": tag_len, "seed": 3600 + n, "len": n,
                              "digest": lt_hash_tagged(tag, data).hex()})
    a = LatticeDigest(struct.pack("<32H", *([0xFFFF, 0x8000, 1, 0] * 8)))
    b = LatticeDigest(struct.pack("<32H", *([1, 0x8000, 0xFFFF, 0] * 8)))
    out["add"].append({"a": a.hex(), "b": b.hex(), "sum": lt_add(a, b).hex(), "diff": lt_sub(a, b).hex()})
    for n in (2, 97, 1000):
        ds = [LatticeDigest(inputs.seeded_bytes(4000 + 131 * n + i, 64)) for i in range(n)]
        out["reduce"].append({"n": n, "seed_base": 4000 + 131 * n, "sum": lt_reduce(ds).hex()})
    return out


def dataset_cases():
    out = []
    for case_id, spec in enumerate(inputs.DATASET_CASES):
        samples = inputs.dataset_samples(**spec)
        for cover in (False, True):
            acc = SourceAccumulator(cover_labels=cover)
            acc.declare(spec["declared"])
            recs = [SampleRecord(sid, src, label, data) for sid, src, label, data in samples]
            for start in range(0, len(recs), 128):
                process_batch(Batch(recs[start:start + 128]), acc)
            fin = finalize(acc)
            out.append({"case": case_id, "cover_labels": cover,
                        "digests": {str(sid): [d.hex(), c] for sid, (d, c) in fin.items()}})
    return out


def attestation_cases():
    pem = inputs.TEST_KEY_PEM.encode()
    from cryptography.hazmat.primitives import serialization
    key = ratt.KeyPair(serialization.load_pem_private_key(pem, password=None))
    stmt = ratt.Statement([ratt.Subject("model-x", {"sha256": "ab" * 32}),
                           ratt.Subject("data:source:3", {"lthash": "cd" * 64})],
                          ratt.MODEL_PREDICATE_TYPE,
                          {"construction": "merkle", "compression": "sha256", "strategy": "in-place",
                           "block_size": 8192, "ordered_per_layer": False, "index_encoding": "le64-prefix-v1",
                           "note": "héllo"})
    bundle = ratt.sign_bundle(stmt, key)
    return {
        "canonical_b64": base64.b64encode(ratt.canonicalize(stmt)).decode(),
        "pae_b64": base64.b64encode(ratt.pae(ratt.PAYLOAD_TYPE, ratt.canonicalize(stmt))).decode(),
        "pae_small": ratt.pae("t", b"body").decode(),
        "key_id": key.key_id,
        "public_point_hex": key.public_point_hex,
        "bundle": bundle.to_dict(),
    }


def bench_cases():
    """Digest column of the reference's strategy-comparison table (bench.py:81-133) on small synthetic
    models, plus a fingerprint of the synthetic bytes themselves (bench.py:32-45)."""
    from sentinel import bench as rbench

    out = {"models": [], "cells": []}
    for shape, scale, seed in (("vgg19", 0.0005, 0), ("resnet152", 0.002, 0), ("gpt2", 0.0003, 5)):
        m = rbench.synthetic_model(shape, scale, seed)
        out["models"].append({"shape": shape, "scale": scale, "seed": seed, "layers": len(m.entries),
                              "total_bytes": m.total_bytes,
                              "sha256_of_bytes": hashlib.sha256(b"".join(b for _, b in m.entries)).hexdigest()})
    for c in rbench.run_bench(shapes=("vgg19", "resnet152"), scale=0.002, worker_counts=(1,), repeats=1,
                              compressions=("sha256", "blake2b", "sha3-256")):
        out["cells"].append({"shape": c.shape, "construction": c.construction, "compression": c.compression,
                             "strategy": c.strategy, "digest": c.digest})
    return out


def main():
    (HERE / "golden_bench.json").write_text(json.dumps(bench_cases(), indent=1, sort_keys=True))
    print("wrote", HERE / "golden_bench.json")
    doc = {
        "generator": "tests/golden/make_golden.py",
        "reference": f"sentinel {sentinel.__version__} imported from /root/reference/pkg/src",
        "kats": kats(),
        "merkle": merkle_cases(),
        "models": model_cases(),
        "lattice": lattice_cases(),
        "datasets": dataset_cases(),
        "attestation": attestation_cases(),
    }
    (HERE / "golden.json").write_text(json.dumps(doc, indent=1, sort_keys=True))
    print("wrote", HERE / "golden.json")


if __name__ == "__main__":
    main()
