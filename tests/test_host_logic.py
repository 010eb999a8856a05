"""Host-side logic that needs no GPU: configuration, block table, manifests, layouts,
shard planning, lattice value algebra, attestation formats, and the no-fallback rule."""

import base64
import json
import random
import struct

import pytest

import inputs
import paper_2510_00554_b200 as pkg
from paper_2510_00554_b200 import distributed as dd
from paper_2510_00554_b200 import shapes, workers
from paper_2510_00554_b200.errors import ConfigError, FormatError, InvalidInput, KeyMaterialError, ResourceError


# ---- public surface --------------------------------------------------------------

def test_public_names_match_the_reference_package():
    # /root/reference/pkg/src/sentinel/__init__.py:3-43
    names = """CompressionAlg Digest compress_block sequential_hash LatticeDigest lt_add lt_hash_block lt_reduce
    lt_sub lt_zero DigestBuffer ReductionState hash_blocks merkle_root reduce_level BlockTable Construction
    HashConfig ModelDigestResult Strategy TensorMap coalesce_hash hash_model inplace_hash load_model
    ordered_lattice_per_layer per_layer_hash save_model Batch DatasetManifest SampleRecord SourceAccumulator
    digest_dataset finalize hash_sample iterate_batches process_batch Bundle Envelope KeyPair Statement Subject
    Verdict canonicalize keygen sign_bundle verify_bundle""".split()
    for n in names:
        assert hasattr(pkg, n), n
    assert pkg.__version__ == "0.1.0"


def test_no_cpu_fallback_without_a_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE)
    with pytest.raises(ResourceError):
        pkg.hash_model(cfg, pkg.TensorMap([("a", b"abc")]))
    with pytest.raises(ResourceError):
        pkg.hash_blocks(pkg.CompressionAlg.SHA256, [b"abc"])
    with pytest.raises(ResourceError):
        pkg.lt_hash_block(1, b"abc")
    with pytest.raises(ResourceError):
        pkg.lt_reduce([pkg.lt_zero(), pkg.lt_zero()])


# ---- configuration (model.py:85-128) ----------------------------------------------------

def test_config_validation_rules():
    C, S, A = pkg.Construction, pkg.Strategy, pkg.CompressionAlg
    for bad in (0, 63, 100, 8191):
        with pytest.raises(ConfigError):
            pkg.HashConfig(C.MERKLE, S.IN_PLACE, A.SHA256, block_size=bad).validate()
    with pytest.raises(ConfigError):
        pkg.HashConfig(C.LATTICE, S.IN_PLACE, A.SHA256).validate()
    with pytest.raises(ConfigError):
        pkg.HashConfig(C.MERKLE, S.PER_LAYER, A.SHA256, ordered_per_layer=True).validate()
    pkg.HashConfig(C.LATTICE, S.PER_LAYER, A.BLAKE2B, ordered_per_layer=True).validate()
    pkg.HashConfig(C.MERKLE, S.IN_PLACE, A.SHA3_256, block_size=64).validate()


def test_predicate_round_trip_and_bad_predicates():
    cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.SHA3_256, 4096)
    pred = cfg.predicate()
    assert pred == {"construction": "merkle", "compression": "sha3-256", "strategy": "in-place",
                    "block_size": 4096, "ordered_per_layer": False, "index_encoding": "le64-prefix-v1"}
    assert pkg.HashConfig.from_predicate(pred) == cfg
    with pytest.raises(FormatError):
        pkg.HashConfig.from_predicate({"construction": "merkle"})
    with pytest.raises(FormatError):
        pkg.HashConfig.from_predicate(dict(pred, compression="md5"))
    with pytest.raises(ConfigError):
        pkg.HashConfig.from_predicate(dict(pred, block_size=100))


def test_algorithm_enum():
    A = pkg.CompressionAlg
    assert [a.value for a in A] == ["sha256", "blake2b", "sha3-256"]
    assert [a.digest_len for a in A] == [32, 64, 32]
    assert A.from_name("sha3-256") is A.SHA3_256
    with pytest.raises(ValueError):
        A.from_name("md5")
    with pytest.raises(ValueError):
        pkg.Digest(A.SHA256, b"short")
    assert pkg.sequential_hash(A.SHA256, [b"ab", b"c"]).hex() == \
        "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"


# ---- tensor map / block table / manifests ----------------------------------------------

def test_tensor_map_rules():
    with pytest.raises(InvalidInput):
        pkg.TensorMap([("a", b"x"), ("a", b"y")])
    tm = pkg.TensorMap([("a", b"xyz"), ("b", bytearray(5)), ("c", memoryview(b"12"))])
    assert len(tm) == 3 and tm.total_bytes == 10 and tm.names() == ["a", "b", "c"]


def test_block_table_matches_reference_rule():
    rng = random.Random(41)
    for _ in range(20):
        sizes = [rng.choice([0, 1, 1023, 1024, 1025, rng.randint(0, 9000)]) for _ in range(rng.randint(1, 7))]
        tm = pkg.TensorMap([(f"t{i}", bytes(s)) for i, s in enumerate(sizes)])
        rows = pkg.BlockTable.build(tm, 1024).rows
        want, k = [], 0
        for t, s in enumerate(sizes):                       # model.py:137-146, restated
            for off in range(0, s, 1024):
                want.append((k, t, off, min(1024, s - off)))
                k += 1
        assert rows == want
        assert sum(r[3] for r in rows) == tm.total_bytes


def test_model_manifest_round_trip(tmp_path):
    rng = random.Random(43)
    tm = pkg.TensorMap([(f"l{i}", rng.randbytes(rng.randint(0, 3000))) for i in range(4)])
    pkg.save_model(tm, tmp_path / "m.json")
    assert pkg.load_model(tmp_path / "m.json").entries == tm.entries
    doc = json.loads((tmp_path / "m.json").read_text())
    assert doc["data"] == "m.bin" and [t["name"] for t in doc["tensors"]] == tm.names()
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(FormatError):
        pkg.load_model(tmp_path / "bad.json")
    (tmp_path / "r.json").write_text('{"tensors": [{"name": "a", "offset": 0, "length": 10}], "data": "r.bin"}')
    (tmp_path / "r.bin").write_bytes(b"short")
    with pytest.raises(FormatError):
        pkg.load_model(tmp_path / "r.json")


def test_model_manifest_large_file_is_read_in_parallel_and_viewed(tmp_path):
    """A data file above the direct-read threshold goes through the C pool (parallel pread); every tensor is a
    read-only view that still compares equal to the ``bytes`` the reference builds (model.py:335-352)."""
    rng = random.Random(44)
    sizes = [5 << 20, 0, 3, (4 << 20) + 17, 8192]
    tm = pkg.TensorMap([(f"l{i}", rng.randbytes(n)) for i, n in enumerate(sizes)])
    pkg.save_model(tm, tmp_path / "big.json")
    loaded = pkg.load_model(tmp_path / "big.json")
    assert loaded.entries == tm.entries and loaded.total_bytes == sum(sizes)
    assert all(memoryview(buf).readonly for _, buf in loaded.entries)
    pkg.save_model(loaded, tmp_path / "again.json")
    assert (tmp_path / "again.bin").read_bytes() == (tmp_path / "big.bin").read_bytes()


def test_dataset_manifest_round_trip_and_validation(tmp_path):
    samples = inputs.dataset_samples(**inputs.DATASET_CASES[0])
    shard, off, ln, ids, src = inputs.pack_samples(samples)
    rows = [(int(ids[i]), int(src[i]), samples[i][2], int(off[i]), int(ln[i])) for i in range(len(samples))]
    man = pkg.DatasetManifest(rows, tmp_path / "s.bin", {1: "ab"})
    man.save(tmp_path / "d.json", shard)
    back = pkg.DatasetManifest.load(tmp_path / "d.json")
    assert back.samples == rows and back.expected_digests == {1: "ab"}
    assert back.source_ids == frozenset(int(s) for s in src)
    seen = []
    for batch in pkg.iterate_batches(back, 37, shuffle_seed=5):
        assert 1 <= batch.size <= 37
        seen += [(s.sample_id, s.source_id, s.label, s.data) for s in batch.samples]
    assert sorted(seen) == sorted(samples)
    with pytest.raises(pkg.errors.ValidationError):
        list(pkg.iterate_batches(back, 0, 0))
    dup = pkg.DatasetManifest(rows + [rows[0]], tmp_path / "s.bin")
    dup.save(tmp_path / "dup.json", shard)
    with pytest.raises(FormatError):
        pkg.DatasetManifest.load(tmp_path / "dup.json")


# ---- benchmark layouts ------------------------------------------

@pytest.mark.parametrize("arch,entries,nbytes,leaves,ragged", [
    ("gpt2", 149, 652_148_736, 79_672, 100),
    ("gpt2-xl", 581, 6_552_089_600, 799_954, 388),
    ("gpt2-model", 148, 497_759_232, 60_825, 99),
    ("gpt2-xl-model", 580, 6_230_444_800, 760_690, 387),
    ("bert-large", 391, 1_340_567_552, 163_753, 219),
    ("vgg19", 38, 574_668_960, 70_164, 18),
    ("bert-base", 199, 437_928_960, 53_534, 125),          # SURVEY.md section 8, context rows
    ("resnet152", 932, 241_378_168, 30_093, 761),
])
def test_state_dict_layouts(arch, entries, nbytes, leaves, ragged):
    st = shapes.layout_stats(shapes.ARCHITECTURES[arch]())
    assert (st["entries"], st["bytes"], st["leaves"], st["ragged"]) == (entries, nbytes, leaves, ragged)


def test_resnet152_layout_equals_torchvision():
    tv = pytest.importorskip("torchvision")
    import torch

    with torch.device("meta"):
        sd = tv.models.resnet152(weights=None).state_dict()
    layout = shapes.ARCHITECTURES["resnet152"]()
    assert [n for n, _, _ in layout] == list(sd.keys())
    assert [shapes.numel(s) * 4 for _, s, _ in layout] == [v.numel() * v.element_size() for v in sd.values()]


def test_gpt2_lm_head_is_tied():
    layout = shapes.gpt2_lm_head(1600, 48)
    assert layout[-1] == ("lm_head.weight", (50257, 1600), "transformer.wte.weight")
    assert len({n for n, _, _ in layout}) == len(layout)


# ---- shard planning -------------------------------------------------

def test_chunk_ranges_rule():
    assert workers.chunk_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert workers.chunk_ranges(2, 8) == [(0, 1), (1, 2)]
    assert workers.chunk_ranges(0, 4) == []
    assert workers.resolve_workers(3) == 3


def test_shard_plans_cover_all_leaves_on_aligned_boundaries():
    for n in (1, 2, 7, 1000, 1024, 1025, 79_672, 799_954):
        for world in (1, 2, 3, 4, 8):
            sp = dd.plan_shards(n, world)
            assert sp.n_shards == -(-n // (1 << sp.levels))
            assert n == 1 or (1 << sp.levels) < n
            covered = 0
            for r in range(world):
                a, b = sp.leaf_range(r)
                assert a % (1 << sp.levels) == 0 and (b % (1 << sp.levels) == 0 or b == n)
                assert a == covered or a == b
                covered = max(covered, b)
                assert sp.shard_count(r) == -(-(b - a) // (1 << sp.levels))
            assert covered == n
    sp = dd.plan_shards(799_954, 8)
    assert sp.levels == 10 and sp.n_shards == 782
    assert sorted({sp.shard_count(r) for r in range(8)}) == [97, 98]       # balanced, no idle GPU


def test_staged_bytes_counts_only_overlapping_tensors():
    tm = pkg.TensorMap([("a", bytes(8192 * 3)), ("b", bytes(100)), ("c", bytes(8192 * 2))])
    assert dd.staged_bytes(tm, 8192, 0, 6) == tm.total_bytes
    assert dd.staged_bytes(tm, 8192, 0, 2) == 8192 * 3
    assert dd.staged_bytes(tm, 8192, 3, 4) == 100
    assert dd.staged_bytes(tm, 8192, 4, 6) == 8192 * 2


# ---- lattice value algebra on the host (lattice.py:69-89) -------------------------------------

def test_lattice_add_sub_vectors(golden):
    for rec in golden["lattice"]["add"]:
        a, b = pkg.LatticeDigest.from_hex(rec["a"]), pkg.LatticeDigest.from_hex(rec["b"])
        assert pkg.lt_add(a, b).hex() == rec["sum"]
        assert pkg.lt_sub(a, b).hex() == rec["diff"]
        assert pkg.lt_sub(pkg.lt_add(a, b), b) == a
        assert pkg.lt_add(a, pkg.lt_zero()) == a
    wrap = pkg.LatticeDigest(struct.pack("<32H", *([0xFFFF] * 32)))
    one = pkg.LatticeDigest(struct.pack("<32H", *([1] * 32)))
    assert pkg.lt_add(wrap, one) == pkg.lt_zero()
    assert pkg.lt_sub(pkg.lt_zero(), one) == wrap
    with pytest.raises(ValueError):
        pkg.LatticeDigest(b"short")
    assert len(pkg.lt_zero().partitions()) == 32 and len(pkg.lt_zero().words()) == 8


def test_source_accumulator_merge_is_commutative():
    a, b = pkg.SourceAccumulator(), pkg.SourceAccumulator()
    a.declare([1, 2])
    x = pkg.LatticeDigest(inputs.seeded_bytes(1, 64))
    y = pkg.LatticeDigest(inputs.seeded_bytes(2, 64))
    a.sums[1], a.counts[1] = x, 3
    b.sums[1], b.counts[1] = y, 4
    b.sums[5], b.counts[5] = x, 1
    a.merge(b)
    assert a.sums[1] == pkg.lt_add(x, y) and a.counts[1] == 7 and a.sums[5] == x
    fin = pkg.finalize(a)
    assert list(fin) == [1, 2, 5] and fin[2] == (pkg.lt_zero(), 0)


# ---- attestation formats (attestation.py:93-106, :231-284) --------------------------------------

def _golden_statement():
    return pkg.Statement([pkg.Subject("model-x", {"sha256": "ab" * 32}),
                          pkg.Subject("data:source:3", {"lthash": "cd" * 64})],
                         pkg.attestation.MODEL_PREDICATE_TYPE,
                         {"construction": "merkle", "compression": "sha256", "strategy": "in-place",
                          "block_size": 8192, "ordered_per_layer": False, "index_encoding": "le64-prefix-v1",
                          "note": "héllo"})


def test_canonical_json_pae_and_deterministic_signature_match_the_reference(golden, tmp_path):
    g = golden["attestation"]
    stmt = _golden_statement()
    assert base64.b64encode(pkg.canonicalize(stmt)).decode() == g["canonical_b64"]
    assert base64.b64encode(pkg.attestation.pae(pkg.attestation.PAYLOAD_TYPE, pkg.canonicalize(stmt))).decode() == g["pae_b64"]
    assert pkg.attestation.pae("t", b"body") == b"DSSEv1 1 t 4 body" == g["pae_small"].encode()
    (tmp_path / "k.pem").write_text(inputs.TEST_KEY_PEM)
    key = pkg.KeyPair.load(tmp_path / "k.pem")
    assert key.key_id == g["key_id"] and key.public_point_hex == g["public_point_hex"]
    bundle = pkg.sign_bundle(stmt, key)
    assert bundle.to_dict() == g["bundle"]                       # RFC 6979: byte-identical signature
    ref_bundle = pkg.Bundle.from_dict(g["bundle"])               # a bundle the reference wrote verifies here
    fresh = {"model-x": {"sha256": "ab" * 32}, "data:source:3": {"lthash": "cd" * 64}}
    assert pkg.verify_bundle(ref_bundle, fresh) is pkg.Verdict.OK


def test_verdict_classes_and_precedence(tmp_path):
    key = pkg.keygen()
    stmt = _golden_statement()
    bundle = pkg.sign_bundle(stmt, key)
    fresh = {"model-x": {"sha256": "ab" * 32}, "data:source:3": {"lthash": "cd" * 64}}
    assert pkg.verify_bundle(bundle, fresh) is pkg.Verdict.OK
    assert pkg.verify_bundle(bundle, {"model-x": {"sha256": "ab" * 32}}) is pkg.Verdict.DIGEST_MISMATCH
    assert pkg.verify_bundle(bundle, dict(fresh, **{"model-x": {"sha256": "00" * 32}})) is pkg.Verdict.DIGEST_MISMATCH
    other = pkg.sign_bundle(stmt, pkg.keygen())
    forged = pkg.Bundle(bundle.verification_material, other.envelope)
    assert pkg.verify_bundle(forged, fresh) is pkg.Verdict.SIGNATURE_INVALID
    # payload flipped: signature check fails before digests are looked at
    raw = bytearray(base64.b64decode(bundle.envelope.payload))
    raw[raw.index(b"model-x")] ^= 1
    flipped = pkg.Bundle(bundle.verification_material,
                         pkg.Envelope(base64.b64encode(bytes(raw)).decode(), bundle.envelope.payload_type,
                                      bundle.envelope.signatures))
    assert pkg.verify_bundle(flipped, {}) is pkg.Verdict.SIGNATURE_INVALID
    broken = pkg.Bundle(bundle.verification_material,
                        pkg.Envelope("!!not base64!!", bundle.envelope.payload_type, bundle.envelope.signatures))
    assert pkg.verify_bundle(broken, fresh) is pkg.Verdict.MALFORMED
    with pytest.raises(FormatError):
        pkg.Bundle.from_json("{truncated")
    with pytest.raises(FormatError):
        pkg.Bundle.from_dict({"verificationMaterial": {"public_key": "00"}, "envelope":
                              {"payload": "", "payloadType": "x", "signatures": []}})
    bundle.save(tmp_path / "b.json")
    assert pkg.Bundle.load_file(tmp_path / "b.json").to_dict() == bundle.to_dict()
    key.save(tmp_path / "priv.pem", tmp_path / "pub.pem")
    with pytest.raises(KeyMaterialError):
        key.save(tmp_path / "priv.pem", tmp_path / "pub.pem")
    assert pkg.KeyPair.load(tmp_path / "priv.pem").public_point_hex == key.public_point_hex
    with pytest.raises(FormatError):
        pkg.canonicalize(pkg.Statement([], "t", {}))
    with pytest.raises(FormatError):
        pkg.canonicalize(pkg.Statement([pkg.Subject("s", {"sha256": "abcd"})], "t", {}))


def test_block_size_above_the_abi_range_is_a_config_error():
    """A block size the uint32 ABI parameter cannot carry is refused before anything is allocated."""
    import paper_2510_00554_b200 as pkg

    for bs in (1 << 32, 1 << 40):
        cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.COALESCED, pkg.CompressionAlg.SHA256, bs)
        with pytest.raises(pkg.errors.ConfigError):
            cfg.validate()
        with pytest.raises(pkg.errors.ConfigError):
            pkg.hash_model(cfg, pkg.TensorMap([("a", b"x" * 10)]))
        pred = dict(cfg.predicate())
        with pytest.raises(pkg.errors.ConfigError):
            pkg.HashConfig.from_predicate(pred)
    pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.SHA256, 1 << 31).validate()


def test_sample_ids_outside_u64_are_rejected_not_wrapped():
    import paper_2510_00554_b200 as pkg
    from paper_2510_00554_b200 import dataset as dsm

    for bad in (-1, 1 << 64):
        with pytest.raises(pkg.errors.ValidationError):
            dsm._checked_ids([0, bad])
        acc = pkg.SourceAccumulator()
        with pytest.raises(pkg.errors.ValidationError):          # raised before anything touches the device
            pkg.process_batch(pkg.Batch([pkg.SampleRecord(bad, 0, b"", b"data")]), acc)
    assert dsm._checked_ids([0, (1 << 64) - 1]).dtype.name == "uint64"
