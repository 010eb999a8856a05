"""GPU parity: the CUDA path (through the C ABI) against the golden vectors and the oracles.

Every comparison is bit-exact. Sizes the oracle finishes in seconds are compared
directly (including full-size GPT-2 small, 652 MB, against the multi-threaded C
oracle); the multi-shard and leaf-range paths are additionally checked through
size-independent properties (shard roots recombine to the whole-model root).
"""

import hashlib
import struct

import numpy as np
import pytest

import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ALGS = ["sha256", "blake2b", "sha3-256"]


@pytest.fixture(scope="module")
def pkg():
    import paper_2510_00554_b200 as pkg
    from paper_2510_00554_b200 import _native, device

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    _native.load()          # the native library must be the thing that runs
    return pkg


def _alg(pkg, name):
    return pkg.CompressionAlg.from_name(name)


# ---- primitives ------------------------------------------------------------------

def test_known_answers_through_hash_blocks(pkg, golden):
    by_alg = {}
    for rec in golden["kats"]:
        data = rec["msg"].encode() if "msg" in rec else inputs.seeded_bytes(rec["seed"], rec["len"])
        by_alg.setdefault(rec["alg"], []).append((data, rec["digest"]))
    for alg, items in by_alg.items():
        buf = pkg.hash_blocks(_alg(pkg, alg), [d for d, _ in items])
        assert buf.count == len(items)
        for i, (_, want) in enumerate(items):
            assert buf.entry(i).hex() == want, (alg, i, len(items[i][0]))


def test_compress_block_empty_and_abc(pkg):
    assert pkg.compress_block(pkg.CompressionAlg.SHA256, b"").hex() == \
        "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    assert pkg.compress_block(pkg.CompressionAlg.SHA3_256, b"abc").hex() == \
        "3a985da74fe225b2045c172d6bd390bd855f086e3e9d525b46bfe24511431532"
    assert len(pkg.compress_block(pkg.CompressionAlg.BLAKE2B, b"x").data) == 64


def test_hash_blocks_unaligned_device_views(pkg, porc):
    """Blocks addressed in place at every byte alignment and ragged length."""
    from paper_2510_00554_b200 import device as dev

    raw = inputs.seeded_bytes(77, 70_000)
    base = dev.as_device_bytes(raw)
    rng = np.random.default_rng(5)
    offs = np.concatenate([np.arange(0, 40), rng.integers(0, 60_000, 200)]).astype(np.uint64)
    lens = np.concatenate([np.arange(0, 40) * 7 % 300, rng.integers(0, 9000, 200)]).astype(np.uint64)
    d_off = torch.from_numpy(offs.view(np.int64)).cuda()
    d_len = torch.from_numpy(lens.view(np.int64)).cuda()
    for alg in ALGS:
        out = dev.hash_blocks_device(alg, base, d_off, d_len).cpu().numpy().tobytes()
        dl = porc.DIGEST_LEN[alg]
        for i, (o, l) in enumerate(zip(offs, lens)):
            assert out[i * dl:(i + 1) * dl] == porc.h(alg, raw[int(o):int(o + l)]), (alg, i, int(o), int(l))


def test_hash_blocks_zero_blocks_rejected(pkg):
    with pytest.raises(pkg.errors.InvalidInput):
        pkg.hash_blocks(pkg.CompressionAlg.SHA256, [])


# ---- merkle ------------------------------------------------------------------------

def test_merkle_roots_golden(pkg, golden):
    for rec in golden["merkle"]:
        alg = _alg(pkg, rec["alg"])
        n = rec["n"]
        leaves = inputs.seeded_bytes(rec["seed"], n * alg.digest_len)
        buf = pkg.DigestBuffer(alg, bytearray(leaves), n)
        assert pkg.merkle_root(alg, buf).hex() == rec["root"], (rec["alg"], n)


def test_reduce_level_matches_oracle_and_state_machine(pkg, porc):
    for name in ALGS:
        alg = _alg(pkg, name)
        for n in (2, 3, 8, 33):
            leaves = inputs.seeded_bytes(600 + n, n * alg.digest_len)
            state = pkg.ReductionState.from_leaves(pkg.DigestBuffer(alg, bytearray(leaves), n))
            level, count = leaves, n
            while count > 1:
                got = pkg.reduce_level(state)
                level = bytes(porc.reduce_level(name, level, count))
                count = (count + 1) // 2
                assert got == count
                assert bytes(state.input_buffer.data[:count * alg.digest_len]) == level
            with pytest.raises(pkg.errors.InvalidState):
                pkg.reduce_level(state)


def test_reduce_levels_forced_ranges(pkg, porc):
    """The shard rule on the device: any aligned node range, any forced level count."""
    from paper_2510_00554_b200 import device as dev

    for name in ALGS:
        dl = porc.DIGEST_LEN[name]
        for n in (1, 5, 100, 1500, 5000):
            leaves = inputs.seeded_bytes(900 + n, n * dl)
            nodes = dev.as_device_bytes(leaves)
            for levels in (1, 2, 3, 6, 10, 11, 13):
                if levels > max(1, (n - 1).bit_length()) + 1:
                    continue
                width = 1 << levels
                # whole range
                got = dev.merkle_reduce_levels_device(name, nodes, 0, n, n, levels).cpu().numpy().tobytes()
                want = porc.reduce_levels_forced(name, leaves, 0, n, n, levels)
                assert got == want, (name, n, levels)
                # a sub-range starting on a shard boundary
                if n > 2 * width:
                    first = width
                    n_in = min(n - first, 2 * width) if (n - first) >= 2 * width else n - first
                    sub = dev.as_device_bytes(leaves[first * dl:(first + n_in) * dl])
                    got = dev.merkle_reduce_levels_device(name, sub, first, n_in, n, levels).cpu().numpy().tobytes()
                    want = porc.reduce_levels_forced(name, leaves[first * dl:(first + n_in) * dl], first, n_in, n, levels)
                    assert got == want, (name, n, levels, "sub")


# ---- models --------------------------------------------------------------------------

def test_reference_suite_golden_inplace_digest(pkg):
    import random

    rng = random.Random(2024)
    model = pkg.TensorMap([(f"t{i}", rng.randbytes(s)) for i, s in enumerate([100, 8192, 5000, 0, 20000])])
    res = pkg.hash_model(pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE), model)
    assert res.digest_hex() == "5d70823521307e19d8a9451a8c264c8cd156ee99a9d7f46e9406867d712c9a7e"
    assert res.block_count == 6
    assert res.layer_digests is None and res.aux_data_bytes == 0


def test_seeded_models_root_and_every_leaf(pkg, golden):
    from paper_2510_00554_b200 import device as dev

    for rec in golden["models"]:
        if rec["kind"] != "seeded":
            continue
        tensors = inputs.model_tensors(rec["seed"], rec["sizes"])
        model = pkg.TensorMap([(f"t{i}", t) for i, t in enumerate(tensors)])
        bs = rec["block_size"]
        for name in ALGS:
            cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, _alg(pkg, name), bs)
            res = pkg.hash_model(cfg, model)
            assert res.digest_hex() == rec[f"merkle_inplace_{name}"], (rec["case"], bs, name)
            assert res.block_count == rec["n_blocks"]
            plan = dev.ModelPlan([dev.as_device_bytes(t) for t in tensors], bs)
            hasher = dev.MerkleModelHasher(plan, name)
            hasher.run()
            assert hashlib.sha256(hasher.leaf_bytes()).hexdigest() == rec[f"leaves_sha256_{name}"]
            assert hasher.out_bytes().hex() == rec[f"merkle_inplace_{name}"]
            cfg_c = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.COALESCED, _alg(pkg, name), bs)
            assert pkg.hash_model(cfg_c, model).digest_hex() == rec[f"merkle_coalesced_{name}"]
            cfg_p = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.PER_LAYER, _alg(pkg, name), bs)
            pl = pkg.hash_model(cfg_p, model)
            assert pl.digest_hex() == rec[f"merkle_per_layer_{name}"], (rec["case"], bs, name)
            assert list(pl.layer_digests) == model.names()
            assert hashlib.sha256(b"".join(d.data for d in pl.layer_digests.values())).hexdigest() == \
                rec[f"merkle_layers_sha256_{name}"]
            assert pl.block_count == rec["per_layer_block_count"]
        for ordered in (False, True):
            cfg_l = pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.PER_LAYER, pkg.CompressionAlg.BLAKE2B, bs,
                                   ordered_per_layer=ordered)
            pl = pkg.hash_model(cfg_l, model)
            assert pl.digest_hex() == rec["lattice_per_layer"], (rec["case"], bs, ordered)
            assert hashlib.sha256(b"".join(d.data for d in pl.layer_digests.values())).hexdigest() == \
                rec["lattice_layers_sha256"]
        lat = pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.BLAKE2B, bs)
        assert pkg.hash_model(lat, model).digest_hex() == rec["lattice_inplace"], (rec["case"], bs)
        lat_c = pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.COALESCED, pkg.CompressionAlg.BLAKE2B, bs)
        assert pkg.hash_model(lat_c, model).digest_hex() == rec["lattice_coalesced"]


def test_unaligned_device_tensors_hashed_in_place(pkg, porc):
    """Views at 1-, 2-, 4-, 8-byte offsets into one allocation (storage offsets of real checkpoints)."""
    raw = inputs.seeded_bytes(31, 200_000)
    base = torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()
    cuts = [(1, 9000), (9003, 8192), (17200, 33000), (50204, 1), (50208, 70000), (120216, 16384)]
    entries = [(f"v{i}", base[o:o + l]) for i, (o, l) in enumerate(cuts)]
    host = [raw[o:o + l] for o, l in cuts]
    for name in ALGS:
        for bs in (64, 8192):
            cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, _alg(pkg, name), bs)
            assert pkg.hash_model(cfg, pkg.TensorMap(entries)).model_digest.data == porc.inplace_merkle(name, host, bs)
    cfg = pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.BLAKE2B, 1024)
    assert pkg.hash_model(cfg, pkg.TensorMap(entries)).model_digest.data == porc.inplace_lattice(host, 1024)


def test_host_model_staged_in_overlapped_chunks(pkg, corc, monkeypatch):
    """Large host models take the copy/hash pipeline: same root, with CUDA entries mixed in."""
    from paper_2510_00554_b200 import model as mm

    monkeypatch.setattr(mm, "STAGE_CHUNK_BYTES", 3 << 20)          # several chunks at test size
    monkeypatch.setattr(mm, "STAGE_PIECE_BYTES", 1 << 20)          # tensors travel in pieces, the device ring wraps
    rng = np.random.default_rng(11)
    sizes = [5 << 20, 100, 0, (7 << 20) + 13, 8192, 3, (9 << 20) + 4096, 12 << 20, 6400, (2 << 20) + 1]
    host = [rng.integers(0, 256, size=s, dtype=np.uint8) for s in sizes]
    entries = []
    for i, h in enumerate(host):
        if i in (3, 8):
            entries.append((f"t{i}", torch.from_numpy(h).cuda()))          # already resident
        elif i % 2:
            entries.append((f"t{i}", torch.from_numpy(h).pin_memory()))    # pinned host tensor
        else:
            entries.append((f"t{i}", h.tobytes()))                         # plain bytes
    assert sum(sizes) >= mm.STAGE_PIPELINE_MIN_BYTES
    tl = corc.TensorList(host)
    for name in ALGS:
        cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, _alg(pkg, name), 8192)
        res = pkg.hash_model(cfg, pkg.TensorMap(entries))
        assert res.model_digest.data == corc.inplace_merkle(name, tl, 8192, 4), name
        assert res.block_count == tl.leaf_count(8192)


def test_page_locked_model_copy_first_with_small_tensors_through_the_gather(pkg, corc, monkeypatch):
    """Every host tensor page-locked (plus CUDA entries): the copy-first path. Tensors below SMALL_H2D_BYTES are
    fetched by one gather launch straight from the pinned host memory, the others by the copy engine; sizes on both
    sides of the threshold, empty tensors, odd lengths, several copy/hash groups."""
    from paper_2510_00554_b200 import model as mm

    monkeypatch.setattr(mm, "STAGE_CHUNK_BYTES", 6 << 20)
    monkeypatch.setattr(mm, "STAGE_PIECE_BYTES", 2 << 20)          # ring = 4 x 8 MB < the model: it wraps
    rng = np.random.default_rng(17)
    small = mm.SMALL_H2D_BYTES
    sizes = [17 << 20, 3, 0, small - 1, small, small + 1, (7 << 20) + 13, 6400, 8192, 1, (15 << 20) + 5, 100, 0, 4096 * 3]
    host = [rng.integers(0, 256, size=s, dtype=np.uint8) for s in sizes]
    entries = [(f"t{i}", torch.from_numpy(h).cuda() if i in (6, 11) else torch.from_numpy(h).pin_memory())
               for i, h in enumerate(host)]
    assert sum(sizes) >= mm.STAGE_PIPELINE_MIN_BYTES
    taken = []
    real = mm._inplace_merkle_host
    monkeypatch.setattr(mm, "_inplace_merkle_host", lambda cfg, model, workers=1: taken.append(1) or real(cfg, model, workers))
    tl = corc.TensorList(host)
    for name in ALGS:
        cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, _alg(pkg, name), 8192)
        for _ in range(2):
            res = pkg.hash_model(cfg, pkg.TensorMap(entries))
            assert res.model_digest.data == corc.inplace_merkle(name, tl, 8192, 4), name
            assert res.block_count == tl.leaf_count(8192)
    assert len(taken) == 2 * len(ALGS)
    assert mm.LAST_HOST_STAGING["ring_bytes"] < mm.LAST_HOST_STAGING["host_bytes"]      # bounded device memory
    lat = pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.BLAKE2B, 8192)
    assert pkg.hash_model(lat, pkg.TensorMap(entries)).model_digest.data == corc.inplace_lattice(tl, 8192, 4)
    # block sizes on both sides of the piece size (a piece is a whole number of blocks, at least one)
    for bs in (64, 4 << 20):
        cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, _alg(pkg, "sha256"), bs)
        assert pkg.hash_model(cfg, pkg.TensorMap(entries)).model_digest.data == corc.inplace_merkle("sha256", tl, bs, 4), bs


@pytest.mark.parametrize("slot_kb,piece_kb", [(1024, 256), (768, 1000), (32768, 4096)])
def test_pageable_inputs_through_the_staging_ring(pkg, corc, monkeypatch, slot_kb, piece_kb):
    """bytes / numpy / unpinned tensors ride the pinned ring: tensors straddle transfers, slots wrap around."""
    from paper_2510_00554_b200 import device as dv, model as mm

    monkeypatch.setattr(dv, "STAGE_SLOT_BYTES", slot_kb << 10)
    monkeypatch.setattr(dv, "STAGE_PIECE_BYTES", piece_kb << 10)
    monkeypatch.setattr(mm, "STAGE_CHUNK_BYTES", 5 << 20)
    monkeypatch.setattr(mm, "STAGE_PIECE_BYTES", (1 << 20) if slot_kb < 32768 else (64 << 20))   # wrapping device ring / one arena
    rng = np.random.default_rng(12)
    sizes = [(3 << 20) + 77, 1, 0, 8192 * 300, (6 << 20) + 8191, 255, 257, (11 << 20) + 5, 4096, (9 << 20)]
    host = [rng.integers(0, 256, size=s, dtype=np.uint8) for s in sizes]
    entries = []
    for i, h in enumerate(host):
        kind = i % 4
        buf = h.tobytes() if kind == 0 else h if kind == 1 else torch.from_numpy(h.copy()) if kind == 2 \
            else torch.from_numpy(h).view(torch.uint8)
        if i == 4:
            buf = torch.from_numpy(h[:-3].copy()).view(torch.float32)      # a float tensor, pageable
            host[i] = h[:-3]
        if i == 7:
            buf = torch.from_numpy(h).pin_memory()                         # one pinned entry in between
        entries.append((f"t{i}", buf))
    tl = corc.TensorList(host)
    for name in ALGS:
        cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, _alg(pkg, name), 8192)
        for workers in (1, 3):
            res = pkg.hash_model(cfg, pkg.TensorMap(entries), workers=workers)
            assert res.model_digest.data == corc.inplace_merkle(name, tl, 8192, 4), (name, workers)
    lat = pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.BLAKE2B, 8192)
    assert pkg.hash_model(lat, pkg.TensorMap(entries)).model_digest.data == corc.inplace_lattice(tl, 8192, 4)
    # the generic helper behind as_device_bytes (dataset shards, lattice / per-layer / coalesced model paths)
    monkeypatch.setattr(dv, "STAGE_DIRECT_MAX_BYTES", 1 << 20)
    big = rng.integers(0, 256, size=(7 << 20) + 321, dtype=np.uint8)
    for src in (big.tobytes(), big, torch.from_numpy(big.copy())):
        assert bytes(dv.as_device_bytes(src).cpu().numpy().tobytes()) == big.tobytes()


def test_per_layer_full_size_vgg19_against_oracle(pkg, porc):
    """38 layer digests of the VGG19 layout (scaled) for both constructions, against the oracle."""
    sd = _synthetic("vgg19", scale=0.06)
    model = pkg.TensorMap(list(sd))
    host = [t.cpu().numpy().tobytes() for _, t in sd]
    for name in ("sha256", "sha3-256"):
        res = pkg.hash_model(pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.PER_LAYER, _alg(pkg, name)), model)
        root, layers = porc.per_layer_merkle(name, host, 8192)
        assert len(res.layer_digests) == 38
        assert [d.data for d in res.layer_digests.values()] == layers and res.model_digest.data == root
    res = pkg.hash_model(pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.PER_LAYER, pkg.CompressionAlg.BLAKE2B), model)
    root, layers = porc.per_layer_lattice(host, 8192)
    assert [d.data for d in res.layer_digests.values()] == layers and res.model_digest.data == root
    with pytest.raises(pkg.errors.ConfigError):
        pkg.ordered_lattice_per_layer(pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.PER_LAYER,
                                                     pkg.CompressionAlg.BLAKE2B), model)


def test_empty_model_and_bad_config(pkg):
    cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE)
    with pytest.raises(pkg.errors.InvalidInput):
        pkg.hash_model(cfg, pkg.TensorMap([("a", b"")]))
    with pytest.raises(pkg.errors.InvalidInput):
        pkg.hash_model(cfg, pkg.TensorMap([]))
    with pytest.raises(pkg.errors.ConfigError):
        pkg.hash_model(pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.SHA256),
                       pkg.TensorMap([("a", b"x")]))
    single = pkg.hash_model(cfg, pkg.TensorMap([("t", b"z" * 100)]))
    assert single.model_digest.data == hashlib.sha256(b"z" * 100).digest() and single.block_count == 1


def _synthetic(arch, scale=1.0):
    from paper_2510_00554_b200 import shapes

    return shapes.synthetic_state_dict(arch, torch.device("cuda"), seed=0, scale=scale)


@pytest.mark.parametrize("arch,alg", [("gpt2", "sha256"), ("gpt2-xl", "sha256"),
                                      ("vgg19", "blake2b"), ("vgg19", "sha3-256"),
                                      ("bert-large", "blake2b"), ("bert-large", "sha3-256")])
def test_full_size_models_against_c_oracle(pkg, corc, arch, alg):
    """BASELINE configs 1, 2 and 4 at full size: root AND every leaf digest, bit-exact."""
    from paper_2510_00554_b200 import device as dev

    sd = _synthetic(arch)
    flat = [dev.as_device_bytes(t) for _, t in sd]
    plan = dev.ModelPlan(flat, 8192)
    hasher = dev.MerkleModelHasher(plan, alg)
    hasher.run()
    host = [t.cpu().numpy() for t in flat]
    tl = corc.TensorList(host)
    threads = corc.threads_default()
    want_leaves = corc.inplace_leaves(alg, tl, 8192, threads)
    assert plan.leaf_count * corc.DLEN[alg] == len(want_leaves)
    got_leaves = hasher.leaf_bytes()
    assert got_leaves == want_leaves
    assert hasher.out_bytes() == corc.merkle_root(alg, want_leaves, plan.leaf_count, threads)
    # the reference-shaped API gives the same root
    cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, _alg(pkg, alg), 8192)
    res = pkg.hash_model(cfg, pkg.TensorMap(list(sd)))
    assert res.model_digest.data == hasher.out_bytes()


@pytest.mark.parametrize("arch", ["gpt2", "bert-large"])
def test_full_size_lattice_model_against_c_oracle(pkg, corc, arch):
    """LATTICE in-place hashing at full model size, through both LtHash schedules for model blocks
    (persistent chains, plain grid), against the multi-threaded C oracle."""
    from paper_2510_00554_b200 import _native

    sd = _synthetic(arch)
    host = [t.reshape(-1).view(torch.uint8).cpu().numpy() for _, t in sd]
    want = corc.inplace_lattice(corc.TensorList(host), 8192, corc.threads_default())
    cfg = pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.BLAKE2B, 8192)
    lib = _native.load()
    try:
        for schedule in (_native.SCHEDULE_PERSISTENT, _native.SCHEDULE_GRID):
            lib.snt_merkle_schedule(schedule)
            assert pkg.hash_model(cfg, pkg.TensorMap(list(sd))).model_digest.data == want, schedule
    finally:
        lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT)


def test_shard_roots_recombine_to_whole_root(pkg):
    """Size-independent property of the multi-GPU rule, on one GPU at GPT-2-small size."""
    from paper_2510_00554_b200 import device as dev
    from paper_2510_00554_b200 import distributed as dd

    sd = _synthetic("gpt2")
    plan = dev.ModelPlan([dev.as_device_bytes(t) for _, t in sd], 8192)
    for alg in ("sha256", "blake2b"):
        whole = dev.MerkleModelHasher(plan, alg)
        whole.run()
        root = whole.out_bytes()
        for world in (2, 3, 8):
            sp = dd.plan_shards(plan.leaf_count, world)
            parts = []
            for rank in range(world):
                a, b = sp.leaf_range(rank)
                if b > a:
                    h = dev.MerkleModelHasher(plan, alg, a, b, sp.levels)
                    h.run()
                    parts.append(h.out)
            nodes = torch.cat(parts)
            assert nodes.numel() == sp.n_shards * dev.DIGEST_LEN[alg]
            assert dev.merkle_root_device(alg, nodes, sp.n_shards).cpu().numpy().tobytes() == root, (alg, world)


# ---- lattice / dataset -------------------------------------------------------------------

def test_lattice_vectors(pkg, golden):
    lat = golden["lattice"]
    for rec in lat["hash_block"]:
        data = inputs.seeded_bytes(rec["seed"], rec["len"])
        assert pkg.lt_hash_block(rec["index"], data).hex() == rec["digest"], rec
    for rec in lat["tagged"]:
        tag = inputs.seeded_bytes(rec["tag_seed"], rec["tag_len"])
        data = inputs.seeded_bytes(rec["seed"], rec["len"])
        assert pkg.lattice.lt_hash_tagged(tag, data).hex() == rec["digest"]
    for rec in lat["reduce"]:
        ds = [pkg.LatticeDigest(inputs.seeded_bytes(rec["seed_base"] + i, 64)) for i in range(rec["n"])]
        assert pkg.lt_reduce(ds).hex() == rec["sum"]
        assert pkg.lattice.lt_reduce_pairwise(ds).hex() == rec["sum"]
    assert pkg.lt_reduce([]).data == bytes(64)
    assert pkg.lt_hash_block(0, b"").data == hashlib.blake2b(bytes(8)).digest()


def test_dataset_golden_process_batch_and_device_path(pkg, golden, tmp_path):
    for rec in golden["datasets"]:
        spec = inputs.DATASET_CASES[rec["case"]]
        samples = inputs.dataset_samples(**spec)
        want = {int(k): (v[0], v[1]) for k, v in rec["digests"].items()}
        # (a) the reference's host-object protocol, batch by batch
        acc = pkg.SourceAccumulator(cover_labels=rec["cover_labels"])
        acc.declare(spec["declared"])
        recs = [pkg.SampleRecord(*s) for s in samples]
        for start in range(0, len(recs), 50):
            pkg.process_batch(pkg.Batch(recs[start:start + 50]), acc)
        got = {sid: (d.hex(), c) for sid, (d, c) in pkg.finalize(acc).items()}
        assert got == want
        # (b) manifest -> digest_dataset (whole shard resident, one launch)
        shard, off, ln, ids, src = inputs.pack_samples(samples)
        rows = [(int(ids[i]), int(src[i]), samples[i][2], int(off[i]), int(ln[i])) for i in range(len(samples))]
        man = pkg.DatasetManifest(rows, tmp_path / "shard.bin")
        man.save(tmp_path / "m.json", shard)
        loaded = pkg.DatasetManifest.load(tmp_path / "m.json")
        got = {sid: (d.hex(), c) for sid, (d, c) in
               pkg.digest_dataset(loaded, batch_size=13, shuffle_seed=4, cover_labels=rec["cover_labels"]).items()}
        assert got == {sid: v for sid, v in want.items() if sid in loaded.source_ids}


def test_undeclared_source_rejected(pkg):
    acc = pkg.SourceAccumulator()
    acc.declare([1, 2])
    with pytest.raises(pkg.errors.ValidationError):
        pkg.process_batch(pkg.Batch([pkg.SampleRecord(5, 3, b"", b"abc")]), acc)


def test_cifar_shaped_dataset_against_c_oracle(pkg, corc):
    """BASELINE config 3 at full size: 50,000 x 3,072-byte samples, 16 sources, every sample digest."""
    from paper_2510_00554_b200 import dataset as ds
    from paper_2510_00554_b200 import device as dev

    n, ln, n_src = 50_000, 3072, 16
    rng = np.random.default_rng(0)
    shard = rng.integers(0, 256, size=n * ln, dtype=np.uint8)
    ids = np.arange(n, dtype=np.uint64)
    probs = np.random.default_rng(1).dirichlet(np.ones(n_src))
    src = np.random.default_rng(1).choice(n_src, size=n, p=probs)
    offs = (np.arange(n, dtype=np.uint64) * ln)
    lens = np.full(n, ln, dtype=np.uint64)
    dset = ds.DeviceDataset.from_host(shard, offs, lens, ids, src, list(range(n_src)))
    acc = dev.LatticeAccumulator(n_src)
    per_sample = torch.empty(n * 64, dtype=torch.uint8, device="cuda")
    dset.accumulate(acc, digests=per_sample)
    out, counts, status = acc.digests()
    want_sums, want_counts, want_digests = corc.lthash_samples(shard, offs, lens, ids, src.astype(np.uint32), n_src,
                                                               corc.threads_default(), want_digests=True)
    assert status == 0
    assert per_sample.cpu().numpy().tobytes() == want_digests
    assert out == want_sums and counts == want_counts
    # split into ranges (the multi-GPU partition) and accumulate: same sums
    acc2 = dev.LatticeAccumulator(n_src)
    for a, b in [(0, 7), (7, 20_001), (20_001, n)]:
        dset.accumulate(acc2, a, b)
    assert acc2.digests()[:2] == (want_sums, want_counts)


def test_hellaswag_shaped_variable_length_samples(pkg, corc):
    """BASELINE config 5 shape: 4*len-byte int32 token arrays, ragged, hashed at true length."""
    from paper_2510_00554_b200 import dataset as ds
    from paper_2510_00554_b200 import device as dev

    n, n_src = 40_000, 16
    rng = np.random.default_rng(2)
    toks = np.clip(np.round(rng.lognormal(np.log(90), 0.4, size=n)), 16, 256).astype(np.int64)
    lens = (toks * 4).astype(np.uint64)
    offs = np.zeros(n, dtype=np.uint64)
    np.cumsum(lens[:-1], out=offs[1:])
    shard = rng.integers(0, 50257, size=int(toks.sum()), dtype=np.int32).view(np.uint8)
    src = np.random.default_rng(3).integers(0, n_src, size=n)
    ids = np.arange(n, dtype=np.uint64) * 7 + 3
    dset = ds.DeviceDataset.from_host(shard, offs, lens, ids, src, list(range(n_src)))
    acc = dev.LatticeAccumulator(n_src)
    dset.accumulate(acc)
    out, counts, _ = acc.digests()
    want_sums, want_counts = corc.lthash_samples(shard, offs, lens, ids, src.astype(np.uint32), n_src, 4)
    assert out == want_sums and counts == want_counts
    assert sum(counts) == n


def test_other_block_sizes_at_scale(pkg, corc):
    """Block sizes 64 B and 1 MiB over a 48 MB ragged model (tree depth 20 and 6)."""
    from paper_2510_00554_b200 import device as dev

    rng = np.random.default_rng(21)
    sizes = [(20 << 20) + 77, 3, (1 << 20), (26 << 20) + 4096 + 5, 64, 8191]
    host = [rng.integers(0, 256, size=s, dtype=np.uint8) for s in sizes]
    flat = [torch.from_numpy(h).cuda() for h in host]
    tl = corc.TensorList(host)
    for bs, algs in ((64, ["sha256"]), (1 << 20, ALGS)):
        plan = dev.ModelPlan(flat, bs)
        for name in algs:
            h = dev.MerkleModelHasher(plan, name)
            h.run()
            want_leaves = corc.inplace_leaves(name, tl, bs, corc.threads_default())
            assert h.leaf_bytes() == want_leaves, (bs, name)
            assert h.out_bytes() == corc.merkle_root(name, want_leaves, plan.leaf_count, 4), (bs, name)


def test_many_sources_take_the_global_accumulator_path(pkg, corc):
    from paper_2510_00554_b200 import dataset as ds
    from paper_2510_00554_b200 import device as dev

    n, n_src = 3000, 300           # > LT_SMEM_SOURCES
    rng = np.random.default_rng(9)
    lens = rng.integers(0, 400, size=n).astype(np.uint64)
    offs = np.zeros(n, dtype=np.uint64)
    np.cumsum(lens[:-1], out=offs[1:])
    shard = rng.integers(0, 256, size=int(lens.sum()) + 16, dtype=np.uint8)
    src = rng.integers(0, n_src, size=n)
    ids = rng.integers(0, 2**63, size=n).astype(np.uint64)
    dset = ds.DeviceDataset.from_host(shard, offs, lens, ids, src, list(range(n_src)))
    acc = dev.LatticeAccumulator(n_src)
    dset.accumulate(acc)
    out, counts, _ = acc.digests()
    want_sums, want_counts = corc.lthash_samples(shard, offs, lens, ids, src.astype(np.uint32), n_src, 2)
    assert out == want_sums and counts == want_counts


def test_lthash_ragged_unaligned_and_empty_samples(pkg, corc):
    """Every byte alignment, lengths around the BLAKE2b block boundaries, empty samples; also the model path."""
    from paper_2510_00554_b200 import dataset as ds
    from paper_2510_00554_b200 import device as dev

    n, n_src = 2500, 7
    rng = np.random.default_rng(41)
    lens = rng.choice([0, 1, 7, 8, 9, 119, 120, 121, 127, 128, 129, 247, 248, 249, 256, 1000, 3072], size=n).astype(np.uint64)
    lens[:200] = rng.integers(0, 5000, size=200)
    gaps = rng.integers(0, 5, size=n).astype(np.uint64)            # every byte alignment
    offs = np.zeros(n, dtype=np.uint64)
    np.cumsum((lens + gaps)[:-1], out=offs[1:])
    offs += 3
    shard = rng.integers(0, 256, size=int(offs[-1] + lens[-1]) + 64, dtype=np.uint8)
    src = rng.integers(0, n_src, size=n)
    ids = rng.integers(0, 2**63, size=n).astype(np.uint64)
    want_sums, want_counts, want_digests = corc.lthash_samples(shard, offs, lens, ids, src.astype(np.uint32), n_src, 4,
                                                               want_digests=True)
    dset = ds.DeviceDataset.from_host(shard, offs, lens, ids, src, list(range(n_src)))
    acc = dev.LatticeAccumulator(n_src)
    per_sample = torch.empty(n * 64, dtype=torch.uint8, device="cuda")
    dset.accumulate(acc, digests=per_sample)
    out, counts, status = acc.digests()
    # the model lattice path (leaf items) through the same kernel
    tensors = inputs.model_tensors(17, [40000, 123, 8192 * 3, 9999, 1, 2, 70001])
    cfg = pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.BLAKE2B, 1024)
    got_model = pkg.hash_model(cfg, pkg.TensorMap([(f"t{i}", t) for i, t in enumerate(tensors)])).model_digest.data
    assert status == 0
    assert per_sample.cpu().numpy().tobytes() == want_digests
    assert out == want_sums and counts == want_counts
    assert got_model == corc.inplace_lattice(corc.TensorList(tensors), 1024, 2)


def test_sharded_entry_point_on_one_rank_and_sparse_staging(pkg, porc):
    """hash_model_sharded with world == 1 equals hash_model; a rank stages only the tensors it needs."""
    from paper_2510_00554_b200 import distributed as dd

    tensors = inputs.model_tensors(16, [40000, 123, 8192 * 3, 9999, 1, 2, 70001, 8192 * 300 + 5])
    model = pkg.TensorMap([(f"t{i}", t) for i, t in enumerate(tensors)])
    for name in ALGS:
        cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, _alg(pkg, name), 8192)
        want = porc.inplace_merkle(name, tensors, 8192)
        assert dd.hash_model_sharded(cfg, model, 0, 1).model_digest.data == want
    # emulate rank r of a 3-rank job without a process group: its shard roots from sparsely staged tensors
    from paper_2510_00554_b200 import device as dev
    sizes = [len(t) for t in tensors]
    first = dd._first_leaves(sizes, 8192)
    sp = dd.plan_shards(first[-1], 3, levels=4)
    parts = []
    for rank in range(3):
        a, b = sp.leaf_range(rank)
        if b <= a:
            continue
        placeholder = torch.zeros(16, dtype=torch.uint8, device="cuda")
        staged = [dev.as_device_bytes(t) if (first[i] < b and first[i + 1] > a) else placeholder
                  for i, t in enumerate(tensors)]
        plan = dev.ModelPlan(staged, 8192, sizes_override=sizes)
        h = dev.MerkleModelHasher(plan, "sha256", a, b, sp.levels)
        h.run()
        parts.append(h.out.clone())
    nodes = torch.cat(parts)
    assert dev.merkle_root_device("sha256", nodes, sp.n_shards).cpu().numpy().tobytes() == \
        porc.inplace_merkle("sha256", tensors, 8192)


def test_multi_curator_dataset_sign_and_verify(pkg):
    """BASELINE config 5 shape: per-source LtHash on the GPU, one P-256 key per curator on the host."""
    samples = inputs.dataset_samples(**inputs.DATASET_CASES[2])          # 16 sources
    acc = pkg.SourceAccumulator()
    acc.declare(inputs.DATASET_CASES[2]["declared"])
    pkg.process_batch(pkg.Batch([pkg.SampleRecord(*s) for s in samples]), acc)
    digests = pkg.finalize(acc)
    keys = {sid: pkg.keygen() for sid in digests}
    bundles = {}
    for sid, (digest, count) in digests.items():
        stmt = pkg.Statement([pkg.Subject(f"ds:source:{sid}", {"lthash": digest.hex()})],
                             pkg.attestation.DATASET_PREDICATE_TYPE,
                             {"source_id": sid, "sample_count": count, "cover_labels": False,
                              "index_encoding": "le64-prefix-v1"})
        bundles[sid] = pkg.sign_bundle(stmt, keys[sid])
    # verifier: recompute on the GPU in another order / batching, check every curator's bundle
    acc2 = pkg.SourceAccumulator()
    acc2.declare(inputs.DATASET_CASES[2]["declared"])
    recs = [pkg.SampleRecord(*s) for s in reversed(samples)]
    for start in range(0, len(recs), 33):
        pkg.process_batch(pkg.Batch(recs[start:start + 33]), acc2)
    fresh = pkg.finalize(acc2)
    for sid, bundle in bundles.items():
        name = f"ds:source:{sid}"
        assert pkg.verify_bundle(bundle, {name: {"lthash": fresh[sid][0].hex()}}) is pkg.Verdict.OK
        other = next(k for k in keys if k != sid)
        forged = pkg.Bundle({"public_key": keys[other].public_point_hex}, bundle.envelope)
        assert pkg.verify_bundle(forged, {name: {"lthash": fresh[sid][0].hex()}}) is pkg.Verdict.SIGNATURE_INVALID
    # drop one sample of one source: only that curator's bundle fails
    victim = samples[0][1]
    acc3 = pkg.SourceAccumulator()
    acc3.declare(inputs.DATASET_CASES[2]["declared"])
    pkg.process_batch(pkg.Batch([pkg.SampleRecord(*s) for s in samples[1:]]), acc3)
    tampered = pkg.finalize(acc3)
    for sid, bundle in bundles.items():
        verdict = pkg.verify_bundle(bundle, {f"ds:source:{sid}": {"lthash": tampered[sid][0].hex()}})
        assert verdict is (pkg.Verdict.DIGEST_MISMATCH if sid == victim else pkg.Verdict.OK)


def test_sign_and_verify_gpu_digests_end_to_end(pkg):
    """Config 5's last step: digest on the GPU, sign and verify on the host."""
    import random

    rng = random.Random(3)
    model = pkg.TensorMap([(f"l{i}", rng.randbytes(rng.randint(1, 30000))) for i in range(5)])
    cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE)
    res = pkg.hash_model(cfg, model)
    key = pkg.keygen()
    stmt = pkg.Statement([pkg.Subject("m", {cfg.alg.value: res.digest_hex()})],
                         pkg.attestation.MODEL_PREDICATE_TYPE, cfg.predicate())
    bundle = pkg.sign_bundle(stmt, key)
    replay = pkg.HashConfig.from_predicate(bundle.statement().predicate)
    again = pkg.hash_model(replay, model)
    assert pkg.verify_bundle(bundle, {"m": {cfg.alg.value: again.digest_hex()}}) is pkg.Verdict.OK
    tampered = pkg.TensorMap([(n, (b[:-1] + bytes([b[-1] ^ 1])) if n == "l2" else b) for n, b in model.entries])
    bad = pkg.hash_model(replay, tampered)
    assert pkg.verify_bundle(bundle, {"m": {cfg.alg.value: bad.digest_hex()}}) is pkg.Verdict.DIGEST_MISMATCH


# ---- streaming loader hook, CUDA-graph replay --------------------------------------------------

def test_streaming_hasher_equals_whole_dataset_pass(pkg, porc):
    """Batches of a [N, 3, 8, 8] uint8 tensor in shuffled order == one pass == the oracle."""
    from paper_2510_00554_b200 import dataset as dsm

    n, n_src = 1000, 7
    rng = np.random.default_rng(5)
    data = rng.integers(0, 256, size=(n, 3, 8, 8), dtype=np.uint8)
    ids = rng.permutation(n).astype(np.int64) + 10_000
    declared = [3, 4, 8, 15, 16, 23, 42]
    src = np.array(declared)[rng.integers(0, n_src, size=n)]
    want = porc.dataset_digests([(int(ids[i]), int(src[i]), b"", data[i].tobytes()) for i in range(n)],
                                declared=declared)
    order = rng.permutation(n)
    for batch in (1, 128, 333):
        h = dsm.StreamingDatasetHasher(declared)
        dev_data = torch.from_numpy(data).cuda()
        for s in range(0, n, batch):
            idx = order[s:s + batch]
            rows = dev_data[torch.from_numpy(idx).cuda()] if batch != 128 else torch.from_numpy(data[idx])  # CUDA and host batches
            h.update(rows, torch.from_numpy(ids[idx]), torch.from_numpy(src[idx]))
        got = h.finalize()
        assert {k: (v[0].data, v[1]) for k, v in got.items()} == {k: (v[0], v[1]) for k, v in want.items()}


def test_streaming_hasher_flags_undeclared_source(pkg):
    from paper_2510_00554_b200 import dataset as dsm
    from paper_2510_00554_b200.errors import ValidationError

    h = dsm.StreamingDatasetHasher([1, 2])
    h.update(torch.zeros(4, 16, dtype=torch.float32), torch.arange(4), torch.tensor([1, 2, 5, 1]))
    with pytest.raises(ValidationError):
        h.finalize()


def test_graph_replay_rehashes_current_bytes(pkg, porc):
    from paper_2510_00554_b200 import device as dev

    tensors = inputs.model_tensors(77, [8192 * 300 + 5, 100, 8192 * 64, 0, 70001])
    dts = [dev.as_device_bytes(t) for t in tensors]
    plan = dev.ModelPlan(dts, 8192)
    hasher = dev.MerkleModelHasher(plan, "sha256")
    graph = hasher.capture()
    graph.replay()
    assert hasher.out_bytes() == porc.inplace_merkle("sha256", tensors, 8192)
    dts[0][12345] ^= 0x40                                   # the model changes in place ...
    changed = [bytes(dts[0].cpu().numpy().tobytes())] + tensors[1:]
    graph.replay()                                          # ... and the same graph hashes the new bytes
    assert hasher.out_bytes() == porc.inplace_merkle("sha256", changed, 8192)


def test_memory_accounting_trend(pkg):
    """The reference's acceptance criterion 8 (tests/test_acceptance.py:260-275): the coalesced strategy pays one
    padded copy of the model, per-layer and in-place stay below 2 % of the model size."""
    from paper_2510_00554_b200 import bench as sbench
    from paper_2510_00554_b200.model import coalesce_hash, inplace_hash, per_layer_hash

    model = sbench.synthetic_model("bert", scale=0.125, seed=8)            # ~67 MiB, 199 layers
    total = model.total_bytes
    assert total >= 64 << 20
    cfg = lambda strat: pkg.HashConfig(pkg.Construction.MERKLE, strat, pkg.CompressionAlg.SHA256)
    co = coalesce_hash(cfg(pkg.Strategy.COALESCED), model)
    bs = co.config.block_size
    assert co.aux_data_bytes == -(-total // bs) * bs
    pl = per_layer_hash(cfg(pkg.Strategy.PER_LAYER), model)
    ip = inplace_hash(cfg(pkg.Strategy.IN_PLACE), model)
    assert ip.aux_data_bytes == 0 and pl.aux_data_bytes == 0
    assert pl.aux_bytes <= 0.02 * total and ip.aux_bytes <= 0.02 * total
    assert len(pl.layer_digests) == 199 and ip.layer_digests is None


def test_length_sorted_rows_give_the_same_digests(pkg, corc):
    from paper_2510_00554_b200 import dataset as dsm, device as dev

    rng = np.random.default_rng(31)
    n, n_src = 5000, 5
    lens = rng.integers(0, 1500, size=n).astype(np.uint64)
    offs = np.zeros(n, dtype=np.uint64)
    np.cumsum(lens[:-1], out=offs[1:])
    shard = rng.integers(0, 256, size=int(lens.sum()) + 16, dtype=np.uint8)
    ids = rng.permutation(n).astype(np.uint64)
    src = rng.integers(0, n_src, size=n)
    ds = dsm.DeviceDataset.from_host(shard, offs, lens, ids, src, list(range(n_src)))
    outs = []
    for d in (ds, ds.sorted_by_length()):
        acc = dev.LatticeAccumulator(n_src)
        d.accumulate(acc)
        outs.append(acc.digests())
    assert outs[0] == outs[1]
    assert bool((ds.sorted_by_length().lengths[1:] >= ds.sorted_by_length().lengths[:-1]).all())


def test_gather_spans_any_alignment(pkg):
    """snt_gather_spans against numpy: every source/destination byte phase, zero padding, empty spans, >1 chunk."""
    from paper_2510_00554_b200 import device as dev

    rng = np.random.default_rng(99)
    pool = torch.from_numpy(rng.integers(1, 256, size=6 << 20, dtype=np.uint8)).cuda()
    host = pool.cpu().numpy()
    for pad_block in (0, 64, 8192):
        lens, src_off, dst_off, pos = [], [], [], 0
        for k in range(200):
            n = int(rng.choice([0, 1, 3, 15, 16, 17, 255, 4096, 8191, 8192, 40000, 70001, 300000][: 13 if k % 7 else 11]))
            so = int(rng.integers(0, host.size - n - 1))
            so = so - so % 16 + (k % 16)                       # every source phase
            pos += (k * 5) % 16 if pad_block == 0 else 0       # every destination phase (packed layout only)
            padded = n if not pad_block else -(-n // pad_block) * pad_block
            if pad_block:
                pos = -(-pos // pad_block) * pad_block
            lens.append(n); src_off.append(so); dst_off.append(pos)
            pos += padded
        dst = torch.full((pos + 64,), 0xEE, dtype=torch.uint8, device="cuda")
        dev.gather_spans(np.uint64(pool.data_ptr()) + np.array(src_off, dtype=np.uint64), np.array(lens, dtype=np.uint64),
                         np.array(dst_off, dtype=np.uint64), pad_block, dst)
        got = dst.cpu().numpy()
        want = np.full(pos + 64, 0xEE, dtype=np.uint8)
        for n, so, do in zip(lens, src_off, dst_off):
            padded = n if not pad_block else -(-n // pad_block) * pad_block
            want[do:do + n] = host[so:so + n]
            want[do + n:do + padded] = 0
        assert np.array_equal(got, want), pad_block


def test_hash_model_from_several_threads(pkg, porc):
    """The hashing entry points are callable from any number of threads: resident models,
    staged host models (which take turns on the pinned ring) and datasets at the same time."""
    import threading

    from paper_2510_00554_b200 import device as dv

    rng = np.random.default_rng(77)
    host = [rng.integers(0, 256, size=s, dtype=np.uint8) for s in ((9 << 20) + 5, 8192 * 700, 333, (12 << 20), 4096 * 3)]
    want = {a: porc.inplace_merkle(a, [h.tobytes() for h in host], 8192) for a in ALGS}
    as_bytes = pkg.TensorMap([(f"t{i}", h.tobytes()) for i, h in enumerate(host)])
    on_gpu = pkg.TensorMap([(f"t{i}", torch.from_numpy(h).cuda()) for i, h in enumerate(host)])
    errors = []

    def work(k):
        try:
            for rep in range(3):
                alg = ALGS[(k + rep) % 3]
                cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, _alg(pkg, alg))
                model = as_bytes if (k + rep) % 2 else on_gpu
                got = pkg.hash_model(cfg, model, workers=2).model_digest.data
                if got != want[alg]:
                    errors.append((k, rep, alg))
        except Exception as exc:          # noqa: BLE001
            errors.append((k, repr(exc)))

    threads = [threading.Thread(target=work, args=(k,)) for k in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(120)
    assert not any(t.is_alive() for t in threads), "a hashing thread is stuck"
    assert errors == []


def test_tensor_larger_than_4_gib(pkg, corc):
    """Byte offsets past 2^32 inside one tensor and past 2^33 in the model: root, every leaf digest of the far
    end, lattice digest -- against the C oracle on the same bytes (maximum-size edge of model.py:137-146)."""
    import os

    from paper_2510_00554_b200 import device as dev

    big = (4 << 30) + 8192 * 3 + 1234                      # one tensor > 4 GiB with a ragged tail
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    parts = [torch.randint(0, 256, (big,), dtype=torch.uint8, device="cuda", generator=gen),
             torch.randint(0, 256, (12345,), dtype=torch.uint8, device="cuda", generator=gen),
             torch.randint(0, 256, ((1 << 30) + 64,), dtype=torch.uint8, device="cuda", generator=gen)]
    host = [p.cpu().numpy() for p in parts]
    tl = corc.TensorList(host)
    threads = os.cpu_count() or 4
    n_leaves = tl.leaf_count(8192)
    assert n_leaves > (1 << 19) and sum(h.size for h in host) > 5 * (1 << 30)
    plan = dev.ModelPlan(parts, 8192)
    for alg in ("sha256", "blake2b"):
        hasher = dev.MerkleModelHasher(plan, alg)
        hasher.run()
        want_leaves = corc.inplace_leaves(alg, tl, 8192, threads)
        assert hasher.leaf_bytes() == want_leaves, alg            # every one of the ~655k leaf digests
        assert hasher.out_bytes() == corc.inplace_merkle(alg, tl, 8192, threads), alg
    lat = pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.BLAKE2B)
    got = pkg.hash_model(lat, pkg.TensorMap([(f"t{i}", p) for i, p in enumerate(parts)]))
    assert got.model_digest.data == corc.inplace_lattice(tl, 8192, threads)


@pytest.mark.parametrize("cover_labels", [False, True])
def test_digest_dataset_large_shard_file_with_gaps_and_labels(pkg, porc, tmp_path, cover_labels):
    """digest_dataset on a shard FILE above the direct-copy threshold (read by the staging threads into the pinned
    ring), rows in shuffled order with gaps between samples, empty samples, labels of 0-11 bytes laid out by the
    device gather; every per-source digest and count against the oracle (dataset.py:41-49, :166-195)."""
    rng = np.random.default_rng(11)
    n, n_src = 6000, 7
    lens = rng.integers(0, 4200, size=n)
    lens[rng.integers(0, n, size=40)] = 0
    gaps = rng.integers(0, 9, size=n)
    offs = np.cumsum(lens + gaps) - lens
    shard = rng.integers(0, 256, size=int(offs[-1] + lens[-1]) + 5, dtype=np.uint8).tobytes()
    assert len(shard) > (8 << 20)
    labels = [bytes(rng.integers(97, 123, size=int(k), dtype=np.uint8)) for k in rng.integers(0, 12, size=n)]
    ids = rng.integers(0, 1 << 63, size=n, dtype=np.uint64) * 2 + rng.integers(0, 2, size=n, dtype=np.uint64)
    src = rng.integers(10, 10 + n_src, size=n)
    order = rng.permutation(n)
    rows = [(int(ids[i]), int(src[i]), labels[i], int(offs[i]), int(lens[i])) for i in order]
    man = pkg.DatasetManifest(rows, tmp_path / "big.bin")
    (tmp_path / "big.bin").write_bytes(shard)
    want = porc.dataset_digests(((sid, s, lab, shard[o:o + ln]) for sid, s, lab, o, ln in rows), cover_labels=cover_labels)
    got = pkg.digest_dataset(man, cover_labels=cover_labels)
    assert {k: (d.data, c) for k, (d, c) in got.items()} == want
    # a row that runs past the end of the file is a FormatError, as in the reference
    bad = pkg.DatasetManifest(rows + [(1, 10, b"", len(shard) - 3, 4)], tmp_path / "big.bin")
    with pytest.raises(pkg.errors.FormatError):
        pkg.digest_dataset(bad, cover_labels=cover_labels)
    with pytest.raises(pkg.errors.FormatError):
        pkg.digest_dataset(pkg.DatasetManifest(rows, tmp_path / "missing.bin"))


def test_process_batch_helper_and_python_packer_agree(pkg):
    """process_batch through the C packer (_hostpack.pack_records) and through the Python packer: same sums, and the
    same errors in the same order (undeclared source before a bad id)."""
    from paper_2510_00554_b200 import device as dev

    rng = np.random.default_rng(5)
    recs = [pkg.SampleRecord(int(rng.integers(0, 1 << 62)), int(rng.integers(0, 40)), b"L%d" % (i % 3),
                             bytes(rng.integers(0, 256, size=int(rng.integers(0, 700)), dtype=np.uint8))) for i in range(1000)]
    assert dev._hostpack is not None, "the packing helper must be built in-tree (build.build_hostpack)"

    def run(cover):
        acc = pkg.SourceAccumulator(cover_labels=cover)
        for s in range(0, len(recs), 128):
            pkg.process_batch(pkg.Batch(recs[s:s + 128]), acc)
        return {k: (d.data, c) for k, (d, c) in pkg.finalize(acc).items()}

    helper = dev._hostpack
    try:
        for cover in (False, True):
            with_c = run(cover)
            dev._hostpack = None
            assert run(cover) == with_c
            dev._hostpack = helper
        for packer in (helper, None):
            dev._hostpack = packer
            acc = pkg.SourceAccumulator()
            acc.declare([1])
            with pytest.raises(pkg.errors.ValidationError, match="undeclared source 9"):
                pkg.process_batch(pkg.Batch([pkg.SampleRecord(-5, 1, b"", b"x"), pkg.SampleRecord(3, 9, b"", b"y")]), acc)
            with pytest.raises(pkg.errors.ValidationError, match="64-bit"):
                pkg.process_batch(pkg.Batch([pkg.SampleRecord(1 << 64, 1, b"", b"x")]), acc)
    finally:
        dev._hostpack = helper


def test_loaded_checkpoint_file_hashes_like_its_bytes(pkg, porc, tmp_path):
    """load_model hands out lazy views of the data file (FileTensor): the in-place path preads them straight into
    the pinned ring, every other strategy reads the file once; all seven configurations must equal the hash of the
    same tensors held as bytes, and the in-place Merkle root the oracle's (model.py:298-315, :335-352)."""
    import random

    rng = random.Random(77)
    sizes = [100, 8192, 0, 5000, (29 << 20) + 13, 3, 40 * 8192, (5 << 20)]      # above the pipelined path's threshold
    host = [rng.randbytes(s) for s in sizes]
    tm = pkg.TensorMap([(f"t{i}", h) for i, h in enumerate(host)])
    pkg.save_model(tm, tmp_path / "ckpt.json")
    C, S, A = pkg.Construction, pkg.Strategy, pkg.CompressionAlg
    for cons, strat, alg, ordered in [(C.MERKLE, S.IN_PLACE, A.SHA256, False), (C.MERKLE, S.IN_PLACE, A.SHA3_256, False),
                                      (C.MERKLE, S.PER_LAYER, A.BLAKE2B, False), (C.MERKLE, S.COALESCED, A.SHA256, False),
                                      (C.LATTICE, S.IN_PLACE, A.BLAKE2B, False), (C.LATTICE, S.PER_LAYER, A.BLAKE2B, True),
                                      (C.LATTICE, S.COALESCED, A.BLAKE2B, False)]:
        cfg = pkg.HashConfig(cons, strat, alg, 8192, ordered)
        loaded = pkg.load_model(tmp_path / "ckpt.json")          # fresh: nothing materialised yet
        got, want = pkg.hash_model(cfg, loaded), pkg.hash_model(cfg, tm)
        assert got.model_digest.data == want.model_digest.data, (cons, strat, alg)
        assert got.block_count == want.block_count
        if want.layer_digests is not None:
            assert {k: d.data for k, d in got.layer_digests.items()} == {k: d.data for k, d in want.layer_digests.items()}
        if cons is C.MERKLE and strat is S.IN_PLACE:
            assert got.model_digest.data == porc.inplace_merkle(alg.value, host, 8192)
            assert loaded.entries[4][1].file._whole is None      # the file was never copied into host memory
    # a file-backed tensor mixed with bytes, a numpy array and a CUDA tensor in one model
    import torch

    loaded = pkg.load_model(tmp_path / "ckpt.json")
    mixed = pkg.TensorMap([("a", loaded.entries[4][1]), ("b", host[1]), ("c", np.frombuffer(host[6], dtype=np.uint8)),
                           ("d", torch.frombuffer(bytearray(host[7]), dtype=torch.uint8).cuda()), ("e", loaded.entries[3][1])])
    cfg = pkg.HashConfig(C.MERKLE, S.IN_PLACE, A.SHA256, 8192)
    assert pkg.hash_model(cfg, mixed).model_digest.data == porc.inplace_merkle("sha256", [host[4], host[1], host[6], host[7], host[3]], 8192)
