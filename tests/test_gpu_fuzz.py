"""Randomised parity: models and datasets drawn at random (sizes, alignments, where the bytes live, block size,
algorithm, construction, schedule), hashed through the public API and compared with the C oracle. Every case is a
function of its seed, printed on failure. The default budget is a few seconds; SNT_FUZZ_SECONDS=600 makes it a soak.
"""

import os
import time

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ALGS = ("sha256", "blake2b", "sha3-256")
BUDGET = float(os.environ.get("SNT_FUZZ_SECONDS", "12"))


@pytest.fixture(scope="module")
def pkg():
    import paper_2510_00554_b200 as pkg
    from paper_2510_00554_b200 import _native

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    _native.load()
    return pkg


def _random_sizes(rng, n, big):
    kinds = rng.integers(0, 6, size=n)
    out = []
    for k in kinds:
        if k == 0:
            out.append(0)
        elif k == 1:
            out.append(int(rng.integers(1, 300)))
        elif k == 2:
            out.append(int(rng.integers(1, 40)) * 8192)                       # whole blocks
        elif k == 3:
            out.append(int(rng.integers(1, 40)) * 8192 + int(rng.integers(1, 8192)))
        elif k == 4:
            out.append(int(rng.integers(60_000, 70_000)))                     # around the small-tensor threshold
        else:
            out.append(int(rng.integers(1, big)))
    return out


def test_random_models_against_the_c_oracle(pkg, corc, monkeypatch):
    from paper_2510_00554_b200 import _native, device as dv, model as mm

    lib = _native.load()
    deadline = time.monotonic() + BUDGET
    seed0 = int(os.environ.get("SNT_FUZZ_SEED", "1000"))
    case = 0
    try:
        while time.monotonic() < deadline or case < 3:
            seed = seed0 + case
            case += 1
            rng = np.random.default_rng(seed)
            n = int(rng.integers(1, 24))
            host_mode = int(rng.integers(0, 4))            # 0 all CUDA, 1 all pinned, 2 pageable mix, 3 everything mixed
            big = int(rng.choice([20_000, 3 << 20, 12 << 20])) if host_mode else int(rng.choice([20_000, 1 << 20]))
            sizes = _random_sizes(rng, n, big)
            if sum(sizes) == 0:
                sizes[0] = 77
            arena = rng.integers(0, 256, size=sum(sizes) + 64 * n + 64, dtype=np.uint8)
            host, entries, pos, base_cuda = [], [], 0, None
            for i, s in enumerate(sizes):
                pos += int(rng.integers(0, 17)) if rng.random() < 0.3 else 0     # odd addresses now and then
                h = arena[pos:pos + s]
                pos += s
                host.append(h)
                where = {0: 0, 1: 1, 2: int(rng.integers(2, 5)), 3: int(rng.integers(0, 5))}[host_mode]
                if where == 0:
                    if base_cuda is None:
                        base_cuda = torch.from_numpy(arena).cuda()                          # views into ONE device buffer
                    entries.append((f"t{i}", base_cuda[pos - s:pos]))
                elif where == 1:
                    entries.append((f"t{i}", torch.from_numpy(h.copy()).pin_memory()))
                elif where == 2:
                    entries.append((f"t{i}", h.tobytes()))
                elif where == 3:
                    entries.append((f"t{i}", h))                                           # numpy view, any alignment
                else:
                    entries.append((f"t{i}", torch.from_numpy(h.copy())))
            bs = int(rng.choice([64, 1024, 8192, 8192, 1 << 16]))
            alg = ALGS[int(rng.integers(0, 3))]
            lattice = rng.random() < 0.25
            schedule = int(rng.integers(0, 3))
            # small staging parameters so that rings wrap and pieces split at test sizes
            monkeypatch.setattr(mm, "STAGE_PIPELINE_MIN_BYTES", int(rng.choice([1 << 16, 32 << 20])))
            monkeypatch.setattr(mm, "STAGE_CHUNK_BYTES", int(rng.choice([1 << 20, 3 << 20, 256 << 20])))
            monkeypatch.setattr(mm, "STAGE_PIECE_BYTES", int(rng.choice([1 << 19, 1 << 20, 64 << 20])))
            monkeypatch.setattr(dv, "STAGE_SLOT_BYTES", int(rng.choice([1 << 20, 32 << 20])))
            monkeypatch.setattr(dv, "STAGE_PIECE_BYTES", int(rng.choice([1 << 18, 4 << 20])))
            lib.snt_merkle_schedule(schedule)
            tl = corc.TensorList(host)
            what = (seed, sizes, host_mode, bs, alg, lattice, schedule)
            model = pkg.TensorMap(entries)
            if lattice:
                cfg = pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.BLAKE2B, bs)
                want = corc.inplace_lattice(tl, bs, 4)
            else:
                cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.from_name(alg), bs)
                want = corc.inplace_merkle(alg, tl, bs, 4)
            for _ in range(2):                                                              # the second call may hit the cache
                res = pkg.hash_model(cfg, model)
                assert res.model_digest.data == want, what
                assert res.block_count == tl.leaf_count(bs), what
    finally:
        lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT)
    print(f"{case} random models")


def test_random_datasets_against_the_c_oracle(pkg, corc):
    from paper_2510_00554_b200 import _native, dataset as dsm, device as dev

    lib = _native.load()
    deadline = time.monotonic() + BUDGET
    seed0 = int(os.environ.get("SNT_FUZZ_SEED", "5000"))
    case = 0
    try:
        while time.monotonic() < deadline or case < 3:
            seed = seed0 + case
            case += 1
            rng = np.random.default_rng(seed)
            n = int(rng.choice([1, 7, 33, 500, 5000, 40_000]))
            shape = int(rng.integers(0, 4))
            if shape == 0:
                lens = np.full(n, int(rng.choice([0, 8, 120, 128, 3072])), dtype=np.uint64)        # one length
            elif shape == 1:
                lens = (rng.integers(4, 260, size=n) * 4).astype(np.uint64)                          # token arrays
            elif shape == 2:
                lens = rng.integers(0, 700, size=n).astype(np.uint64)
            else:
                lens = rng.choice(np.array([0, 1, 119, 120, 121, 127, 128, 129, 248, 256, 9000], dtype=np.uint64), size=n)
            gap = int(rng.choice([0, 0, 1, 3, 4, 8]))
            offs = np.zeros(n, dtype=np.uint64)
            if n > 1:
                np.cumsum(lens[:-1] + np.uint64(gap), out=offs[1:])
            shard = rng.integers(0, 256, size=int(offs[-1] + lens[-1]) + 16, dtype=np.uint8)
            n_src = int(rng.choice([1, 3, 16, 129, 300]))
            src = rng.integers(0, n_src, size=n)
            ids = rng.integers(0, 2**63, size=n).astype(np.uint64)
            schedule = int(rng.integers(0, 3))
            lib.snt_merkle_schedule(schedule)
            what = (seed, n, shape, gap, n_src, schedule)
            want_sums, want_counts = corc.lthash_samples(shard, offs, lens, ids, src.astype(np.uint32), n_src, 4)
            ds = dsm.DeviceDataset.from_host(shard, offs, lens, ids, src, list(range(n_src)))
            if rng.random() < 0.3:
                ds.uniform = None                                                                    # "not known": lanes
            acc = dev.LatticeAccumulator(n_src)
            a = int(rng.integers(0, n))
            ds.accumulate(acc, 0, a)                                                                 # two launches: ranges add up
            ds.accumulate(acc, a, n)
            out, counts, status = acc.digests()
            assert (status, counts) == (0, list(want_counts)), what
            assert out == want_sums, what
    finally:
        lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT)
    print(f"{case} random datasets")


def test_random_models_per_layer_and_coalesced_against_the_python_oracle(pkg, porc):
    """The strategies that move data before hashing: per-layer digests + model digest and the
    coalesced digest, both constructions, on small random models whose tensors live on the GPU or on the host."""
    deadline = time.monotonic() + BUDGET
    seed0 = int(os.environ.get("SNT_FUZZ_SEED", "9000"))
    case = 0
    while time.monotonic() < deadline or case < 3:
        seed = seed0 + case
        case += 1
        rng = np.random.default_rng(seed)
        n = int(rng.integers(1, 12))
        bs = int(rng.choice([64, 256, 1024]))
        sizes = [int(rng.choice([0, 1, bs - 1, bs, bs + 1, 3 * bs, int(rng.integers(1, 20 * bs))])) for _ in range(n)]
        if sum(sizes) == 0:
            sizes[0] = 5
        host = [rng.integers(0, 256, size=s, dtype=np.uint8).tobytes() for s in sizes]
        on_gpu = rng.random() < 0.5
        entries = [(f"l{i}", torch.frombuffer(bytearray(h), dtype=torch.uint8).cuda() if (on_gpu and h) else h)
                   for i, h in enumerate(host)]
        model = pkg.TensorMap(entries)
        alg = ALGS[int(rng.integers(0, 3))]
        what = (seed, sizes, bs, alg, on_gpu)
        m_cfg = lambda strat: pkg.HashConfig(pkg.Construction.MERKLE, strat, pkg.CompressionAlg.from_name(alg), bs)   # noqa: E731
        l_cfg = lambda strat: pkg.HashConfig(pkg.Construction.LATTICE, strat, pkg.CompressionAlg.BLAKE2B, bs)          # noqa: E731
        root, layers = porc.per_layer_merkle(alg, host, bs)
        res = pkg.hash_model(m_cfg(pkg.Strategy.PER_LAYER), model)
        assert res.model_digest.data == root and [d.data for d in res.layer_digests.values()] == layers, what
        root, layers = porc.per_layer_lattice(host, bs)
        res = pkg.hash_model(l_cfg(pkg.Strategy.PER_LAYER), model)
        assert res.model_digest.data == root and [d.data for d in res.layer_digests.values()] == layers, what
        assert pkg.hash_model(m_cfg(pkg.Strategy.COALESCED), model).model_digest.data == porc.coalesced_merkle(alg, host, bs), what
        assert pkg.hash_model(l_cfg(pkg.Strategy.COALESCED), model).model_digest.data == porc.coalesced_lattice(host, bs), what
    print(f"{case} random models x 4 strategy/construction pairs")


def test_random_host_object_calls_against_the_python_oracle(pkg, porc, tmp_path):
    """The reference-shaped calls on Python objects and files (session 4: C packers, file -> pinned ring, lazy
    checkpoint views): hash_blocks on mixed bytes-like blocks, process_batch on random batches, digest_dataset on
    a manifest + shard file, load_model + hash_model on a checkpoint file -- against the hashlib oracle."""
    deadline = time.monotonic() + BUDGET
    seed0 = int(os.environ.get("SNT_FUZZ_SEED", "13000"))
    case = 0
    C, S = pkg.Construction, pkg.Strategy
    while time.monotonic() < deadline or case < 3:
        seed = seed0 + case
        case += 1
        rng = np.random.default_rng(seed)

        def blob(n):
            return rng.integers(0, 256, size=int(n), dtype=np.uint8).tobytes()

        def dressed(b):                                   # the same bytes as another bytes-like type
            k = int(rng.integers(0, 4))
            return b if k == 0 else bytearray(b) if k == 1 else memoryview(b) if k == 2 else np.frombuffer(b, dtype=np.uint8)

        # ---- hash_blocks + merkle_root over a list of blocks (total below or above the threaded / streaming threshold)
        alg = ALGS[int(rng.integers(0, 3))]
        n_blocks = int(rng.choice([1, 2, 9, 300, 1500]))
        big = int(rng.choice([700, 9000]))
        blocks = [blob(rng.integers(0, big)) for _ in range(n_blocks)]
        leaves = pkg.hash_blocks(pkg.CompressionAlg.from_name(alg), [dressed(b) for b in blocks])
        assert bytes(leaves.data) == bytes(porc.hash_blocks(alg, blocks)), ("hash_blocks", seed)
        assert pkg.merkle_root(pkg.CompressionAlg.from_name(alg), leaves).data == \
            porc.merkle_root(alg, bytes(leaves.data), n_blocks), ("merkle_root", seed)

        # ---- process_batch over random batches, and digest_dataset over the same samples as a manifest + shard file
        n = int(rng.choice([1, 40, 700, 3000]))
        n_src = int(rng.choice([1, 5, 40]))
        cover = bool(rng.integers(0, 2))
        lens = rng.integers(0, int(rng.choice([40, 700, 4000])), size=n)
        gaps = rng.integers(0, 5, size=n)
        offs = np.cumsum(lens + gaps) - lens
        shard = blob(int(offs[-1] + lens[-1]) + 3)
        ids = rng.integers(0, 1 << 63, size=n, dtype=np.uint64) * 2 + rng.integers(0, 2, size=n, dtype=np.uint64)
        src = rng.integers(0, n_src, size=n)
        labels = [blob(k) for k in rng.integers(0, 9, size=n)]
        samples = [(int(ids[i]), int(src[i]), labels[i], shard[int(offs[i]):int(offs[i] + lens[i])]) for i in range(n)]
        want = porc.dataset_digests(samples, cover_labels=cover)
        acc = pkg.SourceAccumulator(cover_labels=cover)
        order = rng.permutation(n)
        bs = int(rng.choice([1, 7, 128, 1000]))
        for s in range(0, n, bs):
            recs = [pkg.SampleRecord(samples[i][0], samples[i][1], samples[i][2], dressed(samples[i][3]) if i % 5 == 0 else samples[i][3])
                    for i in order[s:s + bs]]
            pkg.process_batch(pkg.Batch(recs), acc)
        assert {k: (d.data, c) for k, (d, c) in pkg.finalize(acc).items()} == want, ("process_batch", seed, cover)
        rows = [(samples[i][0], samples[i][1], labels[i], int(offs[i]), int(lens[i])) for i in order]
        (tmp_path / "shard.bin").write_bytes(shard)
        man = pkg.DatasetManifest(rows, tmp_path / "shard.bin")
        got = pkg.digest_dataset(man, cover_labels=cover)
        assert {k: (d.data, c) for k, (d, c) in got.items()} == want, ("digest_dataset", seed, cover)

        # ---- a checkpoint file through load_model (lazy file views), one random configuration
        sizes = _random_sizes(rng, int(rng.integers(1, 12)), int(rng.choice([20_000, 6 << 20, 40 << 20])))
        if sum(sizes) == 0:
            sizes[0] = 17
        host = [blob(s) for s in sizes]
        pkg.save_model(pkg.TensorMap([(f"t{i}", h) for i, h in enumerate(host)]), tmp_path / "ckpt.json")
        loaded = pkg.load_model(tmp_path / "ckpt.json")
        pick = int(rng.integers(0, 4))
        if pick == 0:
            cfg = pkg.HashConfig(C.MERKLE, S.IN_PLACE, pkg.CompressionAlg.from_name(alg), 8192)
            assert pkg.hash_model(cfg, loaded).model_digest.data == porc.inplace_merkle(alg, host, 8192), ("ckpt merkle", seed)
        elif pick == 1:
            cfg = pkg.HashConfig(C.LATTICE, S.IN_PLACE, pkg.CompressionAlg.BLAKE2B, 8192)
            assert pkg.hash_model(cfg, loaded).model_digest.data == porc.inplace_lattice(host, 8192), ("ckpt lattice", seed)
        elif pick == 2:
            cfg = pkg.HashConfig(C.MERKLE, S.COALESCED, pkg.CompressionAlg.from_name(alg), 8192)
            assert pkg.hash_model(cfg, loaded).model_digest.data == porc.coalesced_merkle(alg, host, 8192), ("ckpt coalesced", seed)
        else:
            cfg = pkg.HashConfig(C.MERKLE, S.PER_LAYER, pkg.CompressionAlg.from_name(alg), 8192)
            root, layers = porc.per_layer_merkle(alg, host, 8192)
            res = pkg.hash_model(cfg, loaded)
            assert res.model_digest.data == root and [d.data for d in res.layer_digests.values()] == list(layers), ("ckpt per-layer", seed)
        del loaded
    print(f"{case} random host-object cases")
