"""GPU parity of the persistent kernel (csrc/merkle_fused.cuh) under all three schedules of
``snt_merkle_schedule``: PERSISTENT (time-sliced leaf chains, then the level-reducer launches -- the default),
FUSED (the tree folded into the same launch through completion counters) and GRID (round 1's one thread per
leaf grid).

Every case is checked bit-exact against the C oracle (leaf digests and root), the three schedules against each
other, and the fused launch against itself on repeated launches over the same workspace (the kernel must hand
every completion counter back at zero).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ALGS = ["sha256", "blake2b", "sha3-256"]


@pytest.fixture(scope="module")
def dev():
    from paper_2510_00554_b200 import _native, device

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    _native.load()
    return device


def _ragged_model(seed, n_tensors, max_bytes, arena_bytes, odd_addresses=True):
    """Tensors carved out of one device arena at arbitrary byte offsets: ragged tails, empty tensors,
    tensors smaller than a block, unaligned addresses. Returns (device views, host arrays)."""
    rng = np.random.default_rng(seed)
    host_arena = rng.integers(0, 256, size=arena_bytes, dtype=np.uint8)
    arena = torch.from_numpy(host_arena).cuda()
    views, host, pos = [], [], 0
    for i in range(n_tensors):
        kind = rng.integers(0, 6)
        if kind == 0:
            size = 0
        elif kind == 1:
            size = int(rng.integers(1, 300))
        elif kind == 2:
            size = int(rng.integers(1, 8)) * 8192                       # whole blocks
        else:
            size = int(rng.integers(1, max_bytes))
        align = 1 if (odd_addresses and rng.integers(0, 3) == 0) else 16
        pos = -(-pos // align) * align + (int(rng.integers(1, 16)) if align == 1 else 0)
        if pos + size > arena_bytes:
            break
        views.append(arena[pos:pos + size])
        host.append(host_arena[pos:pos + size])
        pos += size
    return views, host


def _both_paths(dev, plan, alg, begin=0, end=None, levels=None):
    """(leaf digests, output) under every schedule; asserts they agree. Returns the pair and the number of
    launches the fused schedule took."""
    from paper_2510_00554_b200 import _native

    lib = _native.load()
    results = {}
    fused_launches = None
    try:
        for schedule in (_native.SCHEDULE_FUSED, _native.SCHEDULE_PERSISTENT, _native.SCHEDULE_GRID):
            lib.snt_merkle_schedule(schedule)
            hasher = dev.MerkleModelHasher(plan, alg, begin, end, levels)
            launches = lib.snt_debug_launch_count()
            hasher.run()
            if schedule == _native.SCHEDULE_FUSED:
                fused_launches = lib.snt_debug_launch_count() - launches
            results[schedule] = (hasher.leaf_bytes(), hasher.out_bytes())
            if schedule == _native.SCHEDULE_FUSED:
                for _ in range(2):                           # counters are back at zero: same answer again
                    hasher.leaves.zero_()
                    hasher.out.zero_()
                    hasher.run()
                    assert (hasher.leaf_bytes(), hasher.out_bytes()) == results[schedule]
    finally:
        lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT)
    got = results[_native.SCHEDULE_FUSED]
    for schedule, other in results.items():
        assert got[0] == other[0], f"leaf digests differ between the fused schedule and schedule {schedule}"
        assert got[1] == other[1], f"tree output differs between the fused schedule and schedule {schedule}"
    return got, fused_launches


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("block_size", [64, 1024, 8192])
def test_ragged_models_fused_vs_oracle(dev, corc, alg, block_size):
    budget = {64: 3 << 20, 1024: 24 << 20, 8192: 96 << 20}[block_size]
    views, host = _ragged_model(100 + block_size, 400, max(budget // 40, 4096), budget)
    plan = dev.ModelPlan(views, block_size)
    (leaves, root), launches = _both_paths(dev, plan, alg)
    tl = corc.TensorList(host)
    threads = corc.threads_default()
    want_leaves = corc.inplace_leaves(alg, tl, block_size, threads)
    assert leaves == want_leaves
    assert root == corc.merkle_root(alg, want_leaves, plan.leaf_count, threads)
    assert launches == 1, "the fused schedule is one launch per hash"


@pytest.mark.parametrize("alg", ALGS)
def test_tree_shapes_around_group_boundaries(dev, corc, alg):
    """Leaf counts around every stage boundary (32-leaf chains, 256-leaf groups, 2^14-node stages) at a
    small block size: single ragged groups, one node past a full group, exact powers of two."""
    bs = 64
    counts = [32, 33, 255, 256, 257, 511, 513, 1000, 4096, 16383, 16384, 16385, 16384 + 257, 40000]
    rng = np.random.default_rng(7)
    for n in counts:
        data = rng.integers(0, 256, size=n * bs - int(rng.integers(0, bs)), dtype=np.uint8)
        views = [torch.from_numpy(data).cuda()]
        plan = dev.ModelPlan(views, bs)
        assert plan.leaf_count == n
        (leaves, root), _ = _both_paths(dev, plan, alg)
        tl = corc.TensorList([data])
        want_leaves = corc.inplace_leaves(alg, tl, bs, 4)
        assert leaves == want_leaves, n
        assert root == corc.merkle_root(alg, want_leaves, n, 4), n


@pytest.mark.parametrize("alg", ALGS)
def test_shard_ranges_forced_levels(dev, porc, alg):
    """levels = k over aligned leaf ranges (the multi-GPU shard rule) through the fused launch."""
    bs = 64
    n = 9000
    rng = np.random.default_rng(17)
    data = rng.integers(0, 256, size=n * bs - 5, dtype=np.uint8)
    plan = dev.ModelPlan([torch.from_numpy(data).cuda()], bs)
    host = data.tobytes()
    dl = porc.DIGEST_LEN[alg]
    all_leaves = b"".join(porc.h(alg, host[i * bs:(i + 1) * bs]) for i in range(n))
    for k in (5, 6, 8, 9, 10, 13):
        width = 1 << k
        ranges = [(0, n), (width, min(n, 3 * width)), ((n // width) * width, n)]
        for begin, end in ranges:
            if begin >= end:
                continue
            (leaves, out), _ = _both_paths(dev, plan, alg, begin, end, k)
            assert leaves == all_leaves[begin * dl:end * dl], (k, begin, end)
            assert out == porc.reduce_levels_forced(alg, all_leaves[begin * dl:end * dl], begin, end - begin, n, k), \
                (k, begin, end)


def test_time_sliced_tail_is_exercised(dev, corc):
    """More chains than worker warps on every SM with a remainder: the parked-state FIFO runs."""
    bs = 8192
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = sms * 32 * 17 + 32 * 5 + 3                      # 17 chains and a bit per SM
    rng = np.random.default_rng(23)
    data = torch.from_numpy(rng.integers(0, 256, size=n * bs - 100, dtype=np.uint8)).cuda()
    a, b, c = bs * 1000 + 64, bs * 1300 + 65, bs * 1600 + 80
    # ragged tails, one tensor at an odd address (~300 irregular SHA-256 leaves), the rest regular
    pieces = [data[:a], data[a:b], data[b:c], data[c:]]
    host = [p.cpu().numpy() for p in pieces]
    for alg in ALGS:
        plan = dev.ModelPlan(pieces, bs)
        (leaves, root), launches = _both_paths(dev, plan, alg)
        tl = corc.TensorList(host)
        threads = corc.threads_default()
        want_leaves = corc.inplace_leaves(alg, tl, bs, threads)
        assert leaves == want_leaves, alg
        assert root == corc.merkle_root(alg, want_leaves, plan.leaf_count, threads), alg
        assert launches == 1


def test_lthash_chain_kernel_matches_grid_and_oracle(dev, corc):
    """LtHash through the persistent chain kernel (time-sliced tail, parked BLAKE2b states) against the plain grid
    and the C oracle: ragged samples, every alignment, more chains than warps per SM, > 128 sources (global
    atomics), undeclared sources, per-sample digests."""
    from paper_2510_00554_b200 import _native

    lib = _native.load()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    rng = np.random.default_rng(41)
    for n, n_src, max_len in ((sms * 32 * 11 + 17, 16, 700), (5000, 200, 3000), (33, 3, 70000), (1, 1, 10)):
        lens = rng.integers(0, max_len, size=n).astype(np.uint64)
        if n > 100:
            lens[::97] = 0                                   # empty samples
            lens[5] = 4 * max_len                            # one chain much longer than its neighbours
        offs = np.zeros(n, dtype=np.uint64)
        np.cumsum(lens[:-1] + rng.integers(0, 3, size=n - 1).astype(np.uint64), out=offs[1:])   # gaps: odd addresses
        shard = rng.integers(0, 256, size=int(offs[-1] + lens[-1]) + 16, dtype=np.uint8)
        slots = rng.integers(0, n_src, size=n).astype(np.uint32)
        bad = rng.choice(n, size=min(3, n - 1), replace=False) if n > 1 else np.array([], dtype=np.int64)
        slots_bad = slots.copy()
        slots_bad[bad] = n_src + 5                           # undeclared sources: skipped and counted
        ids = rng.integers(0, 2**63, size=n).astype(np.uint64)
        d_shard = torch.from_numpy(shard).cuda()
        d_off, d_len, d_ids = (torch.from_numpy(a.view(np.int64)).cuda() for a in (offs, lens, ids))
        keep = np.ones(n, dtype=bool)
        keep[bad] = False
        want_sums, want_counts, want_dig = corc.lthash_samples(shard, offs[keep], lens[keep], ids[keep], slots[keep], n_src,
                                                              4, want_digests=True)
        results = {}
        try:
            for schedule in (_native.SCHEDULE_FUSED, _native.SCHEDULE_PERSISTENT, _native.SCHEDULE_GRID):   # chains forced, auto, grid
                lib.snt_merkle_schedule(schedule)
                acc = dev.LatticeAccumulator(n_src)
                dig = torch.zeros(n * 64, dtype=torch.uint8, device="cuda")
                acc.add_samples(d_shard, d_off, d_len, d_ids, torch.from_numpy(slots_bad.view(np.int32)).cuda(), dig)
                acc.add_samples(d_shard, d_off, d_len, d_ids, torch.from_numpy(slots_bad.view(np.int32)).cuda(), dig)
                out, counts, status = acc.digests()
                results[schedule] = (out, counts, status, dig.cpu().numpy().reshape(n, 64)[keep].tobytes())
        finally:
            lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT)
        for schedule, (out, counts, status, dig) in results.items():
            assert status == 2 * len(bad), (n, schedule)
            assert counts == [2 * c for c in want_counts], (n, schedule)
            doubled = ((np.frombuffer(want_sums, dtype="<u2").astype(np.uint32) * 2) & 0xFFFF).astype("<u2").tobytes()
            assert out == doubled, (n, schedule)
            assert dig == want_dig, (n, schedule)


def test_lthash_lanes_kernel_block_boundaries_and_alignments(dev, corc):
    """The persistent-lane LtHash kernel (default for samples of unknown / ragged length) against the C oracle on the
    lengths where its staging changes shape -- around every 128-byte chunk edge with the 8-byte tag in front (a
    sample of 120 bytes fills block 0 exactly, 121 needs a second block whose data chunk is empty) -- at 8-byte,
    4-byte and odd addresses (cp.async 8 / cp.async 4 / register path), with fewer samples than lanes, exactly one
    ring refill, and many samples per lane; the length hint must never change a result."""
    from paper_2510_00554_b200 import _native

    lib = _native.load()
    assert lib.snt_merkle_schedule(_native.SCHEDULE_PERSISTENT) == 0
    rng = np.random.default_rng(77)
    edge = np.array([0, 1, 7, 8, 9, 119, 120, 121, 127, 128, 129, 247, 248, 249, 255, 256, 257, 1016, 1024, 3072, 5000],
                    dtype=np.uint64)
    for n, align in ((len(edge), 8), (len(edge), 4), (len(edge), 1), (64, 4), (96, 8), (3000, 4), (20000, 1)):
        lens = edge.copy() if n == len(edge) else rng.choice(edge[:17], size=n).astype(np.uint64)
        offs = np.zeros(n, dtype=np.uint64)
        pos = 0
        for i in range(n):
            pos = -(-pos // align) * align
            if align == 1 and i % 2:
                pos += 1 + (i % 3)                               # odd addresses
            if align == 4 and i % 2 and pos % 8 == 0:
                pos += 4                                         # 4-byte aligned but not 8
            offs[i] = pos
            pos += int(lens[i])
        shard = rng.integers(0, 256, size=pos + 16, dtype=np.uint8)
        n_src = 5
        slots = rng.integers(0, n_src, size=n).astype(np.uint32)
        ids = rng.integers(0, 2**63, size=n).astype(np.uint64)
        want_sums, want_counts, want_dig = corc.lthash_samples(shard, offs, lens, ids, slots, n_src, 4, want_digests=True)
        d_shard = torch.from_numpy(shard).cuda()
        d_off, d_len, d_ids = (torch.from_numpy(a.view(np.int64)).cuda() for a in (offs, lens, ids))
        d_slots = torch.from_numpy(slots.view(np.int32)).cuda()
        for uniform in (None, False, True):                      # unknown and ragged: lanes; "uniform" (a lie here): the grid
            acc = dev.LatticeAccumulator(n_src)
            dig = torch.zeros(n * 64, dtype=torch.uint8, device="cuda")
            acc.add_samples(d_shard, d_off, d_len, d_ids, d_slots, dig, uniform=uniform)
            out, counts, status = acc.digests()
            assert (status, counts) == (0, list(want_counts)), (n, align, uniform)
            assert out == want_sums, (n, align, uniform)
            assert dig.cpu().numpy().tobytes() == want_dig, (n, align, uniform)


def test_resident_lattice_model_is_cached_and_revalidated(porc):
    """LATTICE in-place hashing of device-resident tensors re-uses the plan and an accumulator whose read-out lands in
    page-locked host memory; content changes, re-pointed tensors and a change of construction on the same TensorMap
    all give the oracle's answer."""
    import paper_2510_00554_b200 as pkg

    rng = np.random.default_rng(8)
    sizes = [8192 * 20 + 5, 100, 8192 * 64, 0, 7]
    host = [rng.integers(0, 256, size=s, dtype=np.uint8) for s in sizes]
    tensors = [torch.from_numpy(h).cuda() for h in host]
    model = pkg.TensorMap([(f"t{i}", t) for i, t in enumerate(tensors)])
    lat = pkg.HashConfig(pkg.Construction.LATTICE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.BLAKE2B)
    mer = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.BLAKE2B)

    def want_lat():
        return porc.inplace_lattice([h.tobytes() for h in host], 8192)

    assert pkg.hash_model(lat, model).model_digest.data == want_lat()
    entry = model.__dict__["_resident"]
    assert entry.acc is not None and entry.hasher is None
    assert pkg.hash_model(lat, model).model_digest.data == want_lat()
    assert model.__dict__["_resident"] is entry
    host[2][777] ^= 0x55
    tensors[2][777] ^= 0x55
    assert pkg.hash_model(lat, model).model_digest.data == want_lat()
    assert model.__dict__["_resident"] is entry
    host[1] = rng.integers(0, 256, size=100, dtype=np.uint8)
    tensors[1].data = torch.from_numpy(host[1]).cuda()
    assert pkg.hash_model(lat, model).model_digest.data == want_lat()
    assert model.__dict__["_resident"] is not entry
    # the other construction on the same TensorMap: a new entry, then back again
    assert pkg.hash_model(mer, model).model_digest.data == porc.inplace_merkle("blake2b", [h.tobytes() for h in host], 8192)
    assert model.__dict__["_resident"].hasher is not None
    assert pkg.hash_model(lat, model).model_digest.data == want_lat()


def test_resident_model_tiny_trees_root_lands_in_pinned_host_memory(porc):
    """One- and two-leaf device-resident models through the cached path, whose output buffer is page-locked HOST memory
    (the last kernel -- or, for a single leaf, an asynchronous device-to-host copy of the leaf digest -- writes the root
    there): repeated calls, every algorithm."""
    import paper_2510_00554_b200 as pkg

    for alg in ("sha256", "blake2b", "sha3-256"):
        cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.from_name(alg))
        for size in (1, 100, 8192, 8193, 3 * 8192):
            h = np.random.default_rng(size).integers(0, 256, size=size, dtype=np.uint8)
            m = pkg.TensorMap([("a", torch.from_numpy(h).cuda())])
            want = porc.inplace_merkle(alg, [h.tobytes()], 8192)
            for _ in range(3):
                assert pkg.hash_model(cfg, m).model_digest.data == want, (alg, size)
            assert m.__dict__["_resident"].hasher.out.device.type == "cpu"


def test_resident_model_cache_revalidates_every_call(porc):
    """hash_model on a TensorMap of CUDA tensors re-uses plan and workspace, launches before it re-checks the tensors,
    and still never returns a digest for bytes it did not check: content changes, re-pointed tensors, resized tensors
    and replaced entries all give the oracle's answer; a second TensorMap over the same tensors gets its own entry."""
    import paper_2510_00554_b200 as pkg
    from paper_2510_00554_b200 import model as mm

    rng = np.random.default_rng(3)
    sizes = [8192 * 50 + 100, 4096, 8192 * 300, 12, 8192 * 7]
    host = [rng.integers(0, 256, size=s, dtype=np.uint8) for s in sizes]
    tensors = [torch.from_numpy(h).cuda() for h in host]
    model = pkg.TensorMap([(f"t{i}", t) for i, t in enumerate(tensors)])

    def want(alg):
        return porc.inplace_merkle(alg, [h.tobytes() for h in host], 8192)

    for alg in ("sha256", "blake2b"):
        cfg = pkg.HashConfig(pkg.Construction.MERKLE, pkg.Strategy.IN_PLACE, pkg.CompressionAlg.from_name(alg))
        assert pkg.hash_model(cfg, model).model_digest.data == want(alg)
        assert "_resident" in model.__dict__
        entry = model.__dict__["_resident"]
        assert pkg.hash_model(cfg, model).model_digest.data == want(alg)
        assert model.__dict__["_resident"] is entry                      # re-used
        # 1. content changes in place: same plan, new digest
        host[2][12345] ^= 0xFF
        tensors[2][12345] ^= 0xFF
        assert pkg.hash_model(cfg, model).model_digest.data == want(alg)
        assert model.__dict__["_resident"] is entry
        # 2. a tensor object re-pointed to other storage (same id, other address): speculation is discarded
        host[1] = rng.integers(0, 256, size=4096, dtype=np.uint8)
        tensors[1].data = torch.from_numpy(host[1]).cuda()
        assert pkg.hash_model(cfg, model).model_digest.data == want(alg)
        assert model.__dict__["_resident"] is not entry
        entry = model.__dict__["_resident"]
        # 3. an entry replaced by a tensor of another size
        host[3] = rng.integers(0, 256, size=9000, dtype=np.uint8)
        tensors[3] = torch.from_numpy(host[3]).cuda()
        model.entries[3] = ("t3", tensors[3])
        assert pkg.hash_model(cfg, model).model_digest.data == want(alg)
        # 4. a non-contiguous view falls back to the uncached path and hashes the logical bytes
        base = torch.from_numpy(rng.integers(0, 256, size=(64, 256), dtype=np.uint8)).cuda()
        view = base.t()
        m2 = pkg.TensorMap([("v", view), ("w", tensors[0])])
        assert pkg.hash_model(cfg, m2).model_digest.data == \
            porc.inplace_merkle(alg, [view.contiguous().cpu().numpy().tobytes(), host[0].tobytes()], 8192)
        # 5. another TensorMap over the same tensors: its own entry, same digest
        m3 = pkg.TensorMap([(f"t{i}", t) for i, t in enumerate(tensors)])
        assert pkg.hash_model(cfg, m3).model_digest.data == want(alg)
        assert m3.__dict__["_resident"] is not model.__dict__["_resident"]
        # 6. a cached tensor object moved to the host in place (same id, no longer a CUDA tensor): generic path
        assert pkg.hash_model(cfg, m3).model_digest.data == want(alg)
        host[4] = rng.integers(0, 256, size=sizes[4], dtype=np.uint8)
        tensors[4].data = torch.from_numpy(host[4])
        assert pkg.hash_model(cfg, m3).model_digest.data == want(alg)
        assert "_resident" not in m3.__dict__
        tensors[4].data = torch.from_numpy(host[4]).cuda()
        mm.clear_hash_cache(model)
        assert "_resident" not in model.__dict__
        assert pkg.hash_model(cfg, model).model_digest.data == want(alg)


def test_process_batch_keeps_sums_on_the_device(porc):
    """The reference's loader protocol on the device-resident accumulator: many small batches, sources appearing late
    (slot table growth past its first capacity), cover_labels, reads of acc.sums in the middle, merge of two accumulators."""
    import paper_2510_00554_b200 as pkg

    rng = np.random.default_rng(9)
    n, n_src = 3000, 70                                   # more sources than the engine's first 32 slots
    samples = []
    for i in range(n):
        src = int(rng.integers(0, 1 + min(n_src - 1, i // 20)))          # later sources show up as the loop goes on
        data = rng.integers(0, 256, size=int(rng.integers(0, 400)), dtype=np.uint8).tobytes()
        samples.append((10_000 + i, src, f"c{i % 5}".encode(), data))
    for cover in (False, True):
        acc = pkg.SourceAccumulator(cover_labels=cover)
        other = pkg.SourceAccumulator(cover_labels=cover)
        for s in range(0, n, 37):
            recs = [pkg.SampleRecord(*t) for t in samples[s:s + 37]]
            pkg.process_batch(pkg.Batch(recs), acc if (s // 37) % 3 else other)
            if s == 37 * 20:
                assert sum(acc.counts.values()) + sum(other.counts.values()) == s + len(recs)    # mid-stream read
        acc.merge(other)
        got = pkg.finalize(acc)
        want = porc.dataset_digests(samples, cover_labels=cover)
        assert {k: (v[0].data, v[1]) for k, v in got.items()} == {k: (v[0], v[1]) for k, v in want.items()}
