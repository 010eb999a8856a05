"""Per-source dataset digests: every sample LtHashed on the GPU, summed per source.

API mirror of the reference's ``dataset.py`` (:24-195). A sample's digest is
BLAKE2b-512(LE64(sample_id) || data) -- with ``cover_labels`` the label bytes sit
between the id and the data (dataset.py:41-49) -- and a source's digest is the
lane-wise sum modulo 2^16 of its samples' digests, so the result does not depend
on shuffle order, batch size or how the samples are split across GPUs.

Two ways in:

* ``process_batch(batch, acc)`` keeps the reference's host-object protocol: the
  batch is packed, copied to the device, hashed and reduced per source by one
  kernel launch, and the per-source partial sums are folded into ``acc``.
* ``digest_dataset`` / ``DeviceDataset`` is the device-resident path: the whole
  shard and its (offset, length, id, source slot) rows live in HBM and one
  launch digests every sample (the manifest layout of dataset.py:94-100).
"""

from __future__ import annotations

import json
import random
from dataclasses import dataclass, field
from pathlib import Path
from typing import Dict, Iterable, Iterator, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import device as _dev
from .errors import FormatError, ValidationError
from .lattice import LatticeDigest, lt_add, lt_hash_block, lt_hash_tagged, lt_zero


def _slots_of(src: np.ndarray, table: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Accumulator slot of every sample's source id (index into the sorted ``table`` of declared ids) and whether the
    id is declared at all. Source ids are small integers in practice: a lookup table over [table[0], table[-1]]
    (0.1 ms for 50,000 samples) instead of a binary search per sample (numpy's searchsorted: 1 ms)."""
    if table.size and src.size and int(table[-1]) - int(table[0]) < (1 << 20):
        lo = int(table[0])
        if int(src.min()) >= lo and int(src.max()) <= int(table[-1]):
            lut = np.full(int(table[-1]) - lo + 1, table.size, dtype=np.int64)
            lut[table - lo] = np.arange(table.size, dtype=np.int64)
            slots = lut[src - lo]
            return slots, slots < table.size
    slots = np.searchsorted(table, src)
    if table.size:
        return slots, table[np.minimum(slots, table.size - 1)] == src
    return slots, np.zeros(src.shape, dtype=bool)


def _all_equal(lengths: np.ndarray) -> bool:
    """Do all samples have one length? Selects the launch (uniform samples: one thread per sample on a plain
    grid; ragged ones: the persistent-lane kernel, which needs no length sort), never the result."""
    return lengths.size == 0 or bool((lengths == lengths.flat[0]).all())


def _checked_ids(ids) -> np.ndarray:
    """Sample ids as u64; an id outside [0, 2^64) is an error, as it is for the reference's
    ``struct.pack("<Q", sample_id)`` (dataset.py:45) -- never wrapped into another sample's tag."""
    if ids and not (0 <= min(ids) and max(ids) < (1 << 64)):
        i = next(i for i in ids if not 0 <= i < (1 << 64))
        raise ValidationError(f"sample id {i} does not fit an unsigned 64-bit tag")
    return np.array(ids, dtype=np.uint64)


@dataclass(frozen=True)
class SampleRecord:
    sample_id: int
    source_id: int
    label: bytes
    data: bytes


@dataclass
class Batch:
    samples: List[SampleRecord]

    @property
    def size(self) -> int:
        return len(self.samples)


def hash_sample(s: SampleRecord, cover_labels: bool = False) -> LatticeDigest:
    """LtHash of one sample tagged with its stable id (dataset.py:41-49); one GPU launch."""
    if cover_labels:
        import struct

        return lt_hash_tagged(struct.pack("<Q", s.sample_id) + s.label, s.data)
    return lt_hash_block(s.sample_id, s.data)


def _raise_record_error(code: int, s: "SampleRecord") -> None:
    """The check codes of ``_hostpack.pack_records`` as the exceptions ``process_batch`` raises."""
    if code == 2:
        raise ValidationError(f"sample {s.sample_id} references undeclared source {s.source_id}")
    if code == 3:
        raise ValidationError(f"sample id {s.sample_id} does not fit an unsigned 64-bit tag")


class _BatchEngine:
    """Device side of a ``SourceAccumulator`` that is fed batch by batch (``process_batch``).

    Everything a batch needs travels as ONE block: ``offsets | lengths | ids | slots | sample bytes`` is
    packed into a pinned staging buffer (two of them, used alternately, each re-used once the copy that
    read it has completed), goes to a persistent device buffer with one asynchronous copy, and one
    ``snt_lthash_samples`` launch adds the batch into per-source lane sums that stay in HBM. Nothing is
    allocated per batch and nothing synchronises until the sums are asked for (``drain``).
    """

    HEADER_ALIGN = 16

    def __init__(self):
        self.device = _dev.require_cuda()
        self.slot_of: Dict[int, int] = {}
        self.capacity = 32
        self.acc = _dev.LatticeAccumulator(self.capacity)
        self.stage: List[Optional[torch.Tensor]] = [None, None]
        self.stage_done: List[Optional[torch.cuda.Event]] = [None, None]
        self.turn = 0
        self.d_block: Optional[torch.Tensor] = None
        self.pending = False
        self._last_need = 0

    def _slot(self, sid: int) -> int:
        slot = self.slot_of.get(sid)
        if slot is None:
            slot = len(self.slot_of)
            if slot >= self.capacity:                      # more sources than slots: carry the sums over to a bigger state
                grown = _dev.LatticeAccumulator(self.capacity * 4)
                n = self.capacity
                grown.acc[:n * _dev.LT_LANES].copy_(self.acc.acc)
                grown.counts[:n].copy_(self.acc.counts)
                grown.status.copy_(self.acc.status)
                self.acc, self.capacity = grown, self.capacity * 4
            self.slot_of[sid] = slot
        return slot

    def _stage_for(self, need: int) -> Tuple[int, torch.Tensor]:
        """A staging block of at least ``need`` bytes whose last transfer has completed, and its index."""
        turn = self.turn
        self.turn ^= 1
        if self.stage[turn] is None or self.stage[turn].numel() < need:
            self.stage[turn] = torch.empty(max(need * 2, 1 << 20), dtype=torch.uint8, pin_memory=True)
            self.stage_done[turn] = None
        if self.stage_done[turn] is not None:
            self.stage_done[turn].synchronize()            # the copy that last read this staging buffer
        if self.d_block is None or self.d_block.numel() < need:
            self.d_block = torch.empty(max(need * 2, 1 << 20), dtype=torch.uint8, device=self.device)
        return turn, self.stage[turn]

    def _launch(self, turn: int, n: int, header: int, need: int, uniform: bool) -> None:
        d = self.d_block
        d[:need].copy_(self.stage[turn][:need], non_blocking=True)
        done = torch.cuda.Event()
        done.record()
        self.stage_done[turn] = done
        self.acc.add_packed(d, n, header, uniform=uniform)
        self.pending = True

    def add_records(self, samples: Sequence[SampleRecord], cover_labels: bool, declared: Optional[frozenset]) -> bool:
        """Pack the records with the C helper (one pass: checks, header, payload bytes straight into the pinned
        block) and launch. False when the helper is not built; the checks raise what ``process_batch`` raises."""
        pack = _dev._hostpack
        if pack is None:
            return False
        n = len(samples)
        turn, stage = self._stage_for(max(self._last_need, 1 << 20))
        while True:
            code, a, b = pack.pack_records(samples, cover_labels, self.slot_of, declared, stage.data_ptr(), stage.numel())
            if code == 0:
                break
            if code == 1:                                   # block too small: grow it and pack again
                self.turn ^= 1
                turn, stage = self._stage_for(a)
            elif code == 4:                                 # a source seen for the first time
                self._slot(samples[a].source_id)
            else:
                _raise_record_error(code, samples[a])
        total, header = a, b
        need = header + max(total, 16)
        self._last_need = need
        if self.d_block.numel() < need:
            self.d_block = torch.empty(need * 2, dtype=torch.uint8, device=self.device)
        lens = stage[8 * n:16 * n].numpy().view(np.uint64)
        self._launch(turn, n, header, need, _all_equal(lens))
        return True

    def add(self, payloads: Sequence[bytes], ids: np.ndarray, source_ids: Sequence[int]) -> None:
        n = len(payloads)
        lengths = np.fromiter(map(len, payloads), dtype=np.uint64, count=n)
        total = int(lengths.sum())
        header = -(-28 * n // self.HEADER_ALIGN) * self.HEADER_ALIGN
        need = header + max(total, 16)
        turn, stage = self._stage_for(need)
        view = stage.numpy()
        offsets = view[0:8 * n].view(np.uint64)
        offsets[0] = 0
        np.cumsum(lengths[:-1], out=offsets[1:])
        view[8 * n:16 * n].view(np.uint64)[:] = lengths
        view[16 * n:24 * n].view(np.uint64)[:] = ids
        try:
            slots = list(map(self.slot_of.__getitem__, source_ids))      # sources seen before: one dict lookup each
        except KeyError:
            slots = [self._slot(s) for s in source_ids]
        view[24 * n:28 * n].view(np.int32)[:] = slots
        view[header:header + total] = np.frombuffer(b"".join(payloads), dtype=np.uint8)
        self._launch(turn, n, header, need, _all_equal(lengths))

    def drain(self) -> Dict[int, Tuple[bytes, int]]:
        """Per-source (64 digest bytes, count) accumulated since the last drain; synchronises, then starts from zero."""
        out, counts, status = self.acc.digests()
        if status:
            raise ValidationError("a sample references an undeclared source")
        self.acc.zero_()
        self.pending = False
        return {sid: (out[64 * slot:64 * slot + 64], counts[slot]) for sid, slot in self.slot_of.items() if counts[slot]}


class SourceAccumulator:
    """Per-source running lattice sums and sample counts (mirror of dataset.py:52-71).

    ``process_batch`` keeps the running sums on the device (``_BatchEngine``); ``sums`` and ``counts``
    are the reference's host dictionaries and fold the device state in whenever they are read, so the
    object behaves like the reference's dataclass while a loader loop never waits for the GPU.
    """

    def __init__(self, sums: Optional[Dict[int, LatticeDigest]] = None, counts: Optional[Dict[int, int]] = None,
                 declared_sources: Optional[frozenset] = None, cover_labels: bool = False):
        self._sums: Dict[int, LatticeDigest] = {} if sums is None else sums
        self._counts: Dict[int, int] = {} if counts is None else counts
        self.declared_sources = declared_sources
        self.cover_labels = cover_labels
        self._engine: Optional[_BatchEngine] = None

    def _sync(self) -> None:
        if self._engine is not None and self._engine.pending:
            for sid, (digest, count) in self._engine.drain().items():
                self._sums[sid] = lt_add(self._sums.get(sid, lt_zero()), LatticeDigest(digest))
                self._counts[sid] = self._counts.get(sid, 0) + count

    @property
    def sums(self) -> Dict[int, LatticeDigest]:
        self._sync()
        return self._sums

    @sums.setter
    def sums(self, value: Dict[int, LatticeDigest]) -> None:
        self._sync()
        self._sums = value

    @property
    def counts(self) -> Dict[int, int]:
        self._sync()
        return self._counts

    @counts.setter
    def counts(self, value: Dict[int, int]) -> None:
        self._sync()
        self._counts = value

    def declare(self, source_ids: Iterable[int]) -> None:
        self.declared_sources = frozenset(source_ids)
        for sid in self.declared_sources:
            self.sums.setdefault(sid, lt_zero())
            self.counts.setdefault(sid, 0)

    def merge(self, other: "SourceAccumulator") -> None:
        """Fold another accumulator in; any merge order gives the same sums."""
        for sid, digest in other.sums.items():
            self.sums[sid] = lt_add(self.sums.get(sid, lt_zero()), digest)
            self.counts[sid] = self.counts.get(sid, 0) + other.counts.get(sid, 0)

    def __repr__(self) -> str:
        return (f"SourceAccumulator(sums={self.sums!r}, counts={self.counts!r}, "
                f"declared_sources={self.declared_sources!r}, cover_labels={self.cover_labels!r})")

    def __eq__(self, other) -> bool:
        if not isinstance(other, SourceAccumulator):
            return NotImplemented
        return (self.sums, self.counts, self.declared_sources, self.cover_labels) == \
               (other.sums, other.counts, other.declared_sources, other.cover_labels)


class DeviceDataset:
    """A shard and its sample rows resident in HBM (the GPU input format).

    ``shard``: flat uint8 tensor; ``offsets``/``lengths``/``ids``: int64 tensors
    (bit patterns of u64); ``slots``: int32 index into ``source_ids``.
    """

    def __init__(self, shard: torch.Tensor, offsets: torch.Tensor, lengths: torch.Tensor,
                 ids: torch.Tensor, slots: torch.Tensor, source_ids: Sequence[int], uniform: Optional[bool] = None):
        self.shard, self.offsets, self.lengths, self.ids, self.slots = shard, offsets, lengths, ids, slots
        self.source_ids = list(source_ids)
        self.uniform = uniform           # all lengths equal? (None = not known; see LatticeAccumulator.add_samples)

    @property
    def n_samples(self) -> int:
        return int(self.offsets.numel())

    @classmethod
    def from_host(cls, shard, offsets, lengths, ids, source_of_sample, source_ids: Sequence[int],
                  pinned: bool = True) -> "DeviceDataset":
        """Copy host arrays to the device. ``source_of_sample`` holds source ids, not slots.

        The shard copy is enqueued first (asynchronous when the shard is pinned) so that the
        host-side slot mapping overlaps it; the four row arrays then travel as ONE packed,
        pinned buffer (3 x u64 + 1 x u32 per sample) instead of four pageable copies.
        """
        dev = _dev.require_cuda()
        shard_t = _dev.as_device_bytes(shard, dev)
        if shard_t.numel() == 0:
            shard_t = torch.zeros(16, dtype=torch.uint8, device=dev)
        source_ids = sorted(set(int(s) for s in source_ids))
        src = np.asarray(source_of_sample, dtype=np.int64)
        n = int(src.shape[0])
        table = np.asarray(source_ids, dtype=np.int64)
        slots, hit = _slots_of(src, table)
        if not hit.all():
            i = int(np.nonzero(~hit)[0][0])
            raise ValidationError(f"sample {int(np.asarray(ids)[i])} references undeclared source {int(src[i])}")

        packed = torch.empty(max(n, 1) * 28, dtype=torch.uint8, pin_memory=True)
        view = packed.numpy()
        view[0:8 * n].view(np.uint64)[:] = np.asarray(offsets, dtype=np.uint64)
        lengths = np.asarray(lengths, dtype=np.uint64)
        view[8 * n:16 * n].view(np.uint64)[:] = lengths
        view[16 * n:24 * n].view(np.uint64)[:] = np.asarray(ids, dtype=np.uint64)
        view[24 * n:28 * n].view(np.int32)[:] = slots.astype(np.int32, copy=False)
        rows = packed.to(dev, non_blocking=True)
        ds = cls(shard_t, rows[0:8 * n].view(torch.int64), rows[8 * n:16 * n].view(torch.int64),
                 rows[16 * n:24 * n].view(torch.int64), rows[24 * n:28 * n].view(torch.int32), source_ids,
                 uniform=_all_equal(lengths))
        ds._staging = packed      # the pinned staging block outlives the asynchronous copy
        return ds

    def sorted_by_length(self) -> "DeviceDataset":
        """The same samples with the rows ordered by length (device-side argsort, shard untouched).

        Per-source sums do not depend on the order (dataset.py:67-71). Round 1 hashed large ragged datasets
        in this order because the one-thread-per-sample grid runs a warp as long as its longest sample
        (2 M hellaswag-shaped samples: 2.94 ms unsorted, 1.26 ms sorted + 0.42 ms of sorting). The
        persistent-lane kernel takes them unsorted in 1.09 ms (tools/lthash_lanes_probe.py), so nothing in the
        package sorts any more; the method stays for callers that want length order for their own reasons.
        """
        order = torch.argsort(self.lengths)
        return DeviceDataset(self.shard, self.offsets[order], self.lengths[order], self.ids[order], self.slots[order],
                             self.source_ids, uniform=self.uniform)

    def accumulate(self, acc: "_dev.LatticeAccumulator", begin: int = 0, end: Optional[int] = None,
                   digests: Optional[torch.Tensor] = None) -> None:
        """Enqueue the LtHash of samples [begin, end) into ``acc`` (no synchronisation)."""
        end = self.n_samples if end is None else end
        if end <= begin:
            return
        acc.add_samples(self.shard, self.offsets[begin:end], self.lengths[begin:end], self.ids[begin:end],
                        self.slots[begin:end], digests, uniform=self.uniform)


def _finalize_device(acc: "_dev.LatticeAccumulator", source_ids: Sequence[int]) -> Dict[int, Tuple[LatticeDigest, int]]:
    out, counts, status = acc.digests()
    if status:
        raise ValidationError("a sample references an undeclared source")
    return {sid: (LatticeDigest(out[64 * i:64 * i + 64]), counts[i]) for i, sid in enumerate(source_ids)}


def process_batch(batch: Batch, acc: SourceAccumulator) -> SourceAccumulator:
    """Hash a batch on the GPU and add it to the running per-source sums (dataset.py:74-86).

    The batch is packed into a reused pinned block, copied with one asynchronous transfer and hashed by
    one launch into sums that stay on the device; the call returns without waiting for the GPU. The
    host-side ``acc.sums`` / ``acc.counts`` catch up when they are read (``finalize`` does).
    """
    samples = batch.samples
    if samples and _dev._hostpack is not None:
        if acc._engine is None:
            # first batch: the checks alone (no destination), so that a bad batch raises before anything touches the device
            code, at, _ = _dev._hostpack.pack_records(samples, acc.cover_labels, {}, acc.declared_sources, 0, 0)
            _raise_record_error(code, samples[at] if code in (2, 3) else None)
            acc._engine = _BatchEngine()
        acc._engine.add_records(samples, acc.cover_labels, acc.declared_sources)
        return acc
    source_ids = [s.source_id for s in samples]
    if acc.declared_sources is not None and not acc.declared_sources.issuperset(source_ids):
        s = next(s for s in samples if s.source_id not in acc.declared_sources)
        raise ValidationError(f"sample {s.sample_id} references undeclared source {s.source_id}")
    if not samples:
        return acc
    payloads = [s.label + s.data for s in samples] if acc.cover_labels else [s.data for s in samples]
    ids = _checked_ids([s.sample_id for s in samples])
    if acc._engine is None:
        acc._engine = _BatchEngine()
    acc._engine.add(payloads, ids, source_ids)
    return acc


def finalize(acc: SourceAccumulator) -> Dict[int, Tuple[LatticeDigest, int]]:
    """Per-source digests and counts, ordered by source id (dataset.py:89-91)."""
    return {sid: (acc.sums[sid], acc.counts.get(sid, 0)) for sid in sorted(acc.sums)}


@dataclass
class DatasetManifest:
    """Sample index over a flat binary shard (format of dataset.py:94-137)."""

    samples: List[Tuple[int, int, bytes, int, int]]   # (sample_id, source_id, label, offset, length)
    data_path: Path
    expected_digests: Dict[int, str] = field(default_factory=dict)

    @property
    def source_ids(self) -> frozenset:
        return frozenset(rec[1] for rec in self.samples)

    @classmethod
    def load(cls, manifest_path) -> "DatasetManifest":
        manifest_path = Path(manifest_path)
        try:
            doc = json.loads(manifest_path.read_text())
            rows = [(int(r["sample_id"]), int(r["source_id"]), str(r.get("label", "")).encode(),
                     int(r["offset"]), int(r["length"])) for r in doc["samples"]]
            data_path = manifest_path.parent / doc["data"]
            expected = {int(k): v for k, v in doc.get("expected_digests", {}).items()}
        except (OSError, KeyError, ValueError, TypeError) as exc:
            raise FormatError(f"bad dataset manifest {manifest_path}: {exc}") from exc
        if len({r[0] for r in rows}) != len(rows):
            raise FormatError("sample ids must be unique within a dataset")
        return cls(rows, data_path, expected)

    def save(self, manifest_path, shard: bytes) -> None:
        manifest_path = Path(manifest_path)
        rows = [{"sample_id": sid, "source_id": src, "label": label.decode(), "offset": off, "length": ln}
                for sid, src, label, off, ln in self.samples]
        (manifest_path.parent / self.data_path.name).write_bytes(shard)
        manifest_path.write_text(json.dumps({"samples": rows, "data": self.data_path.name,
                                             "expected_digests": self.expected_digests}))


def iterate_batches(manifest: DatasetManifest, batch_size: int, shuffle_seed: int) -> Iterator[Batch]:
    """Every sample exactly once, in a seed-determined shuffle (dataset.py:140-163)."""
    if batch_size < 1:
        raise ValidationError("batch_size must be >= 1")
    try:
        shard = memoryview(manifest.data_path.read_bytes())
    except OSError as exc:
        raise FormatError(f"cannot read data shard {manifest.data_path}: {exc}") from exc
    order = list(range(len(manifest.samples)))
    random.Random(shuffle_seed).shuffle(order)
    for start in range(0, len(order), batch_size):
        recs = []
        for idx in order[start:start + batch_size]:
            sid, src, label, off, ln = manifest.samples[idx]
            if off < 0 or off + ln > len(shard):
                raise FormatError(f"sample {sid} range [{off}, {off + ln}) exceeds shard")
            recs.append(SampleRecord(sid, src, label, bytes(shard[off:off + ln])))
        yield Batch(recs)


def digest_dataset(manifest: DatasetManifest, batch_size: int = 128, shuffle_seed: int = 0,
                   cover_labels: bool = False, workers: int = 1) -> Dict[int, Tuple[LatticeDigest, int]]:
    """Digest a whole manifest (dataset.py:166-195) with the shard resident in HBM.

    The digests are invariant to ``batch_size``, ``shuffle_seed`` and ``workers``
    (SPEC.md:402), so the device path hashes all samples in one launch; the
    arguments are validated and otherwise unused.
    """
    if batch_size < 1:
        raise ValidationError("batch_size must be >= 1")
    try:
        shard = _dev.file_to_device(manifest.data_path)      # read by the staging threads straight into pinned memory
    except OSError as exc:
        raise FormatError(f"cannot read data shard {manifest.data_path}: {exc}") from exc
    n = len(manifest.samples)
    if n == 0:
        return {}
    ids, src, off, ln = _manifest_columns(manifest.samples)
    source_ids = np.unique(src).tolist()
    shard_len = int(shard.numel())
    bad = np.nonzero((off < 0) | (ln < 0) | (off + ln > shard_len))[0]
    if bad.size:
        i = int(bad[0])
        raise FormatError(f"sample {int(ids[i])} range [{int(off[i])}, {int(off[i] + ln[i])}) exceeds shard")
    if cover_labels:
        shard, off, ln = _prefix_labels(shard, [r[2] for r in manifest.samples], off, ln)
    ds = DeviceDataset.from_host(shard, off.astype(np.uint64), ln.astype(np.uint64), ids, src, source_ids)
    acc = _dev.LatticeAccumulator(len(source_ids))
    ds.accumulate(acc)
    return _finalize_device(acc, ds.source_ids)


def _manifest_columns(rows) -> Tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """(ids u64, source ids, offsets, lengths i64) of manifest rows: one C pass when the helper is built."""
    n = len(rows)
    if _dev._hostpack is not None:
        ids = np.empty(n, dtype=np.uint64)
        src, off, ln = (np.empty(n, dtype=np.int64) for _ in range(3))
        code, at = _dev._hostpack.manifest_columns(rows, ids.ctypes.data, src.ctypes.data, off.ctypes.data, ln.ctypes.data)
        if code == 0:
            return ids, src, off, ln
        if code == 3:
            raise ValidationError(f"sample id {rows[at][0]} does not fit an unsigned 64-bit tag")
    return (_checked_ids([r[0] for r in rows]), np.array([r[1] for r in rows], dtype=np.int64),
            np.array([r[3] for r in rows], dtype=np.int64), np.array([r[4] for r in rows], dtype=np.int64))


def _prefix_labels(shard: torch.Tensor, labels: Sequence[bytes], off: np.ndarray, ln: np.ndarray):
    """``cover_labels``: the message of sample i is LE64(id) ‖ label ‖ data (dataset.py:47-48). The shard is already in
    HBM; the labels follow as one small block and ONE gather launch lays ``label_i ‖ data_i`` out back to back in a
    second device buffer (the host used to rebuild the whole shard: 140 of 218 ms for 50,000 CIFAR-sized samples)."""
    n = len(labels)
    dev = shard.device
    lab_len = np.fromiter(map(len, labels), dtype=np.int64, count=n)
    lab_off = np.zeros(n, dtype=np.int64)
    np.cumsum(lab_len[:-1], out=lab_off[1:])
    blob = _dev.as_device_bytes(b"".join(labels) or bytes(16), dev)
    new_ln = lab_len + ln
    new_off = np.zeros(n, dtype=np.int64)
    np.cumsum(new_ln[:-1], out=new_off[1:])
    total = int(new_ln.sum())
    packed = torch.empty(max(total, 16), dtype=torch.uint8, device=dev)
    src_addr = np.concatenate([blob.data_ptr() + lab_off, shard.data_ptr() + off]).astype(np.uint64)
    _dev.gather_spans(src_addr, np.concatenate([lab_len, ln]).astype(np.uint64),
                      np.concatenate([new_off, new_off + lab_len]).astype(np.uint64), 0, packed)
    packed._sources = (blob, shard)          # read by the gather launch: keep them until the stream is synchronised
    return packed, new_off, new_ln


class StreamingDatasetHasher:
    """Per-source LtHash folded into a training loop, batch by batch, with no host round trip.

    The reference's loader-side protocol is ``process_batch(batch, acc)`` over host records
    (dataset.py:74-86, the on-the-fly use of PAPER.md:504-515). Here a batch is what a GPU data
    loader already holds: a ``[B, ...]`` tensor of fixed-size samples (any dtype, CUDA or pinned
    host memory) plus ``sample_ids`` and ``source_ids`` tensors. ``update`` enqueues ONE launch on the
    current stream (``snt_lthash_rows``: the kernel maps source ids to accumulator slots itself) and
    returns at once; nothing is synchronised until ``finalize``. The result equals
    ``digest_dataset`` over the same samples for any batch size and order.
    """

    def __init__(self, source_ids: Iterable[int]):
        self._dev = _dev.require_cuda()
        self.source_ids = sorted(set(int(s) for s in source_ids))
        if not self.source_ids:
            raise ValidationError("at least one declared source is required")
        self._table = torch.tensor(self.source_ids, dtype=torch.int64, device=self._dev)
        self._acc = _dev.LatticeAccumulator(len(self.source_ids))

    def _int64_on_device(self, values, n: int, what: str) -> torch.Tensor:
        t = values if isinstance(values, torch.Tensor) else torch.as_tensor(values)
        if t.device != self._dev or t.dtype != torch.int64 or not t.is_contiguous():
            t = t.to(self._dev, dtype=torch.int64, non_blocking=True).contiguous()
        t = t.reshape(-1)
        if t.numel() != n:
            raise ValidationError(f"{what} needs one entry per row of the batch")
        return t

    def update(self, data: torch.Tensor, sample_ids, source_ids) -> None:
        """Fold one batch in: row i of ``data`` is sample ``sample_ids[i]`` of source ``source_ids[i]``.

        ONE launch (``snt_lthash_rows``): the kernel derives row addresses from the row size and looks the source id
        of every row up in the table of declared ids itself; an undeclared id is flagged in the status word and
        raises in ``finalize``."""
        if data.dim() < 1 or data.shape[0] == 0:
            return
        n = int(data.shape[0])
        flat = _dev.as_device_bytes(data, self._dev)
        ids = self._int64_on_device(sample_ids, n, "sample_ids")
        src = self._int64_on_device(source_ids, n, "source_ids")
        self._acc.add_rows(flat, flat.numel() // n, n, ids, src, self._table)

    def finalize(self) -> Dict[int, Tuple[LatticeDigest, int]]:
        """Per-source digests and counts, ordered by source id; raises if any batch named an undeclared source."""
        return _finalize_device(self._acc, self.source_ids)

    def allreduce(self, group=None) -> None:
        """Combine the per-rank sums of a data-parallel job (one all-reduce, see distributed.py)."""
        from . import distributed as _dd

        _dd.allreduce_lattice(self._acc.state, group)
