"""Wall time of the manifest-level call digest_dataset(manifest) (dataset.py:166-195) on a CIFAR10-shaped shard
written to a temporary directory: this package against the reference package (oracle/_ref, checker only), same
files, results compared. cProfile of one call of ours on stderr."""
import cProfile
import io
import json
import pstats
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2510_00554_b200 as snt  # noqa: E402

n, ln, n_src = 50_000, 3072, 16
data = np.random.default_rng(0).integers(0, 256, size=n * ln, dtype=np.uint8).tobytes()
r1 = np.random.default_rng(1)
src = r1.choice(n_src, size=n, p=r1.dirichlet(np.ones(n_src)))
out = {}
with tempfile.TemporaryDirectory() as tmp:
    rows = [(i, int(src[i]), b"cat%d" % (i % 10), i * ln, ln) for i in range(n)]
    man = snt.DatasetManifest(rows, Path(tmp) / "shard.bin")
    man.save(Path(tmp) / "manifest.json", data)
    for cover in (False, True):
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            m = snt.DatasetManifest.load(Path(tmp) / "manifest.json")
            t1 = time.perf_counter()
            got = snt.digest_dataset(m, cover_labels=cover)
            ts.append((time.perf_counter() - t1, t1 - t0))
        out[f"ours_cover{int(cover)}_ms"] = round(min(t[0] for t in ts) * 1e3, 1)
        out["manifest_load_ms"] = round(min(t[1] for t in ts) * 1e3, 1)
        if cover:
            prof = cProfile.Profile()
            prof.enable()
            snt.digest_dataset(m, cover_labels=cover)
            prof.disable()
            s = io.StringIO()
            pstats.Stats(prof, stream=s).sort_stats("tottime").print_stats(14)
            print(s.getvalue()[:4000], file=sys.stderr)
        ref_dir = ROOT / "oracle" / "_ref"
        if (ref_dir / "sentinel").is_dir():
            sys.path.insert(0, str(ref_dir))
            import sentinel as ref  # noqa: E402
            rm = ref.DatasetManifest.load(Path(tmp) / "manifest.json")
            t0 = time.perf_counter()
            want = ref.digest_dataset(rm, cover_labels=cover)
            out[f"reference_cover{int(cover)}_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
            assert {k: (v[0].data, v[1]) for k, v in want.items()} == {k: (v[0].data, v[1]) for k, v in got.items()}
            out["parity"] = "identical"
print(json.dumps(out))
