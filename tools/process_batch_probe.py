"""Host cost of the reference-shaped loader loop: process_batch over batches of 128 prebuilt SampleRecords
(CIFAR10-shaped, 50,000 x 3,072 B), records built outside the timed region; cProfile of the loop on stderr."""
import cProfile
import io
import json
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_00554_b200 import dataset as dsm  # noqa: E402

n, ln, n_src, bs = 50_000, 3072, 16, 128
data = np.random.default_rng(0).integers(0, 256, size=n * ln, dtype=np.uint8).tobytes()
src = np.random.default_rng(1).integers(0, n_src, size=n)
batches = [dsm.Batch([dsm.SampleRecord(i, int(src[i]), b"", data[i * ln:(i + 1) * ln]) for i in range(s, min(n, s + bs))])
           for s in range(0, n, bs)]


def loop():
    acc = dsm.SourceAccumulator()
    acc.declare(range(n_src))
    for b in batches:
        dsm.process_batch(b, acc)
    return dsm.finalize(acc)


ref = loop()
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    out = loop()
    ts.append(time.perf_counter() - t0)
assert out == ref
prof = cProfile.Profile()
prof.enable()
loop()
prof.disable()
s = io.StringIO()
pstats.Stats(prof, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue()[:6000], file=sys.stderr)
print(json.dumps({"batches": len(batches), "loop_ms": round(min(ts) * 1e3, 2), "us_per_batch": round(min(ts) / len(batches) * 1e6, 1),
                  "samples_per_s": round(n / min(ts))}))
