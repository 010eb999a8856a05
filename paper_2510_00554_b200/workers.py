"""Work partitioning helpers.

In the reference (``workers.py:20-66``) a thread pool fans contiguous index
ranges out to CPU workers. Here the CUDA grid plays that role, so ``workers``
arguments are accepted everywhere for API compatibility and ignored by the
kernels. ``chunk_ranges`` survives because the multi-GPU layer uses the same
contiguous-range rule to split shards across ranks.
"""

from __future__ import annotations

import os
from typing import Callable, List, Optional, Tuple, TypeVar

T = TypeVar("T")

WORKERS_ENV = "SENTINEL_WORKERS"


def resolve_workers(requested: Optional[int] = None) -> int:
    """Explicit argument, else ``SENTINEL_WORKERS``, else the CPU count (workers.py:20-27)."""
    if requested is not None:
        return max(1, int(requested))
    env = os.environ.get(WORKERS_ENV)
    return max(1, int(env)) if env else (os.cpu_count() or 1)


def chunk_ranges(n: int, workers: int) -> List[Tuple[int, int]]:
    """At most ``workers`` contiguous half-open ranges covering [0, n); sizes differ by <= 1."""
    if n <= 0:
        return []
    parts = min(max(1, workers), n)
    q, r = divmod(n, parts)
    bounds = [i * q + min(i, r) for i in range(parts + 1)]
    return list(zip(bounds[:-1], bounds[1:]))


def run_chunked(n: int, workers: int, fn: Callable[[int, int], T]) -> List[T]:
    """Call ``fn(start, stop)`` per contiguous chunk, results in chunk order.

    Host-side helper kept for API parity; the device work it used to spread
    over threads is a single kernel launch here, so chunks run one after another.
    """
    return [fn(a, b) for a, b in chunk_ranges(n, workers)]


def run_tasks(tasks: List[Callable[[], T]], workers: int) -> List[T]:
    """Run thunks in submission order (launches are asynchronous already)."""
    return [task() for task in tasks]
