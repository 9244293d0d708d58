"""Run oracle work over host cores (test infrastructure; the oracle is the checker).

The NumPy oracle is single-threaded; distribution checks at 10^3..10^4
problems split the problems into chunks and map them over a fork pool.
Functions passed in must be module-level (picklable by reference).
"""

from __future__ import annotations

import os

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")


def workers() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def par_map(fn, items):
    """[fn(x) for x in items] over a fork pool (serial with one core)."""
    items = list(items)
    w = min(workers(), len(items))
    if w <= 1:
        return [fn(x) for x in items]
    import multiprocessing as mp

    with mp.get_context("fork").Pool(w) as pool:
        return pool.map(fn, items)


def chunks(n: int, parts: int | None = None):
    """Contiguous [lo, hi) ranges covering range(n)."""
    parts = max(1, min(n, parts or 2 * workers()))
    step = -(-n // parts)
    return [(lo, min(n, lo + step)) for lo in range(0, n, step)]
