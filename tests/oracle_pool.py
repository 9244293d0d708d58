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


_JOB = {}


def _run_chunk(rng):
    lo, hi = rng
    kw = {k: (v[lo:hi] if k in _JOB["split"] else v) for k, v in _JOB["kw"].items()}
    return _JOB["fn"](*_JOB["args"], **kw)


def _concat(parts):
    import dataclasses

    import numpy as np

    p0 = parts[0]
    if p0 is None:
        return None
    if isinstance(p0, np.ndarray):
        return np.concatenate(parts, axis=0)
    if isinstance(p0, dict):
        return {k: _concat([p[k] for p in parts]) for k in p0}
    if dataclasses.is_dataclass(p0):
        return type(p0)(**{f.name: _concat([getattr(p, f.name) for p in parts]) for f in dataclasses.fields(p0)})
    return parts


def par_batched(fn, *args, split=(), **kw):
    """fn(*args, **kw) with the keyword arrays named in ``split`` cut into row chunks that run
    on a fork pool; array / dict / dataclass results are concatenated back in row order."""
    n = len(kw[split[0]])
    _JOB.update(fn=fn, args=args, kw=kw, split=set(split))
    return _concat(par_map(_run_chunk, chunks(n)))


def assert_fp64_beam_parity(h_dev, h_ref, diag, frac=0.95, gap=1e-12, tol=1e-6):
    """FP64 IK-Beam parity bar: >= ``frac`` of the targets keep their
    winner history within ``tol`` (relative) of the oracle's, and EVERY other target is an
    oracle near-tie -- an accept, prune or winner decision whose relative cost gap in the
    oracle run is below ``gap`` (oracle.ik_oracle.explain_divergence)."""
    import numpy as np

    from oracle import ik_oracle as o

    rel = np.abs(np.asarray(h_dev) - h_ref) / np.maximum(np.abs(h_ref), 1e-300)
    within = float(np.mean(rel.max(axis=1) < tol))
    ex = o.explain_divergence(h_dev, h_ref, diag, tol)
    assert within >= frac, (within, ex[:10])
    assert all(g < gap for _, _, _, g in ex), [e for e in ex if e[3] >= gap][:10]
    return within, ex
