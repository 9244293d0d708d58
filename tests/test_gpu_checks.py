"""Checking builds vs the normal build (-m gpu) -- the substitute for
compute-sanitizer, which is closed on this GPU pool (its runs left GPUs
needing a reset).  csrc/kop_check.cuh:

* poison: every kernel starts by filling its dynamic shared memory with 0xFF
  (NaN) bytes: a read of never-written shared memory (the stage-1 prune keys,
  the tree kernels' double-buffered pivot rows, the trajectory factor's band)
  would poison the outputs;
* jitter: a pseudo-random __nanosleep before and after every barrier
  (__syncthreads, __syncwarp, the trajectory solve's named barriers), so
  threads reach and leave barriers in a different order on every run: a
  missing barrier shows up as different outputs.

tools/kernel_smoke.py runs every kernel family (FP32 and FP64) at small sizes
and saves its outputs; each checking build must reproduce the normal build's
outputs bit for bit (NaN in the same places).  Out-of-bounds global writes are
checked separately with guard bands around the output buffers.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, lib, name):
    out = str(tmp_path / f"{name}.npz")
    env = dict(os.environ)
    if lib:
        env["KOP_LIB"] = lib
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "kernel_smoke.py"), "both", "--out", out],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    if name == "poison":  # positive control: the build is the poison build and its probe sees the poison
        assert "shared-memory poison" in r.stdout and "smem probe all-poison: True" in r.stdout, r.stdout[:2000]
    if name == "jitter":
        assert "barrier jitter" in r.stdout, r.stdout[:2000]
    return dict(np.load(out))


@pytest.fixture(scope="module")
def normal(tmp_path_factory):
    return _run(tmp_path_factory.mktemp("normal"), None, "normal")


@pytest.mark.parametrize("variant", ["poison", "jitter"])
def test_checking_build_reproduces_normal_build(tmp_path, normal, variant):
    from paper_2505_03728_b200 import _build

    lib = _build.variant_lib(variant)
    if not os.path.exists(lib):  # build it here (nvcc is on the box)
        _build.build(variant=variant)
    got = _run(tmp_path, lib, variant)
    assert set(got) == set(normal)
    bad = [key for key in normal if normal[key].shape != got[key].shape
           or not np.array_equal(normal[key], got[key], equal_nan=True)]
    assert not bad, bad
    assert len(normal) > 100  # every family saved its outputs


def test_output_guard_bands(models):
    """Outputs written into the middle of a canary-filled buffer: nothing outside the
    rows of the batch changes (out-of-bounds global writes)."""
    import paper_2505_03728_b200 as k
    from paper_2505_03728_b200.benchmark import reachable_target_array
    from paper_2505_03728_b200.tasks import BeamBatch, IkBeamSolver

    m = models["arm7"]
    for b, seeds, keep in ((7, 64, 4), (33, 37, 7)):
        tg = reachable_target_array(m, "flange", b, 5)
        for prec in ("fp32", "fp64"):
            s = IkBeamSolver(m, "flange", seeds=seeds, keep=keep, rng_seed=5, precision=prec)
            pad = 64

            def guarded(shape, dtype=torch.float64):
                full = torch.full((b + 2 * pad,) + shape, float("nan") if dtype.is_floating_point else 77,
                                  dtype=dtype, device="cuda")
                return full, full[pad:pad + b]
            bufs = {f: guarded(sh) for f, sh in (("q", (7,)), ("cost", ()), ("history", (17,)), ("pos_error", ()),
                                                  ("rot_error", ()))}
            bufs["success"] = guarded((), torch.uint8)
            out = BeamBatch(*(bufs[f][1] for f in ("q", "cost", "history", "pos_error", "rot_error", "success")))
            s.solve_device(tg, out)
            torch.cuda.synchronize()
            for f, (full, _) in bufs.items():
                head, tail = full[:pad], full[pad + b:]
                if full.dtype.is_floating_point:
                    assert torch.isnan(head).all() and torch.isnan(tail).all(), (f, prec)
                else:
                    assert (head == 77).all() and (tail == 77).all(), (f, prec)
            assert not torch.isnan(out.cost).any()
