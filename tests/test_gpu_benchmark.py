"""Benchmark protocols on the device (run on a B200: -m gpu): the blocked
trajectory scenes reproduce the reference's _blocked_scene draws, and every
run_benchmark task returns the reference's result layout."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2505_03728_b200 as k  # noqa: E402
from conftest import robot_file  # noqa: E402
from paper_2505_03728_b200 import benchmark as bm  # noqa: E402


@pytest.fixture(scope="module")
def arm7():
    return k.load_robot(robot_file("arm7.urdf"), robot_file("arm7.sidecar.json"))


@pytest.mark.parametrize("i", [0, 1, 2])
def test_blocked_scene_matches_reference(arm7, golden_traj, i):
    pa, pb, world = bm._blocked_scene(arm7, "flange", 3000, i)
    g = lambda s: golden_traj[f"traj_scene{i}_{s}"]
    np.testing.assert_allclose(pa.as_array(), g("pa"), atol=1e-12)
    np.testing.assert_allclose(pb.as_array(), g("pb"), atol=1e-12)
    obs = g("obstacles")
    assert len(world.obstacles) == 1
    np.testing.assert_allclose(world.obstacles[0].center, obs[0, 1:4], atol=1e-9)
    assert world.obstacles[0].radius == obs[0, 7]


def test_run_benchmark_tasks(arm7):
    spec = bm.BenchmarkSpec(urdf=robot_file("arm7.urdf"), sidecar=robot_file("arm7.sidecar.json"), task="ik",
                            num_targets=256, rng_seed=77, batch_sizes=[1, 64], target_link="flange")
    ik = bm.run_benchmark(spec)
    assert set(ik["results"]["per_batch_size"]) == {"1", "64"}
    assert ik["results"]["per_batch_size"]["64"]["success_rate"] >= 0.99
    spec.task = "ik_mobile"
    mob = bm.run_benchmark(spec)
    assert mob["results"]["optimized"]["success_rate"] >= 0.99
    assert mob["results"]["static"]["success_rate"] < mob["results"]["optimized"]["success_rate"]
    spec.task, spec.num_targets, spec.rng_seed = "traj", 2, 3000
    traj = bm.run_benchmark(spec)
    assert traj["results"]["collision_free_rate"] == 1.0
    assert traj["results"]["min_signed_distance"] >= 0.0
    assert traj["results"]["worst_endpoint_pos_error"] < 0.005
    for r in (ik, mob, traj):
        assert bm.format_table(r).startswith("task: ")
