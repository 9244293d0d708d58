import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")
GOLDEN_TRAJ = os.path.join(ROOT, "tests", "golden", "reference_golden_traj.npz")
ROBOTS = os.path.join(ROOT, "paper_2505_03728_b200", "robots")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


def robot_file(name):
    return os.path.join(ROBOTS, name)


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def golden_traj():
    return np.load(GOLDEN_TRAJ)


@pytest.fixture(scope="session")
def chains():
    from oracle import ik_oracle as o

    return {
        "arm7": o.load_chain_files(robot_file("arm7.urdf"), robot_file("arm7.sidecar.json")),
        "planar_2r": o.load_chain_files(robot_file("planar_2r.urdf"), robot_file("planar_2r.sidecar.json")),
        "arm7_gripper": o.load_chain_files(robot_file("arm7_gripper.urdf")),
    }


@pytest.fixture(scope="session")
def models():
    import paper_2505_03728_b200 as k

    return {
        "arm7": k.load_robot(robot_file("arm7.urdf"), robot_file("arm7.sidecar.json")),
        "planar_2r": k.load_robot(robot_file("planar_2r.urdf"), robot_file("planar_2r.sidecar.json")),
        "arm7_gripper": k.load_robot(robot_file("arm7_gripper.urdf")),
    }
