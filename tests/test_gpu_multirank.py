"""The multi-rank path executed on one B200 (-m gpu): two ranks (processes) on
cuda:0 in a gloo group each solve their contiguous shard of the targets with the
device IK-Beam (shard.solve_sharded, no collective in the solve), gather the
results through host memory (shard.gather_rows) and must reproduce the one-rank
solve bit for bit (results never depend on the rank count).
The kernels of the two ranks never wait on each other."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

TOTAL = 3001  # not a multiple of the world size
FIELDS = ("q", "cost", "history", "pos_error", "rot_error", "success")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch.distributed as dist

    import paper_2505_03728_b200 as k
    from paper_2505_03728_b200.benchmark import reachable_target_array
    from paper_2505_03728_b200.shard import solve_sharded
    from paper_2505_03728_b200.tasks import IkBeamSolver

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
    solver = IkBeamSolver(model, "flange", rng_seed=77)
    full = solve_sharded(solver, lambda s, e: reachable_target_array(model, "flange", e - s, 77, start=s), TOTAL)
    torch.cuda.synchronize()
    dist.barrier()
    q.put((rank, {f: full[f].cpu().numpy() for f in FIELDS}))
    dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_single_rank():
    import multiprocessing as mp

    import paper_2505_03728_b200 as k
    from paper_2505_03728_b200.benchmark import reachable_target_array
    from paper_2505_03728_b200.tasks import IkBeamSolver

    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, qu)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(qu.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    model = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
    one = IkBeamSolver(model, "flange", rng_seed=77).solve_device(
        reachable_target_array(model, "flange", TOTAL, 77)).cpu()
    for r in (0, 1):
        for f in FIELDS:
            assert np.array_equal(got[r][f], getattr(one, f)), (r, f)
