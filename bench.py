#!/usr/bin/env python
"""Batched Panda IK-Beam throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--quick]

One step = one IK-Beam pass (64 seeds, 6 LM steps, keep 4, 10 more steps;
tasks.py:119-161) over a batch of synthetic reachable Panda targets
(benchmark.py:83-93, rng 77) resident in HBM.  Weak scaling: every rank
solves its own ``--batch`` targets (distinct Philox index ranges); there is
no collective in the solve -- the ranks only meet for the barrier and the
max-over-ranks time.

Prints ONE JSON line on rank 0.  Beside the headline (device value, e2e,
roofline, clocks, cpu_baseline) the same line carries every other number
north_star names: ``batch_sweep`` (1 .. 1M targets,
device and end to end), ``fp64`` (the headline config in FP64) and
``configs`` (configs 3 / 4 / 5 and the mobile base, each with its
SURVEY 8(d)-convention roofline, success / termination distributions and
the CPU port of the reference on all host cores).
"""

from __future__ import annotations

import os

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse
import json
import math
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batched IK solves/sec (Panda, device-timed) at 1/2/4/8 B200; pos/rot error"
SEEDS, PRUNE, TOTAL, KEEP = 64, 6, 16, 4
RNG_SEED = 77
NOMINAL_FP32_FLOP_PER_CLK_SM = 256  # 128 FP32 lanes x FMA
NOMINAL_FP64_FLOP_PER_CLK_SM = 128  # 64 FP64 lanes x FMA


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=1_000_000, help="targets per GPU per step")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU-baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="headline only (no sweep / fp64 / configs)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N>1 (gloo: several ranks on one GPU, host-staged)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# SURVEY.md 8(d) algorithmic flop convention (FMA = 2 flops; sqrt / div /
# transcendental = 1).  The Panda lane-step reproduces the survey's table term
# by term (4,535 flops); configs 3-5 apply the same per-term rules to their
# own shapes.  These constants, not executed instruction counts, are what every
# roofline.achieved below is built from.
# ---------------------------------------------------------------------------
FK_REVOLUTE, FK_FIXED = 124, 61          # per joint: frame compose + motion quaternion
GEOM_JAC_PER_COL = 12                    # axis x (p - anchor) per ancestor joint
QUAT_TO_MAT, POSE_COMPOSE, SE3_LOG, JR_INV = 30, 61, 110, 560
BODY_ROT_PER_COL = 36                    # R^T (3x3) . J_lin / J_ang per column
JRINV_TIMES_J_PER_COL = 54               # block-triangular 6x6 . 6-column
CAND_BOOKKEEPING = 57                    # q + delta, accept test, damping update, history


def chol_flops(n: int) -> float:
    """n^3/3 FMAs + two triangular solves (n^2 FMAs each) + n sqrt/div: 340 at n = 7."""
    return 2.0 * n ** 3 / 3.0 + 2.0 * n * n + 2.0 * n


def fk_flops(n_revolute: int, n_fixed: int) -> float:
    return FK_REVOLUTE * n_revolute + FK_FIXED * n_fixed


def pose_lane_step(fk: float, n: int, nks, extra_eval=0.0, extra_jac=0.0, extra_rows=0):
    """One beam.py lane step (J-eval at q, damped solve, candidate eval at q + delta)
    over K pose blocks with nks[k] ancestor columns, limit + rest rows (2n), and
    optional extra dense rows (collision) whose evaluation / Jacobian costs are given.
    Returns (lane_step_flops, lane_init_flops)."""
    K = len(nks)
    m = 6 * K + 2 * n + extra_rows
    pose_eval = K * (POSE_COMPOSE + SE3_LOG)
    jac = (sum(GEOM_JAC_PER_COL * c + BODY_ROT_PER_COL * c + JRINV_TIMES_J_PER_COL * c for c in nks)
           + K * (QUAT_TO_MAT + JR_INV))
    weighting = sum(6 * c for c in nks) + m
    jtj = sum(6 * c * (c + 1) for c in nks) + 2 * (2 * n)  # pose rows dense, limit / rest rows diagonal;
    # the J^T J / J^T r share of extra (collision) rows is part of extra_jac
    jtr = sum(12 * c for c in nks) + 4 * n
    damping = 3 * n
    cand = fk + pose_eval + 4 * n + 2 * m + n + CAND_BOOKKEEPING + extra_eval
    step = fk + pose_eval + jac + weighting + jtj + jtr + damping + chol_flops(n) + cand + extra_eval + extra_jac
    init = fk + pose_eval + 4 * n + 2 * m + extra_eval
    return step, init


def panda_counts():
    """Panda (arm7): 7 revolute + 1 fixed joint, one end effector over all 7 columns."""
    return dict(fk=fk_flops(7, 1), n=7, nks=[7])


def beam_flops(lane_step, lane_init, final_err=1.1e3, seeds=SEEDS, prune=PRUNE, total=TOTAL, keep=KEEP, n_ee=1):
    """IK-Beam solve: seeds x (init + prune steps) + keep x (total - prune) steps + final errors.
    Returns (per_solve, stage1_per_target)."""
    s1 = seeds * (lane_init + prune * lane_step)
    s2 = keep * (total - prune) * lane_step + n_ee * final_err
    return s1 + s2, s1


PANDA_STEP, PANDA_INIT = pose_lane_step(**panda_counts())          # 4,535 / 1,168
FLOP_PER_SOLVE, STAGE1_FLOP_PER_TARGET = beam_flops(PANDA_STEP, PANDA_INIT)  # 2.0 M / 1.82 M
STAGE2_FLOP_PER_TARGET = FLOP_PER_SOLVE - STAGE1_FLOP_PER_TARGET

# collision row costs (per sphere term / per row), same counting rules
SPHERE_CENTRE = 30                       # quaternion rotate + translate
DIST = {"sphere": 11, "capsule": 30, "halfspace": 6}
SOFTMIN_TERM, SOFTMIN_ROW, ACTIVATION_ROW = 5, 6, 4
POINT_JAC_TERM = GEOM_JAC_PER_COL + 6 + 2  # per column: point Jacobian, grad . J, soft-min weight


def collision_extra(n_spheres, world_terms, self_terms, rows, ancestors_per_row, term_cols):
    """(extra_eval, extra_jac, rows) of a collision row stack: world_terms / self_terms are lists of
    distance kinds; term_cols the ancestor columns of each term's sphere(s)."""
    ev = SPHERE_CENTRE * n_spheres + sum(DIST[k] for k in world_terms) + DIST["sphere"] * len(self_terms)
    ev += SOFTMIN_TERM * (len(world_terms) + len(self_terms)) + (SOFTMIN_ROW + ACTIVATION_ROW) * rows
    jac = sum(POINT_JAC_TERM * c for c in term_cols)
    jac += sum(2 * c + c * (c + 1) + 2 * c for c in ancestors_per_row)  # act' scale + J^T J + J^T r per row
    return ev, jac, rows


# ---------------------------------------------------------------------------
# CPU reference arm: the oracle port of kinoptik's IK-Beam, one target per
# call exactly like the reference's solve_ik_beam (benchmark.py:136-151)
# ---------------------------------------------------------------------------
_W = {}


def _chain7():
    from oracle import ik_oracle as o

    if "ch" not in _W:
        robots = os.path.join(ROOT, "paper_2505_03728_b200", "robots")
        _W["ch"] = o.load_chain_files(os.path.join(robots, "arm7.urdf"), os.path.join(robots, "arm7.sidecar.json"))
    return _W["ch"]


def _cpu_worker_init():
    from oracle import ik_oracle as o

    ch = _chain7()
    _W["o"] = o
    _W["seeds"] = o.sample_seeds(ch, SEEDS, RNG_SEED)
    _W["link"] = ch.link("flange")


def _cpu_solve(chunk):
    o, ch = _W["o"], _W["ch"]
    out = []
    for t in chunk:
        r = o.ik_beam(ch, _W["link"], t[None, :4], t[None, 4:], _W["seeds"])
        out.append((float(r.pos_err[0]), float(r.rot_err[0]), bool(r.success[0])))
    return out


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class CpuArm:
    """Pool over every host core; each worker solves whole targets serially."""

    def __init__(self, targets: np.ndarray):
        import multiprocessing as mp

        self.cores = os.cpu_count() or 1
        self.targets = targets
        self.pool = mp.get_context("fork").Pool(self.cores, initializer=_cpu_worker_init)
        # single-core rate (also sizes the bounded samples): 6 targets on this process
        _cpu_worker_init()
        _cpu_solve(targets[:1])
        t0 = time.perf_counter()
        _cpu_solve(targets[1:7])
        self.t1 = (time.perf_counter() - t0) / 6

    def run(self, count: int, offset: int = 0):
        idx = (offset + np.arange(count)) % len(self.targets)
        chunks = np.array_split(self.targets[idx], self.cores * 2)
        t0 = time.perf_counter()
        res = [r for part in self.pool.map(_cpu_solve, [c for c in chunks if len(c)]) for r in part]
        return count / (time.perf_counter() - t0), res

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_targets(n: int) -> np.ndarray:
    """The workload's first n targets, generated on the host by the oracle (no GPU)."""
    from oracle import ik_oracle as o

    ch = _chain7()
    tq, tt, _ = o.reachable_targets(ch, ch.link("flange"), n, RNG_SEED)
    return np.concatenate([tq, tt], axis=1)


def run_reference(args, rank, world):
    if rank != 0:
        return
    targets = cpu_targets(4096)
    arm = CpuArm(targets)
    per_step = max(arm.cores, int(round(4.0 / arm.t1)) * arm.cores)
    for w in range(args.warmup):
        arm.run(arm.cores, offset=w * arm.cores)
    res = []
    t0 = time.perf_counter()
    for s in range(args.steps):
        _, out = arm.run(per_step, offset=s * per_step)
        res += out
    wall = time.perf_counter() - t0
    arm.close()
    value = float(args.steps * per_step / wall)
    sample = (f"{per_step} targets per step (the first {len(targets)} targets of the rng-77 workload, cycled), "
              f"solved one target per call in float64 by the oracle port of kinoptik IK-Beam, multiprocessing "
              f"over {arm.cores} host cores ({cpu_model()}); the reference solves targets one at a time, so its "
              f"per-target cost does not depend on the batch size")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        # the same workload config as our arm; what each reference step actually ran is `ran`
        "data": "synthetic", "config": workload_config(args.batch, args.precision),
        "ran": {"targets_per_step": per_step, "precision": "fp64", "target_pool": len(targets),
                "workload_batch_named_in_config": args.batch},
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": arm.cores, "kind": "port",
                         "sample": sample, "single_core_value": 1.0 / arm.t1, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "accuracy": accuracy(np.array([r[0] for r in res]), np.array([r[1] for r in res]),
                             np.array([r[2] for r in res])),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def workload_config(batch, precision):
    return {
        "workload": f"Panda (arm7.urdf, EE flange) IK-Beam over {batch} synthetic reachable targets per GPU "
                    f"(benchmark.py:83-93, rng {RNG_SEED}); 64 seeds, 6 LM steps, keep 4, 10 more steps",
        "targets_per_gpu": batch, "seeds": SEEDS, "lm_steps": f"{PRUNE}+{TOTAL - PRUNE}", "keep": KEEP,
        "precision": precision, "weights": "CostWeights() defaults (50, 10, 100, 0.01)",
        "l2": f"flushed between timed steps (512 MiB write); inputs {batch * 56 / 1e6:.0f} MB/GPU",
        "parallelism": "targets sharded, no collective in the solve",
    }


def accuracy(pos, rot, succ):
    return {"success_rate": float(np.mean(succ)), "pos_err_p50_m": float(np.percentile(pos, 50)),
            "pos_err_p98_m": float(np.percentile(pos, 98)), "rot_err_p50_rad": float(np.percentile(rot, 50)),
            "rot_err_p98_rad": float(np.percentile(rot, 98))}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms from the start of the
    warm-up to the end of the timed region (all of it under load)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.rows, self.proc = [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 8 for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def fma_peak(torch, lib, fp64=False):
    """Measured FMA-pipe peak (TFLOP/s): immediate-operand FFMA (DFMA) chains, all SMs."""
    import ctypes as C

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    dt = torch.float64 if fp64 else torch.float32
    fn = lib.kop_dfma_peak_kernel if fp64 else lib.kop_fma_peak_kernel
    sink = torch.zeros(4096, device="cuda", dtype=dt)
    flops = C.c_double()
    blocks, threads, iters = sms * 8, 256, (5000 if fp64 else 20000)
    st = torch.cuda.current_stream().cuda_stream
    fn(blocks, threads, 200, sink.data_ptr(), C.byref(flops), st)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(blocks, threads, iters, sink.data_ptr(), C.byref(flops), st)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, flops.value / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best, sms


def load_traffic():
    path = os.path.join(ROOT, "profiles", "stage1_dram_per_launch.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("bytes_per_launch"), d.get("batch")
    except (OSError, ValueError):
        return None, None


def load_share(name):
    """Dominant-kernel share of a workload's device time from a committed ncu launch list summary."""
    path = os.path.join(ROOT, "profiles", "r02_kernel_shares.json")
    try:
        with open(path) as f:
            return json.load(f).get(name)
    except (OSError, ValueError):
        return None


def device_time(torch, fn, reps, flush=None):
    """Per-call device times (ms) with CUDA events on the current stream; L2 flushed before each call."""
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return out


def roof(flops_per_unit, units_per_s, peak, nominal, what, **extra):
    ach = flops_per_unit * units_per_s / 1e12
    d = {"achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak, "frac_of_nominal": ach / nominal,
         "nominal_peak": nominal, "flops_per_unit": flops_per_unit, "basis": what}
    d.update(extra)
    return d


# ---------------------------------------------------------------------------
# CPU legs of the widened configs: the oracle port on all host cores
# ---------------------------------------------------------------------------
_CFG = {}


def _cfg_worker(job):
    kind, payload = job
    from oracle import collision_oracle as co, ik_oracle as o, traj_oracle as to, tree_oracle as tro

    if kind == "col_beam":
        return co.ik_beam_collision(_CFG["ch"], _CFG["sp"], _CFG["obs"], _CFG["fl"], payload[None, :4],
                                    payload[None, 4:], _CFG["seeds"], co.CollisionCosts()).success[0]
    if kind == "col_lm":
        q, cost, hist, it, term = co.solve_lm(_CFG["ch"], _CFG["sp"], _CFG["obs"], _CFG["fl"], payload[:4],
                                              payload[4:], _CFG["rest"].copy(), co.CollisionCosts())
        return it
    if kind == "tree_beam":
        r = tro.multi_ee_beam(_CFG["chh"], _CFG["links"], payload[None, :, :4], payload[None, :, 4:],
                              _CFG["seeds_h"], [50.0] * 4, [10.0] * 4)
        return bool(r["success"][0])
    if kind == "tree_lm":
        poses = [(l, payload[j, :4], payload[j, 4:], 50.0, 10.0) for j, l in enumerate(_CFG["links"])]
        tro.solve_multi_pose(_CFG["chh"], poses, _CFG["rest_h"].copy())
        return True
    if kind == "traj":
        qa, qb, mid = payload
        tc = to.TrajCosts(timesteps=64)
        r = to.solve_traj(_CFG["ch"], _CFG["sp"], [co.sphere(mid, 0.07)], to.straight_line(qa, qb, 64), qa, qb,
                          tc, _CFG["vlim"])
        return r[3]
    if kind == "mobile":
        return bool(o.ik_beam(_CFG["ch"], _CFG["fl"], payload[None, :4], payload[None, 4:], _CFG["seeds"],
                              use_base=True).success[0])
    raise ValueError(kind)


def cpu_leg(kind, payloads, unit, what):
    """Time the oracle port on every host core over one bounded sample (one item per core)."""
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    items = [(kind, p) for p in payloads[:cores]]
    with mp.get_context("fork").Pool(len(items)) as pool:
        pool.map(_cfg_worker, items[:1])  # import / warm the workers' oracle modules
        t0 = time.perf_counter()
        pool.map(_cfg_worker, items, chunksize=1)
        wall = time.perf_counter() - t0
    return {"value": len(items) / wall, "unit": unit, "cores": len(items), "kind": "port",
            "sample": f"{len(items)} {what} of this workload, one per host core, oracle port of kinoptik "
                      f"(float64 NumPy), multiprocessing ({cpu_model()})"}


def _setup_cfg_oracles(model, hum, ees):
    from oracle import collision_oracle as co, ik_oracle as o, traj_oracle as to

    import paper_2505_03728_b200 as k

    ch = _chain7()
    _CFG["ch"] = ch
    _CFG["sp"] = co.load_spheres_files(ch, k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
    _CFG["obs"] = [co.sphere([0.45, 0.1, 0.55], 0.12), co.capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                   co.halfspace([0.0, 0.0, 1.0], -0.3)]
    _CFG["fl"] = ch.link("flange")
    _CFG["seeds"] = o.sample_seeds(ch, SEEDS, RNG_SEED)
    _CFG["rest"] = model.rest_pose
    _CFG["vlim"] = model.velocity_limits
    chh = o.load_chain_files(k.robot_path("humanoid29.urdf"))
    _CFG["chh"] = chh
    _CFG["links"] = [chh.link(e) for e in ees]
    _CFG["seeds_h"] = o.sample_seeds(chh, SEEDS, 0)
    _CFG["rest_h"] = hum.rest_pose


# ---------------------------------------------------------------------------
# extended lines: batch sweep, FP64 headline, configs 3-5 and mobile base
# ---------------------------------------------------------------------------
def ancestors_columns(model, link):
    """Actuated joints on the root -> link path (the columns of that link's pose block)."""
    parent_joint = {j.child_link: j for j in model.joints}
    cols, name = 0, link
    while name in parent_joint:
        j = parent_joint[name]
        if j.kind != "fixed" and j.mimic is None:
            cols += 1
        name = j.parent_link
    return cols


def run_sweep(torch, k, model, solver_for, flush, peak, nominal):
    from paper_2505_03728_b200.benchmark import reachable_target_array

    out = []
    tg_all = reachable_target_array(model, "flange", 1_000_000, RNG_SEED)
    solver = solver_for("fp32")
    for b in (1, 1000, 10_000, 100_000, 1_000_000):
        tg = tg_all[:b].contiguous()
        dev_out = solver.alloc_outputs(b)
        reps = 20 if b <= 10_000 else (5 if b <= 100_000 else 3)
        t = device_time(torch, lambda: solver.solve_device(tg, dev_out), reps, flush)
        host_t = tg.cpu().pin_memory()
        host_out = solver.alloc_host_outputs(b)
        te = device_time(torch, lambda: solver.solve_host(host_t, host_out), reps, flush)
        dev_ms, e2e_ms = float(np.median(t)), float(np.median(te))
        out.append({"targets": b, "device_ms": dev_ms, "device_solves_per_s": b / dev_ms * 1e3,
                    "e2e_ms": e2e_ms, "e2e_solves_per_s": b / e2e_ms * 1e3,
                    "solve_frac": FLOP_PER_SOLVE * b / (dev_ms * 1e-3) / 1e12 / peak,
                    "e2e_api": "IkBeamSolver.solve_host -> C ABI kop_ik_beam_host, pinned host in/out",
                    "reps_median_of": reps})
    return out


def hbm_peak():
    """(GB/s, source): MEASURED_PEAKS.json's copy bandwidth, else the profiling guide's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def run_fk(torch, model, flush, B=1_000_000):
    """fk_arrays (robot.py:404-448) on the device: B configurations in, every link frame and
    every joint anchor / axis out (FP64 outputs) -- HBM-write-bound, bytes roofline."""
    from paper_2505_03728_b200 import _device as dv
    from paper_2505_03728_b200.robot import fk_arrays_device

    q = dv.to_dev(np.random.default_rng(3).uniform(model.lower_limits, model.upper_limits, (B, model.actuated_count)))
    nl, nj, n = len(model.link_names), len(model.joints), model.actuated_count
    byts = B * 8 * (n + 7 * nl + 6 * nj)
    peak, src = hbm_peak()
    out = {"workload": f"fk_arrays of {B} Panda configurations (all {nl} link frames + {nj} joint anchors / axes, "
                       "float64 outputs)", "bytes_per_call": byts}
    for prec in ("fp64", "fp32"):
        ms = float(np.median(device_time(torch, lambda: fk_arrays_device(model, q, prec), 5, flush)))
        gbs = byts / (ms * 1e-3) / 1e9
        out[prec] = {"ms": ms, "configs_per_s": B / ms * 1e3,
                     "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                                  "peak_source": src, "kernel": "k_fk_tree"}}
    return out


def run_fp64_headline(torch, model, solver_for, flush, B, peak64, nominal64):
    from paper_2505_03728_b200.benchmark import reachable_target_array

    tg = reachable_target_array(model, "flange", B, RNG_SEED)
    s = solver_for("fp64")
    o = s.alloc_outputs(B)
    t1 = device_time(torch, lambda: s.solve_device(tg, o, stages=1), 2, flush)
    t2 = device_time(torch, lambda: s.solve_device(tg, o, stages=2), 2, flush)
    s1, ms = float(np.mean(t1)), float(np.mean(t1) + np.mean(t2))
    r = o.cpu()
    return {"precision": "fp64", "targets": B, "ms_per_step": ms, "value": B / ms * 1e3, "unit": "solves/s",
            "roofline": roof(STAGE1_FLOP_PER_TARGET, B / s1 * 1e3, peak64, nominal64,
                             "k_beam_stage1 in FP64, SURVEY 8(d) constants, vs the live DFMA peak", stage1_ms=s1),
            "accuracy": accuracy(r.pos_error, r.rot_error, r.success)}


def run_configs(torch, k, model, flush, peaks, nominals, cpu=True):
    """Configs 3 / 4 / 5 (BASELINE.json) and the mobile base, FP32 and FP64."""
    import ctypes as C

    from paper_2505_03728_b200 import _device as dv
    from paper_2505_03728_b200._lib import check, lib
    from paper_2505_03728_b200.benchmark import disk_translations, reachable_target_array
    from paper_2505_03728_b200.robot import link_poses_device
    from paper_2505_03728_b200.solver import _options, plan
    from paper_2505_03728_b200.tasks import IkBeamSolver

    out = {}
    finals = {}
    legs = []  # CPU legs run after every device timing: forked pools perturb the host enqueue of the timed calls
    demo = k.WorldModel([k.Sphere([0.45, 0.1, 0.55], 0.12), k.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                         k.HalfSpace([0.0, 0.0, 1.0], -0.3)])
    hum = k.load_robot(k.robot_path("humanoid29.urdf"))
    ees = ["left_hand", "right_hand", "left_foot", "right_foot"]
    if cpu:
        _setup_cfg_oracles(model, hum, ees)

    # ---- config 4: collision IK-Beam, Panda, demo world (sphere + capsule + half-space) + self pairs ----
    sl = [nm for nm in model.link_names if model.collision_spheres.get(nm)]
    nsph = {nm: len(model.collision_spheres[nm]) for nm in sl}
    anc = {nm: ancestors_columns(model, nm) for nm in sl}
    kinds = ["sphere", "capsule", "halfspace"]
    world_terms = [kd for nm in sl for kd in kinds for _ in range(nsph[nm])]
    pairs = model.self_collision_pairs
    self_terms = [0 for a, b in pairs for _ in range(nsph[a] * nsph[b])]
    term_cols = [anc[nm] for nm in sl for _ in kinds for _ in range(nsph[nm])] + \
                [anc[a] + anc[b] for a, b in pairs for _ in range(nsph[a] * nsph[b])]
    rows_anc = [anc[nm] for nm in sl for _ in kinds] + [max(anc[a], anc[b]) for a, b in pairs]
    ev, jac, rows = collision_extra(sum(nsph.values()), world_terms, self_terms, len(rows_anc), rows_anc, term_cols)
    c4_step, c4_init = pose_lane_step(**panda_counts(), extra_eval=ev, extra_jac=jac, extra_rows=rows)
    c4_solve, c4_s1 = beam_flops(c4_step, c4_init)
    B4 = 100_000
    tg4 = reachable_target_array(model, "flange", B4, RNG_SEED)
    c4 = {"workload": "config 4: Panda collision IK-Beam, demo world (sphere + capsule + half-space) + 12 self pairs, "
                      f"{B4} targets, 64 seeds, 6+10 steps, keep 4",
          "flop_convention": {"lane_step": c4_step, "lane_init": c4_init, "per_solve": c4_solve,
                              "collision_rows": rows, "sphere_terms": len(world_terms) + len(self_terms)}}
    for prec in ("fp32", "fp64"):
        s = IkBeamSolver(model, "flange", rng_seed=RNG_SEED, precision=prec, world=demo, self_collision=True)
        o4 = s.alloc_outputs(B4)
        t = device_time(torch, lambda: s.solve_device(tg4, o4), 3, flush)
        ms = float(np.median(t))
        share = load_share(f"config4_{prec}")
        c4[prec] = {"ms": ms, "value": B4 / ms * 1e3, "unit": "solves/s",
                    "success_rate": float(o4.success.float().mean()),
                    "roofline": roof(c4_solve, B4 / ms * 1e3, peaks[prec], nominals[prec],
                                     "whole solve (all kernels), SURVEY 8(d) rules",
                                     dominant_kernel="k_col_beam_stage1", dominant_share=share,
                                     dominant_frac=(c4_s1 * B4 / (share * ms * 1e-3) / 1e12 / peaks[prec])
                                     if share else None)}
    if cpu:
        legs.append((c4, ("col_beam", list(tg4[:64].cpu().numpy()), "solves/s", "targets")))
    out["config4_collision_ik_beam"] = c4

    # ---- config 4, solver.solve flavour: the generic LM (k_col_solve) on the same stack ----
    prob = k.Problem(k.VariableSet.of(q=model.rest_pose.copy()), [
        k.pose_cost(model, "q", "flange", k.Transform3.identity(), position_weight=50, orientation_weight=10),
        k.limit_cost(model, "q", weight=100), k.rest_cost("q", model.rest_pose, weight=0.01),
        k.world_collision_cost(model, "q", demo, weight=20), k.self_collision_cost(model, "q", weight=5)])
    p = plan(prob)
    lm_iter = c4_step  # per accepted iteration: J-eval + normal equations + solve + candidate, same terms
    c4lm = {"workload": f"config 4, solver.solve semantics (generic LM, rejection loop): {B4} problems, q0 = rest pose"}
    for prec in ("fp32", "fp64"):
        opts = _options(k.SolveOptions(precision=prec))
        q0 = dv.to_dev(np.tile(model.rest_pose, (B4, 1)))
        outs = [dv.empty((B4, 7)), dv.empty(B4), dv.empty(B4), None,
                torch.empty(B4, dtype=torch.int32, device="cuda"), torch.empty(B4, dtype=torch.int32, device="cuda")]

        def run_lm():
            check(lib().kop_lm_solve(model._handle, 8, C.byref(p.costs), C.byref(opts), dv.ptr(tg4), dv.ptr(q0), B4,
                                     *(dv.ptr(x) for x in outs), dv.stream_handle()), "kop_lm_solve")
        reps = device_time(torch, run_lm, 5, flush)
        ms = float(np.median(reps))
        it = float(outs[4].float().mean())
        finals[("c4", prec)] = outs[1].cpu().numpy()
        c4lm[prec] = {"ms": ms, "rep_ms": [round(x, 3) for x in reps], "value": B4 / ms * 1e3, "unit": "solves/s",
                      "mean_iterations": it,
                      "terminations": torch.bincount(outs[5].long(), minlength=7).tolist(),
                      "roofline": roof(lm_iter * it, B4 / ms * 1e3, peaks[prec], nominals[prec],
                                       "k_col_solve (single kernel): accepted iterations x lane-step constant")}
    if cpu:
        legs.append((c4lm, ("col_lm", list(tg4[:64].cpu().numpy()), "solves/s", "problems")))
    c4lm["fp32_vs_fp64_final_cost"] = final_cost_agreement(finals[("c4", "fp32")], finals[("c4", "fp64")])
    out["config4_generic_lm"] = c4lm

    # ---- config 3: humanoid multi-EE IK-Beam and solver.solve flavour ----
    nh = hum.actuated_count
    nfix = sum(1 for j in hum.joints if j.kind == "fixed")
    hcounts = dict(fk=fk_flops(nh, nfix), n=nh, nks=[ancestors_columns(hum, e) for e in ees])
    c3_step, c3_init = pose_lane_step(**hcounts)
    c3_solve, c3_s1 = beam_flops(c3_step, c3_init, n_ee=len(ees))
    B3 = 100_000
    qt = dv.to_dev(np.random.default_rng(29).uniform(hum.lower_limits, hum.upper_limits, (B3, nh)))
    tgh = torch.stack([link_poses_device(hum, qt, e) for e in ees], dim=1).contiguous()
    c3 = {"workload": f"config 3: humanoid (n={nh}) multi-EE IK-Beam, 4 end effectors (hands, feet) + limit + rest, "
                      f"{B3} targets, 64 seeds, 6+10 steps, keep 4",
          "flop_convention": {"lane_step": c3_step, "lane_init": c3_init, "per_solve": c3_solve,
                              "ee_columns": hcounts["nks"]}}
    for prec in ("fp32", "fp64"):
        box = {}

        def run_tb():
            box["r"] = k.solve_ik_beam_multi(hum, ees, tgh, precision=prec, device_out=True)
        ms = float(np.median(device_time(torch, run_tb, 3, flush)))
        share = load_share(f"config3_{prec}")
        c3[prec] = {"ms": ms, "value": B3 / ms * 1e3, "unit": "solves/s",
                    "success_rate": float(box["r"].success.float().mean()),
                    "roofline": roof(c3_solve, B3 / ms * 1e3, peaks[prec], nominals[prec],
                                     "whole solve (all kernels), SURVEY 8(d) rules",
                                     dominant_kernel="k_tree_beam_stage1", dominant_share=share,
                                     dominant_frac=(c3_s1 * B3 / (share * ms * 1e-3) / 1e12 / peaks[prec])
                                     if share else None)}
    if cpu:
        legs.append((c3, ("tree_beam", list(tgh[:64].cpu().numpy()), "solves/s", "target sets")))
    out["config3_humanoid_ik_beam"] = c3

    w0 = k.CostWeights()
    hprob = k.Problem(k.VariableSet.of(q=hum.rest_pose.copy()),
                      [k.pose_cost(hum, "q", e, k.Transform3.identity(), position_weight=w0.pose_position,
                                   orientation_weight=w0.pose_orientation) for e in ees]
                      + [k.limit_cost(hum, "q", weight=w0.limit), k.rest_cost("q", hum.rest_pose, weight=w0.rest)])
    hp = plan(hprob)
    c3lm = {"workload": f"config 3, solver.solve semantics: {B3} humanoid problems, 4 pose costs + limit + rest, "
                        "q0 = rest pose"}
    for prec in ("fp32", "fp64"):
        opts = _options(k.SolveOptions(precision=prec))
        q0 = dv.to_dev(np.tile(hum.rest_pose, (B3, 1)))
        outs = [dv.empty((B3, nh)), dv.empty(B3), dv.empty(B3), None,
                torch.empty(B3, dtype=torch.int32, device="cuda"), torch.empty(B3, dtype=torch.int32, device="cuda")]

        def run_tl():
            check(lib().kop_multi_pose_solve(hum._handle, C.byref(hp.costs), C.byref(opts), dv.ptr(tgh), dv.ptr(q0),
                                             B3, *(dv.ptr(x) for x in outs), dv.stream_handle()), "tree")
        ms = float(np.median(device_time(torch, run_tl, 3, flush)))
        it = float(outs[4].float().mean())
        finals[("c3", prec)] = outs[1].cpu().numpy()
        c3lm[prec] = {"ms": ms, "value": B3 / ms * 1e3, "unit": "solves/s", "mean_iterations": it,
                      "terminations": torch.bincount(outs[5].long(), minlength=7).tolist(),
                      "final_cost_p50": float(outs[1].median()),
                      "roofline": roof(c3_step * it, B3 / ms * 1e3, peaks[prec], nominals[prec],
                                       "k_tree_solve (single kernel): accepted iterations x lane-step constant")}
    if cpu:
        legs.append((c3lm, ("tree_lm", list(tgh[:64].cpu().numpy()), "solves/s", "problems")))
    c3lm["fp32_vs_fp64_final_cost"] = final_cost_agreement(finals[("c3", "fp32")], finals[("c3", "fp64")])
    out["config3_generic_lm"] = c3lm

    # ---- config 5: trajectories, T = 64, one r = 0.07 sphere at the FK of the joint-space midpoint ----
    NT, TT, n = 10_000, 64, 7
    rng = np.random.default_rng(5)
    qa = rng.uniform(model.lower_limits, model.upper_limits, (NT, n))
    qb = rng.uniform(model.lower_limits, model.upper_limits, (NT, n))
    mid = link_poses_device(model, dv.to_dev(0.5 * (qa + qb)), "flange").cpu().numpy()[:, 4:7]
    obs = np.zeros((NT, 1, 8))
    obs[:, 0, 1:4] = mid
    obs[:, 0, 7] = 0.07
    anchors, obsd = dv.to_dev(np.stack([qa, qb], axis=1)), dv.to_dev(obs)
    c5_iter = traj_iteration_flops(model, TT, anc, nsph, pairs)
    c5 = {"workload": f"config 5: Panda trajectories, T={TT}, dt 0.1, plan_trajectory cost set, one sphere r=0.07 at "
                      f"the joint-space midpoint, {NT} trajectories, solver.solve semantics (max 150 iterations)",
          "flop_convention": {"per_accepted_iteration": c5_iter}}
    for prec in ("fp64", "fp32"):
        pl = k.TrajectoryPlanner(model, "flange", timesteps=TT, precision=prec)
        res = {}

        def run_tr():
            res.update(pl.solve_anchored_device(anchors, obsd, 1, history=False))
        ms = float(np.median(device_time(torch, run_tr, 3, flush)))
        rep = k.trajectory.trajectory_signed_distances_batch(model, res["qs"], obsd, 1, "flange")
        free = float((torch.minimum(rep["min_static"], rep["min_swept"]) >= 0).float().mean())
        it = float(res["iterations"].float().mean())
        finals[("c5", prec)] = res["cost"].cpu().numpy()
        c5[prec] = {"ms": ms, "value": NT / ms * 1e3, "unit": "trajectories/s", "mean_iterations": it,
                    "lm_iterations_per_s": it * NT / ms * 1e3, "collision_free_rate": free,
                    "terminations": torch.bincount(res["termination"].long(), minlength=7).tolist(),
                    "roofline": roof(c5_iter * it, NT / ms * 1e3, peaks[prec], nominals[prec],
                                     "k_traj_solve (single kernel): accepted iterations x per-iteration constant")}
    c5["headline_precision"] = "fp64"
    c5["fp32_vs_fp64_final_cost"] = final_cost_agreement(finals[("c5", "fp32")], finals[("c5", "fp64")])
    c5["termination_codes"] = ["max_iterations", "gradient_converged", "step_converged", "numerical_failure",
                               "rejection_budget", "non_finite", "fp32_resolution (FP32 only)"]
    if cpu:
        legs.append((c5, ("traj", [(qa[i], qb[i], mid[i]) for i in range(64)], "trajectories/s", "trajectories")))
    out["config5_trajectories"] = c5

    # ---- mobile base (SE(2) lanes, f2) ----
    Bm = 100_000
    sh = tg4.cpu().numpy().copy()
    sh[:, 4:] += np.tile(disk_translations(10_000, 2.0, 2024), (Bm // 10_000, 1))
    shd = dv.to_dev(sh)
    mstep, minit = pose_lane_step(**panda_counts())
    mstep += 2 * 6 * 3 * 7 + 200  # base columns (J_r^-1 Ad E, 6x3) + SE(2) retraction, same rules
    msolve, _ = beam_flops(mstep, minit)
    s = IkBeamSolver(model, "flange", rng_seed=RNG_SEED, optimize_base=True)
    om = s.alloc_outputs(Bm)
    ms = float(np.median(device_time(torch, lambda: s.solve_device(shd, om), 3, flush)))
    mob = {"workload": f"mobile-base IK-Beam (Panda + SE(2) base, disk-shifted targets r=2 m), {Bm} targets, FP32",
           "fp32": {"ms": ms, "value": Bm / ms * 1e3, "unit": "solves/s",
                    "success_rate": float(om.success.float().mean()),
                    "roofline": roof(msolve, Bm / ms * 1e3, peaks["fp32"], nominals["fp32"],
                                     "whole solve, SURVEY 8(d) rules")}}
    if cpu:
        legs.append((mob, ("mobile", list(sh[:64]), "solves/s", "targets")))
    out["mobile_base_ik_beam"] = mob
    for box, a in legs:
        box["cpu_baseline"] = cpu_leg(*a)
    return out


def final_cost_agreement(c32, c64):
    """Per-problem relative difference of the FP32 and FP64 final costs (same problems)."""
    rel = (np.asarray(c32) - np.asarray(c64)) / np.abs(np.asarray(c64))
    return {"rel_p10": float(np.percentile(rel, 10)), "rel_p50": float(np.percentile(rel, 50)),
            "rel_p90": float(np.percentile(rel, 90)), "rel_p99": float(np.percentile(rel, 99)),
            "within_1e-3": float(np.mean(np.abs(rel) <= 1e-3))}


def traj_iteration_flops(model, T, anc, nsph, pairs):
    """plan_trajectory Problem, one accepted LM iteration (J-eval + banded normal equations +
    banded Cholesky T * 2 * n^3 FMAs + solves + candidate eval), SURVEY 8(d) rules."""
    n = model.actuated_count
    fk = fk_flops(7, 1)
    sl = list(nsph)
    S = sum(nsph.values())
    # per timestep rows: limit n (nnz 1), self rows, world rows (1 sphere obstacle)
    self_terms = sum(nsph[a] * nsph[b] for a, b in pairs)
    world_terms = S
    ev_t = fk + SPHERE_CENTRE * S + DIST["sphere"] * (self_terms + world_terms) + \
        SOFTMIN_TERM * (self_terms + world_terms) + (SOFTMIN_ROW + ACTIVATION_ROW) * (len(pairs) + len(sl)) + 3 * n
    jac_t = sum(POINT_JAC_TERM * anc[nm] * nsph[nm] for nm in sl) + \
        sum(POINT_JAC_TERM * (anc[a] + anc[b]) * nsph[a] * nsph[b] for a, b in pairs)
    rows_t = [anc[nm] for nm in sl] + [max(anc[a], anc[b]) for a, b in pairs]
    # per pair: smoothness / velocity (nnz 2 each), swept rows (capsule-sphere, both timesteps)
    ev_p = 2 * 3 * n + DIST["capsule"] * S + SOFTMIN_TERM * S + (SOFTMIN_ROW + ACTIVATION_ROW) * len(sl)
    jac_p = sum(2 * POINT_JAC_TERM * anc[nm] * nsph[nm] for nm in sl)
    rows_p = [2 * anc[nm] for nm in sl]
    # per 5-window: acceleration + jerk (n rows each, nnz 5)
    ev_w = 2 * n * 10
    nnz_rows = [1] * n * T + [2] * 2 * n * (T - 1) + [5] * 2 * n * (T - 4) + [1] * 2 * n
    dense_rows = rows_t * T + rows_p * (T - 1)
    normal = sum(c * (c + 1) + 2 * c for c in nnz_rows + dense_rows)  # J^T J + J^T r (FMA = 2)
    chol = 2.0 * T * 2 * n ** 3 + 2 * 2.0 * T * n * (4 * n)             # banded factor + 2 band solves
    evals = T * ev_t + (T - 1) * ev_p + (T - 4) * ev_w
    jacs = T * jac_t + (T - 1) * jac_p
    resid = len(nnz_rows) + len(dense_rows)
    return float(evals + jacs + normal + chol + evals + 2 * resid + T * n)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2505_03728_b200 import _build

    if not os.path.exists(_build.LIB):
        _build.build()
    import paper_2505_03728_b200 as k
    from paper_2505_03728_b200._lib import lib
    from paper_2505_03728_b200.benchmark import reachable_target_array
    from paper_2505_03728_b200.tasks import IkBeamSolver

    dist = world > 1
    gloo = dist and args.backend == "gloo"
    torch.cuda.set_device(local_rank if not gloo else 0)
    B = args.batch
    model = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))

    def solver_for(prec):
        return IkBeamSolver(model, "flange", seeds=SEEDS, total_steps=TOTAL, prune_after=PRUNE, keep=KEEP,
                            rng_seed=RNG_SEED, precision=prec)

    solver = solver_for(args.precision)
    targets = reachable_target_array(model, "flange", B, RNG_SEED, start=rank * B)
    out = solver.alloc_outputs(B)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    peak, sms = fma_peak(torch, lib())

    def all_max(x):
        """Max over ranks (gloo: through a host tensor)."""
        if not dist:
            return x
        tt = torch.tensor([x], dtype=torch.float64, device="cpu" if gloo else "cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        return float(tt.item())

    def barrier():
        if dist:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler() if rank == 0 else None
    if clocks:
        clocks.start()
    for _ in range(args.warmup):
        solver.solve_device(targets, out)
    barrier()

    # ---- device-timed region: K steps, L2 flushed (untimed) between steps ----
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    barrier()
    for s in range(args.steps):
        flush.zero_()
        ev[s][0].record()
        solver.solve_device(targets, out, stages=1)
        ev[s][1].record()
        solver.solve_device(targets, out, stages=2)
        ev[s][2].record()
    barrier()
    clock_info = clocks.stop() if clocks else None
    t_step = [e[0].elapsed_time(e[2]) for e in ev]
    t_s1 = [e[0].elapsed_time(e[1]) for e in ev]
    total_ms = all_max(float(sum(t_step)))
    ms_per_step = total_ms / args.steps
    value = world * B / (ms_per_step * 1e-3)
    s1_ms = float(np.mean(t_s1))
    res = out.cpu()

    # ---- end-to-end through the public API: pinned host in, host results out ----
    # through the C ABI with HOST buffers (kop_ik_beam_host, IkBeamSolver.solve_host): the library
    # pipelines 64K-target chunks over 4 streams, H2D / kernels / D2H overlapped
    host_t = targets.cpu().pin_memory()
    host_out = solver.alloc_host_outputs(B)
    h2d = host_t.numel() * host_t.element_size()
    d2h = sum(getattr(host_out, kk).numel() * getattr(host_out, kk).element_size()
              for kk in ("q", "cost", "history", "pos_error", "rot_error", "success"))
    for _ in range(max(1, args.warmup)):
        solver.solve_host(host_t, host_out)
    barrier()
    e2e_ms = 0.0
    for s in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        solver.solve_host(host_t, host_out)
        e1.record()
        e1.synchronize()
        e2e_ms += e0.elapsed_time(e1)

    # the drop-in numpy path (pageable memory, allocations on every call): solve_ik_beam_batch's body
    np_t = targets.cpu().numpy()
    solver.solve(np_t)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    solver.solve(np_t)
    np_ms = (time.perf_counter() - t0) * 1e3

    # PCIe copy rates on their own (report H2D / D2H GB/s separately)
    def copy_gbs(dst, src, nbytes):
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(3):
            dst.copy_(src, non_blocking=True)
        c1.record()
        c1.synchronize()
        return 3 * nbytes / (c0.elapsed_time(c1) * 1e-3) / 1e9
    h2d_gbs = copy_gbs(torch.empty_like(targets), host_t, h2d)
    d2h_gbs = copy_gbs(host_out.history, out.history, host_out.history.numel() * 8)
    # the pipelined results must equal the device-resident run's
    e2e_match = bool(np.array_equal(host_out.q.numpy(), res.q) and np.array_equal(host_out.cost.numpy(), res.cost))
    e2e_ms = all_max(e2e_ms)
    e2e_value = world * B / (e2e_ms / args.steps * 1e-3)

    if rank != 0:
        return
    # ---- roofline: dominant kernel = stage 1 (seeds + prune) ----
    achieved = STAGE1_FLOP_PER_TARGET * B / (s1_ms * 1e-3) / 1e12
    clk = (clock_info or {}).get("sm_mhz") or 1965.0
    nominal = sms * NOMINAL_FP32_FLOP_PER_CLK_SM * 1965.0e6 / 1e12
    traffic, traffic_batch = load_traffic()
    if traffic is not None and traffic_batch:
        traffic = float(traffic) * B / float(traffic_batch)
    line = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64", "data": "synthetic",
        "config": workload_config(B, args.precision),
        "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": int(h2d * world),
                "d2h_bytes_per_step": int(d2h * world),
                "api": "C ABI kop_ik_beam_host (IkBeamSolver.solve_host): pinned host targets -> all IkResult "
                       "fields in pinned host memory; 16384-target chunks, H2D / kernels / D2H overlapped on 8 "
                       "library streams",
                "launches_per_step": 3 * -(-B // 16384), "bitwise_equal_to_device_run": e2e_match,
                "pcie_h2d_gbs": h2d_gbs, "pcie_d2h_gbs": d2h_gbs,
                "numpy_dropin": {"value": B / np_ms * 1e3, "unit": "solves/s", "wall_ms": np_ms,
                                 "api": "IkBeamSolver.solve(numpy (B,7)) -- the solve_ik_beam_batch path: pageable "
                                        "host arrays (staged by the library through pinned buffers, copy-out "
                                        "threads), output arrays allocated per call, host wall clock"}},
        "gpu_launches": 3 * args.steps,  # stage 1, stage 2, FP64 errors
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "frac_of_nominal": achieved / nominal, "nominal_peak": nominal,
                     "nominal_basis": f"{sms} SMs x 256 flop/clk x 1965 MHz (max SM clock)",
                     "frac_of_nominal_at_sampled_clock": achieved / (sms * NOMINAL_FP32_FLOP_PER_CLK_SM * clk * 1e6 / 1e12),
                     "kernel": "k_beam_stage1 (seeds x 6 LM steps + prune)",
                     "algorithmic_flops_per_launch": STAGE1_FLOP_PER_TARGET * B,
                     "flop_convention": f"SURVEY.md 8(d): {PANDA_STEP:.0f} flop/lane-step, {PANDA_INIT:.0f} "
                                        f"flop/lane init, {FLOP_PER_SOLVE / 1e6:.3f} Mflop/solve",
                     "peak_source": f"live FFMA microbenchmark, {sms} SMs (MEASURED_PEAKS.json has no FP32 entry)",
                     "stage1_ms": s1_ms, "stage1_share": s1_ms / (total_ms / args.steps) if not dist else None,
                     "solve_frac": value / world * FLOP_PER_SOLVE / 1e12 / peak,
                     "hbm_gbs_io": (B * (7 * 8) + B * (7 + 1 + 17 + 2) * 8 + B) / (ms_per_step * 1e-3) / 1e9},
        "clocks": clock_info,
        "accuracy": accuracy(res.pos_error, res.rot_error, res.success),
    }
    if dist:
        line["backend"] = args.backend
    if world == 1 and not args.quick:
        peak64, _ = fma_peak(torch, lib(), fp64=True)
        nominal64 = sms * NOMINAL_FP64_FLOP_PER_CLK_SM * 1965.0e6 / 1e12
        t0 = time.perf_counter()
        line["batch_sweep"] = run_sweep(torch, k, model, solver_for, flush, peak, nominal)
        line["fp64"] = run_fp64_headline(torch, model, solver_for, flush, B, peak64, nominal64)
        line["fk"] = run_fk(torch, model, flush)
        line["configs"] = run_configs(torch, k, model, flush, {"fp32": peak, "fp64": peak64},
                                      {"fp32": nominal, "fp64": nominal64}, cpu=not args.no_cpu_baseline)
        line["configs"]["peaks"] = {"fp32_live_ffma": peak, "fp64_live_dfma": peak64, "fp32_nominal": nominal,
                                    "fp64_nominal": nominal64}
        line["extended_wall_s"] = time.perf_counter() - t0
    # host-CPU baseline last: its forked pool must not overlap any device-timed call
    if world == 1 and not args.no_cpu_baseline:
        targets_cpu = targets[:4096].cpu().numpy()
        arm = CpuArm(targets_cpu)
        n = max(arm.cores, min(len(targets_cpu), int(args.cpu_seconds / arm.t1 * arm.cores)))
        rate, cres = arm.run(n)
        arm.close()
        cpu_succ = np.array([c[2] for c in cres])
        line["cpu_baseline"] = {
            "value": rate, "unit": "solves/s", "cores": arm.cores, "kind": "port",
            "sample": f"first {n} targets of this workload, one IK-Beam call per target (oracle port of "
                      f"kinoptik, float64 NumPy), multiprocessing over {arm.cores} cores",
            "single_core_value": 1.0 / arm.t1, "cpu_model": cpu_model(),
            "accuracy": accuracy(np.array([c[0] for c in cres]), np.array([c[1] for c in cres]), cpu_succ),
            "gpu_success_agreement_same_targets": float(np.mean(res.success[:n].astype(bool) == cpu_succ)),
            "gpu_success_rate_same_targets": float(np.mean(res.success[:n])),
        }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch

        if args.backend == "gloo":  # several ranks may share one GPU; collectives go through host tensors
            torch.cuda.set_device(0 if torch.cuda.device_count() == 1 else local_rank)
            torch.distributed.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch

            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
