#!/usr/bin/env python
"""Batched Panda IK-Beam throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One step = one IK-Beam pass (64 seeds, 6 LM steps, keep 4, 10 more steps;
tasks.py:119-161) over a batch of synthetic reachable Panda targets
(benchmark.py:83-93, rng 77) resident in HBM.  Weak scaling: every rank
solves its own ``--batch`` targets (distinct Philox index ranges); there is
no collective in the solve -- the ranks only meet for the barrier and the
max-over-ranks time.

Prints ONE JSON line on rank 0 (see DESIGN.md section 6 for every key).
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
# SURVEY.md section 8(d) algorithmic flop convention (FMA = 2 flops)
FLOP_LANE_STEP = 4.5e3
FLOP_LANE_INIT = 1.2e3
FLOP_FINAL_ERR = 1.1e3
FLOP_PER_SOLVE = 2.0e6
STAGE1_FLOP_PER_TARGET = SEEDS * (FLOP_LANE_INIT + PRUNE * FLOP_LANE_STEP)
STAGE2_FLOP_PER_TARGET = KEEP * (TOTAL - PRUNE) * FLOP_LANE_STEP + FLOP_FINAL_ERR
RNG_SEED = 77


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
    return ap.parse_args()


# ---------------------------------------------------------------------------
# CPU reference arm: the oracle port of kinoptik's IK-Beam, one target per
# call exactly like the reference's solve_ik_beam (benchmark.py:136-151)
# ---------------------------------------------------------------------------
_W = {}


def _cpu_worker_init():
    from oracle import ik_oracle as o

    robots = os.path.join(ROOT, "paper_2505_03728_b200", "robots")
    ch = o.load_chain_files(os.path.join(robots, "arm7.urdf"), os.path.join(robots, "arm7.sidecar.json"))
    _W["o"], _W["ch"] = o, ch
    _W["seeds"] = o.sample_seeds(ch, SEEDS, RNG_SEED)
    _W["link"] = ch.link("flange")


def _cpu_solve(chunk):
    o, ch = _W["o"], _W["ch"]
    out = []
    for t in chunk:
        r = o.ik_beam(ch, _W["link"], t[None, :4], t[None, 4:], _W["seeds"])
        out.append((float(r.pos_err[0]), float(r.rot_err[0]), bool(r.success[0])))
    return out


class CpuArm:
    """Pool over every host core; each worker solves whole targets serially."""

    def __init__(self, targets: np.ndarray):
        import multiprocessing as mp

        self.cores = os.cpu_count() or 1
        self.targets = targets
        self.pool = mp.get_context("fork").Pool(self.cores, initializer=_cpu_worker_init)
        # per-target single-core cost, to size bounded samples
        _cpu_worker_init()
        t0 = time.perf_counter()
        _cpu_solve(targets[:2])
        self.t1 = (time.perf_counter() - t0) / 2

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

    robots = os.path.join(ROOT, "paper_2505_03728_b200", "robots")
    ch = o.load_chain_files(os.path.join(robots, "arm7.urdf"), os.path.join(robots, "arm7.sidecar.json"))
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
    rates, res = [], []
    t0 = time.perf_counter()
    for s in range(args.steps):
        r, out = arm.run(per_step, offset=s * per_step)
        rates.append(r)
        res += out
    wall = time.perf_counter() - t0
    arm.close()
    value = float(args.steps * per_step / wall)
    pos = np.array([r[0] for r in res])
    rot = np.array([r[1] for r in res])
    sample = (f"{per_step} targets/step (first {len(targets)} of the rng-77 workload, cycled) solved one per "
              f"call by the oracle port of kinoptik IK-Beam, multiprocessing over {arm.cores} host cores")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        # the same config line as our arm; each reference step is the bounded sample named in cpu_baseline
        "data": "synthetic", "config": workload_config(args.batch, args.precision),
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": arm.cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "accuracy": accuracy(pos, rot, np.array([r[2] for r in res])),
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


def fp32_peak(torch, lib):
    """Measured FP32 FMA-pipe peak (TFLOP/s): immediate-operand FFMA chains, all SMs."""
    import ctypes as C

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    sink = torch.zeros(4096, device="cuda", dtype=torch.float32)
    flops = C.c_double()
    blocks, threads, iters = sms * 8, 256, 20000
    st = torch.cuda.current_stream().cuda_stream
    lib.kop_fma_peak_kernel(blocks, threads, 2000, sink.data_ptr(), C.byref(flops), st)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.kop_fma_peak_kernel(blocks, threads, iters, sink.data_ptr(), C.byref(flops), st)
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
    torch.cuda.set_device(local_rank)
    B = args.batch
    model = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
    solver = IkBeamSolver(model, "flange", seeds=SEEDS, total_steps=TOTAL, prune_after=PRUNE, keep=KEEP,
                          rng_seed=RNG_SEED, precision=args.precision)
    targets = reachable_target_array(model, "flange", B, RNG_SEED, start=rank * B)
    out = solver.alloc_outputs(B)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    peak, sms = fp32_peak(torch, lib())

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
    total_ms = float(sum(t_step))
    if dist:
        tt = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(tt.item())
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
    if dist:
        tt = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = world * B / (e2e_ms / args.steps * 1e-3)

    if rank != 0:
        return
    # ---- roofline: dominant kernel = stage 1 (seeds + prune) ----
    achieved = STAGE1_FLOP_PER_TARGET * B / (s1_ms * 1e-3) / 1e12
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
                       "fields in pinned host memory; 65536-target chunks, H2D / kernels / D2H overlapped on 4 "
                       "library streams",
                "launches_per_step": 3 * -(-B // 65536), "bitwise_equal_to_device_run": e2e_match,
                "pcie_h2d_gbs": h2d_gbs, "pcie_d2h_gbs": d2h_gbs},
        "gpu_launches": 3 * args.steps,  # stage 1, stage 2, FP64 errors
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "k_beam_stage1 (seeds x 6 LM steps + prune)",
                     "algorithmic_flops_per_launch": STAGE1_FLOP_PER_TARGET * B,
                     "flop_convention": "SURVEY.md 8(d): 4.5 kflop/lane-step, 1.2 kflop/lane init",
                     "peak_source": f"live FFMA microbenchmark, {sms} SMs (MEASURED_PEAKS.json has no FP32 entry)",
                     "stage1_ms": s1_ms, "stage1_share": s1_ms / (total_ms / args.steps) if not dist else None,
                     "solve_frac": value / world * FLOP_PER_SOLVE / 1e12 / peak,
                     "hbm_gbs_io": (B * (7 * 8) + B * (7 + 1 + 17 + 2) * 8 + B) / (ms_per_step * 1e-3) / 1e9},
        "clocks": clock_info,
        "accuracy": accuracy(res.pos_error, res.rot_error, res.success),
    }
    if world == 1 and not args.no_cpu_baseline:
        targets_cpu = targets[:4096].cpu().numpy()
        arm = CpuArm(targets_cpu)
        n = max(arm.cores, min(len(targets_cpu), int(args.cpu_seconds / arm.t1 * arm.cores)))
        rate, cres = arm.run(n)
        arm.close()
        line["cpu_baseline"] = {
            "value": rate, "unit": "solves/s", "cores": arm.cores, "kind": "port",
            "sample": f"first {n} targets of this workload, one IK-Beam call per target (oracle port of "
                      f"kinoptik, float64 NumPy), multiprocessing over {arm.cores} cores",
            "accuracy": accuracy(np.array([c[0] for c in cres]), np.array([c[1] for c in cres]),
                                 np.array([c[2] for c in cres])),
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
