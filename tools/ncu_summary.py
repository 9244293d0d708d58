"""Summarise an ncu report (details page + key raw metrics) as JSON for profiles/."""
import csv, io, json, subprocess, sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Registers Per Thread", "Theoretical Occupancy",
        "Achieved Occupancy", "Achieved Active Warps Per SM", "Issue Slots Busy", "Issued Warp Per Scheduler",
        "No Eligible", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "Block Limit Registers", "Block Limit Shared Mem", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
       "sm__sass_thread_inst_executed_op_fadd_pred_on.sum", "sm__sass_thread_inst_executed_op_fmul_pred_on.sum",
       "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def run(rep, index=0):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    out = {}
    rows = list(csv.reader(io.StringIO(det)))
    ci = rows[0].index("Metric Name")
    ids = sorted({r[0] for r in rows[1:]}, key=int)
    kid = ids[index]
    for row in rows[1:]:
        if len(row) <= ci + 2 or row[0] != kid:
            continue
        out.setdefault("kernel", row[rows[0].index("Kernel Name")].split("(")[0])
        name, unit, val = row[ci], row[ci + 1], row[ci + 2]
        if name in KEYS and name not in out:
            out[name] = f"{val} {unit}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2 + index]
    stalls = {}
    for h, u, v in zip(hdr, units, vals):
        if h in RAW:
            out[h] = f"{v} {u}".strip()
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls[h.split("stalled_")[1].replace("_per_issue_active.ratio", "")] = float(v)
            except ValueError:
                pass
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:10]
    out["top_stall_reasons_per_issue"] = {k: round(v, 3) for k, v in top}
    return out


if __name__ == "__main__":
    print(json.dumps(run(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0), indent=1))
