"""Summarise an .ncu-rep (details page) into a short text table: python tools/ncu_summary.py rep [...]"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Frequency", "Memory Throughput", "DRAM Throughput",
        "Compute (SM) Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "Issued Warp Per Scheduler", "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Block Limit Registers", "Block Limit Shared Mem", "Dynamic Shared Memory Per Block",
        "Grid Size", "Block Size", "Waves Per SM", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Mem Busy", "Max Bandwidth", "Mem Pipes Busy", "SM Busy"]


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    mi = hdr.index("Metric Name")
    ui = hdr.index("Metric Unit")
    vi = hdr.index("Metric Value")
    seen = {}
    kname = None
    for r in rows[1:]:
        kname = r[ki]
        if r[mi] in WANT and r[mi] not in seen:
            seen[r[mi]] = f"{r[vi]} {r[ui]}"
    lines = [f"# {path}", f"kernel: {kname[:120]}"]
    for w in WANT:
        if w in seen:
            lines.append(f"{w:40s} {seen[w]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        h, u, v = rr[0], rr[1], rr[2]
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                    "smsp__average_warp_latency_issue_stalled_barrier", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
                    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
                    "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
                    "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
                    "smsp__warp_issue_stalled_wait_per_warp_active.pct",
                    "smsp__warp_issue_stalled_not_selected_per_warp_active.pct",
                    "smsp__warp_issue_stalled_selected_per_warp_active.pct",
                    "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
                    "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
                    "smsp__warp_issue_stalled_dispatch_stall_per_warp_active.pct",
                    "smsp__warp_issue_stalled_no_instruction_per_warp_active.pct",
                    "smsp__warp_issue_stalled_drain_per_warp_active.pct",
                    "smsp__warp_issue_stalled_membar_per_warp_active.pct",
                    "smsp__warp_issue_stalled_imc_miss_per_warp_active.pct",
                    "smsp__warp_issue_stalled_branch_resolving_per_warp_active.pct",
                    "smsp__warp_issue_stalled_sleeping_per_warp_active.pct",
                    "smsp__warp_issue_stalled_tex_throttle_per_warp_active.pct",
                    "smsp__warp_issue_stalled_misc_per_warp_active.pct",
                    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"):
            for i, name in enumerate(h):
                if name == key:
                    lines.append(f"{key:70s} {v[i]} {u[i]}")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarize(p))
        print()
