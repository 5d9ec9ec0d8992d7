"""Summarise an ncu --set full report (.ncu-rep) into the numbers the roofline
and DESIGN.md cite: duration, DRAM bytes, throughputs, pipe utilisation,
occupancy, instruction count and the top stall reasons.
    python profiles/tools/ncu_summary.py report.ncu-rep [> summary.txt]"""
import csv
import io
import subprocess
import sys

WANT_DETAILS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
                "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
                "Issue Slots Busy", "Executed Instructions", "Registers Per Thread", "Theoretical Occupancy",
                "Achieved Occupancy", "Achieved Active Warps Per SM", "Dynamic Shared Memory Per Block",
                "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size"]
RAW_PREFIX = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor", "sm__inst_executed_pipe_fp64",
              "sm__pipe_fp64", "sm__pipe_fma_cycles_active", "sm__inst_executed_pipe_tc", "gpu__time_duration.sum",
              "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime", "sm__inst_executed_pipe_tensor_subpipe_hmma",
              "sm__mem_tensor_cycles_active.avg", "smsp__thread_inst_executed_per_inst_executed.ratio",
              "lts__t_sector_hit_rate.pct"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(path):
    det = list(csv.reader(io.StringIO(run([path, "--page", "details", "--csv"]))))
    h = det[0]
    kn, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    kernels = []
    for row in det[1:]:
        if row[kn] not in kernels:
            kernels.append(row[kn])
    print(f"report: {path}")
    for k in kernels:
        print(f"\nkernel: {k[:150]}")
        for row in det[1:]:
            if row[kn] == k and row[mi] in WANT_DETAILS:
                print(f"  {row[mi]:40s} {row[vi]:>16s} {row[ui]}")
    raw = list(csv.reader(io.StringIO(run([path, "--page", "raw", "--csv"]))))
    hdr = raw[0]
    for vals in raw[2:] if len(raw) > 2 else raw[1:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"\nraw metrics ({name[:80]}):")
        stalls = []
        for n, v in zip(hdr, vals):
            if any(n.startswith(p) for p in RAW_PREFIX):
                print(f"  {n:70s} {v}")
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), n))
                except ValueError:
                    pass
        tot = sum(x for x, _ in stalls) or 1.0
        print("  top stall reasons (pc sampling):")
        for x, n in sorted(stalls, reverse=True)[:6]:
            print(f"    {100 * x / tot:5.1f}%  {n.replace('smsp__pcsamp_warps_issue_stalled_', '')}")


if __name__ == "__main__":
    main(sys.argv[1])
