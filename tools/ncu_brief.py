"""Short summary of one .ncu-rep: speed-of-light, pipes, stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
want = ("Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Issue Slots Busy", "Executed Ipc Active", "L2 Hit Rate", "Registers Per Thread", "Achieved Active Warps Per SM",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler")
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name", "") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[-1]
st = []
for name, val in zip(h, v):
    if "issue_stalled" in name and name.endswith("per_issue_active.ratio") and "not_issued" not in name:
        try:
            st.append((float(val.replace(",", "")), name.split("issue_stalled_")[1].split("_per_issue")[0]))
        except ValueError:
            pass
    if name in ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"):
        print(f"{name:70s} {val}")
for p, n in sorted(st, reverse=True)[:8]:
    print(f"stall {n:24s} {p:6.2f} per issue")
