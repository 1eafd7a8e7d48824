"""Summarise one ncu report: SOL %, issue, occupancy, stall mix, and SASS regions (test/tools)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(det.splitlines()))
h = r[0]
want = {"Duration", "L1/TEX Cache Throughput", "L2 Cache Throughput", "DRAM Throughput", "Issue Slots Busy",
        "Executed Ipc Active", "Registers Per Thread", "Achieved Active Warps Per SM", "L1/TEX Hit Rate",
        "Warp Cycles Per Issued Instruction", "Compute (SM) Throughput"}
for row in r[1:]:
    if row[h.index("Metric Name")] in want:
        print(f"{row[h.index('Metric Name')]:40s} {row[h.index('Metric Value')]} {row[h.index('Metric Unit')]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, v = r[0], r[-1]
items = []
for i, k in enumerate(h):
    if "pcsamp_warps_issue_stalled" in k and "not_issued" not in k:
        try:
            items.append((k.split("stalled_")[1], float(v[i].replace(",", ""))))
        except ValueError:
            pass
tot = sum(x for _, x in items) or 1
print("stalls:", ", ".join(f"{k} {x / tot * 100:.0f}%" for k, x in sorted(items, key=lambda t: -t[1])[:7]))
for k in ("smsp__inst_executed.sum", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
          "dram__bytes_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"):
    if k in h:
        print(f"{k:70s} {v[h.index(k)]}")
