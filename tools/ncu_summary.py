"""Summarise ncu reports (gpurun_out/*.ncu-rep, read here without a GPU) into profiles/.

    python tools/ncu_summary.py OUT_PREFIX report1.ncu-rep [report2 ...]

Writes OUT_PREFIX.json (per-launch metrics) and OUT_PREFIX.md (table), and merges per-kernel
DRAM bytes per launch into profiles/ncu_summary.json (read by bench.py for roofline.traffic).
"""

import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "inst",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_sb",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def short_name(full):
    """'void ns::<anon>::factor_rows_pipe_kernel<32>(args)' -> 'factor_rows_pipe_kernel<32>'."""
    head = full.split("(")[0].replace("void ", "")
    depth, cut = 0, len(head)
    for i in range(len(head) - 1, -1, -1):  # last '::' outside template brackets
        c = head[i]
        if c == ">":
            depth += 1
        elif c == "<":
            depth -= 1
        elif c == ":" and depth == 0 and i > 0 and head[i - 1] == ":":
            cut = i + 1
            break
    name = head[cut:] if cut < len(head) else head
    return name if len(name) < 60 else name[:57] + "..."


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short_name(r[hdr.index("Kernel Name")])}
        for m, k in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * SCALE.get(units[i], 1.0)
        res.append(d)
    return res


def main():
    prefix, reps = sys.argv[1], sys.argv[2:]
    launches = []
    for rep in reps:
        for d in read(rep):
            d["report"] = os.path.basename(rep)
            launches.append(d)
    json.dump(launches, open(prefix + ".json", "w"), indent=1)
    cols = ["kernel", "time", "dram_read", "dram_write", "regs", "warps_active_pct",
            "issue_active_pct", "l1_pct", "l2_pct", "dram_pct", "tensor_pct", "stall_short_sb",
            "stall_long_sb", "stall_wait"]
    with open(prefix + ".md", "w") as fh:
        fh.write("| " + " | ".join(cols) + " |\n|" + "---|" * len(cols) + "\n")
        for d in launches:
            vals = []
            for c in cols:
                v = d.get(c, "")
                if c == "time" and v != "":
                    v = f"{v * 1e3:.3f} ms"
                elif c in ("dram_read", "dram_write") and v != "":
                    v = f"{v / 1e9:.3f} GB"
                elif isinstance(v, float):
                    v = f"{v:.2f}"
                vals.append(str(v))
            fh.write("| " + " | ".join(vals) + " |\n")
    summ_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                             "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {"kernels": {}}
    agg = {}
    for d in launches:
        name = d["kernel"].split("<")[0]
        for fam in ("factor_rows", "core_rows", "refresh", "predict"):
            if name.startswith(fam):  # the K3b variants (dual / gram / pipe ...) share a family
                name = fam
                break
        a = agg.setdefault(name, [])
        if "dram_read" in d:
            a.append(d["dram_read"] + d.get("dram_write", 0.0))
    for name, v in agg.items():
        if v:
            summ["kernels"][name] = {"dram_bytes_per_launch": sum(v) / len(v), "launches": len(v),
                                     "source": os.path.basename(prefix)}
    json.dump(summ, open(summ_path, "w"), indent=1)
    print(open(prefix + ".md").read())


if __name__ == "__main__":
    main()
