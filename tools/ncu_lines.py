"""Per-source-line instruction / stall-sample shares of one kernel in an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kre}", "--launch-skip", str(skip), "-c", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ci = h.index("Instructions Executed")
si = h.index("Warp Stall Sampling (All Samples)")
inst, stall, src = defaultdict(float), defaultdict(float), {}
cur = None
fname = "?"
ops = defaultdict(lambda: defaultdict(float))
for r in rows[hi + 1:]:
    if len(r) <= si:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No" or r[0] == "Function Name":
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1]
        continue
    if cur is None:
        continue
    try:
        i, s = float(r[ci]), float(r[si])
    except ValueError:
        continue
    inst[cur] += i
    stall[cur] += s
    op = r[3].split()[0] if r[3].split() else "?"
    if op.startswith("@"):
        op = r[3].split()[1]
    ops[cur][op.split(".")[0]] += i
ti, ts = sum(inst.values()), sum(stall.values())
print(f"total warp-instructions {ti:.4g}, stall samples {ts:.4g}")
for ln in sorted(inst, key=lambda k: -stall[k])[:top]:
    o = sorted(ops[ln].items(), key=lambda kv: -kv[1])[:4]
    os_ = " ".join(f"{k}:{v / ti * 100:.1f}" for k, v in o)
    print(f"{ln[0][:8]}:{ln[1]:<5d} inst {inst[ln] / ti * 100:5.1f}% stall {stall[ln] / ts * 100:5.1f}% | "
          f"{src[ln].strip()[:70]:70s} | {os_}")

tot = defaultdict(float)
for ln in ops:
    for k, v in ops[ln].items():
        tot[k] += v
print("by opcode:", " ".join(f"{k}:{v / ti * 100:.1f}" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]))
