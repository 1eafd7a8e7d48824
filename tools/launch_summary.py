"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py launches.csv OUT.md "command description"
"""
import csv
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import short_name  # noqa: E402

SC = {"ms": 1e3, "us": 1.0, "ns": 1e-3, "s": 1e6, "msecond": 1e3, "usecond": 1.0,
      "nsecond": 1e-3, "second": 1e6}


def main():
    src, out, what = sys.argv[1], sys.argv[2], sys.argv[3]
    hdr, agg = None, defaultdict(lambda: [0, 0.0])
    for r in csv.reader(open(src)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * SC.get(d["Metric Unit"], 1.0)
        n = short_name(d["Kernel Name"])
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as fh:
        fh.write("# Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`)\n\n")
        fh.write(f"{what}\n\nncu serialises launches with cold caches: compare SHARES with bench.py, "
                 "not absolute times.\n\n| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            fh.write(f"| `{k}` | {v[0]} | {v[1] / 1e3:.2f} | {v[1] / tot * 100:.1f}% |\n")
    print(open(out).read())


if __name__ == "__main__":
    main()
