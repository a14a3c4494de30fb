"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel name: launches, total/mean time and share of the profiled device time.
usage: python tools/ncu_summary.py launches.csv [--top N]"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    with open(path) as fh:
        lines = [ln for ln in fh if not ln.startswith("==")]
    agg = defaultdict(lambda: [0, 0.0])
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        name = r["Kernel Name"]
        name = name if len(name) < 90 else name[:87] + "..."
        agg[name][0] += 1
        agg[name][1] += ns
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':90s} {'n':>6s} {'total ms':>10s} {'mean us':>10s} {'share':>7s}")
    for name, (n, ns) in sorted(agg.items(), key=lambda t: -t[1][1])[:top]:
        print(f"{name:90s} {n:6d} {ns / 1e6:10.3f} {ns / n / 1e3:10.2f} {100 * ns / tot:6.2f}%")
    print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main()
