"""Share table of an ncu launch list (`--metrics gpu__time_duration.sum --csv`).

    python tools/launch_summary.py gpurun_out/launches.csv
Per-launch times are cold-cache and serialised: compare shares, not absolutes.
"""
import collections
import csv
import sys


def main(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    r = list(csv.DictReader(lines))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for row in r:
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(row["Metric Value"].replace(",", ""))
        if row.get("Metric Unit") in ("ns", "nsecond"):
            v /= 1000.0
        elif row.get("Metric Unit") in ("ms", "msecond"):
            v *= 1000.0
        k = row["Kernel Name"].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(t for _, t in agg.values())
    print("| share | launches | avg us | kernel |\n|---:|---:|---:|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {100 * t / tot:.1f}% | {n} | {t / n:.1f} | `{k}` |")


if __name__ == "__main__":
    main(sys.argv[1])
