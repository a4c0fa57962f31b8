"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: launches, mean and total device time, share of the total."""
import csv
import sys
from collections import defaultdict


def main(path, header=""):
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))
            if r["Metric Name"] == "gpu__time_duration.sum"]
    agg = defaultdict(list)
    for r in rows:
        name = r["Kernel Name"].split("(")[0]
        scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6}.get(r["Metric Unit"], 1.0)
        agg[name].append(float(r["Metric Value"].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values())
    if header:
        print(header)
    print(f"{'kernel':70s} {'launches':>8s} {'mean_ns':>12s} {'total_ns':>14s} share")
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{name[:70]:70s} {len(v):8d} {sum(v) / len(v):12.1f} {sum(v):14.1f} {sum(v) / tot:.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
