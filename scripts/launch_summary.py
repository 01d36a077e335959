"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) per kernel.

python scripts/launch_summary.py LAUNCHES.csv [--header TEXT]
"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--header", default="")
    a = ap.parse_args()
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    with open(a.csv) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for rec in csv.DictReader(lines):
        if rec.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(rec["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}[rec["Metric Unit"]]
        name = rec["Kernel Name"]
        tot[name] += v * scale
        cnt[name] += 1
    all_ms = sum(tot.values())
    if a.header:
        print(a.header)
    print(f"total ms over all launches: {all_ms:.2f}  ({sum(cnt.values())} launches)")
    for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{ms:10.3f} ms {cnt[name]:6d} launches {100 * ms / all_ms:5.1f}%  {name[:100]}")


if __name__ == "__main__":
    main()
