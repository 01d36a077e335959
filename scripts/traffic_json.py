"""Convert an ncu CSV (--metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum) of `scripts/profile_once.py --nq 1000` into the
per-kernel DRAM-traffic JSON bench.py reads (profiles/<round>/traffic_cfg1.json).

python scripts/traffic_json.py TRAFFIC.csv OUT.json
"""
import collections
import csv
import json
import re
import sys

src, out = sys.argv[1], sys.argv[2]
with open(src) as f:
    lines = [ln for ln in f if ln.startswith('"')]
acc = collections.defaultdict(lambda: {"launches": set(), "dram_bytes": 0.0, "time_s": 0.0})
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "second": 1.0}
for r in csv.DictReader(lines):
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").strip()
    v = float(r["Metric Value"].replace(",", "")) * unit[r["Metric Unit"]]
    k = acc[name]
    k["launches"].add(r["ID"])
    if r["Metric Name"].startswith("dram__bytes"):
        k["dram_bytes"] += v
    elif r["Metric Name"] == "gpu__time_duration.sum":
        k["time_s"] += v
res = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                 "--clock-control none python scripts/profile_once.py --nq 1000 (configs[1]: one build + one "
                 "1000-query batch)",
       "kernels": {n: {"launches": len(v["launches"]), "dram_bytes": v["dram_bytes"], "time_s": v["time_s"]}
                   for n, v in sorted(acc.items()) if not n.startswith("at::")}}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({n: (v["launches"], round(v["dram_bytes"] / 1e6, 1), round(v["time_s"] * 1e3, 3))
                  for n, v in res["kernels"].items()}, indent=0))
