"""Per-kernel summary of an ncu --csv metrics capture of one build + one query
batch (scripts/profile_once.py), in the JSON bench.py reads for
roofline.traffic and the CWS metrics (profiles/<round>/ncu_cfg<cfg>.json).

python scripts/ncu_summary.py CAPTURE.csv OUT.json "<source description>"

Per kernel: launches, DRAM bytes (read + write) and duration summed over the
launches, and duration-weighted means of the percentage metrics.
"""
import collections
import csv
import json
import re
import sys

src, out, desc = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
with open(src) as f:
    lines = [ln for ln in f if ln.startswith('"')]
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "second": 1.0,
        "%": 1.0, "": 1.0}
per_launch = collections.defaultdict(dict)
names = {}
for r in csv.DictReader(lines):
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").strip()
    try:
        v = float(r["Metric Value"].replace(",", "")) * unit.get(r["Metric Unit"], 1.0)
    except ValueError:
        continue
    per_launch[r["ID"]][r["Metric Name"]] = v
    names[r["ID"]] = name
acc = collections.defaultdict(lambda: collections.defaultdict(float))
for lid, mets in per_launch.items():
    k = acc[names[lid]]
    t = mets.get("gpu__time_duration.sum", 0.0)
    k["launches"] += 1
    k["time_s"] += t
    k["dram_bytes"] += mets.get("dram__bytes_read.sum", 0.0) + mets.get("dram__bytes_write.sum", 0.0)
    for mn, v in mets.items():
        if mn.endswith(".pct") or "pct_of_peak" in mn:
            k["w:" + mn] += v * t
kernels = {}
for n, k in sorted(acc.items()):
    if n.startswith("at::"):
        continue
    d = {"launches": int(k["launches"]), "dram_bytes": k["dram_bytes"], "time_s": k["time_s"]}
    for mn, v in k.items():
        if mn.startswith("w:") and k["time_s"] > 0:
            d[mn[2:]] = v / k["time_s"]
    kernels[n] = d
res = {"source": desc, "kernels": kernels}
cws = [v for n, v in kernels.items() if n.startswith("cws_")]
if cws:
    c = max(cws, key=lambda v: v["time_s"])
    res["cws"] = {"l2_hit_rate": c.get("lts__t_sector_hit_rate.pct"),
                  "fp64_pipe_util": c.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                  "issue_active": c.get("sm__issue_active.avg.pct_of_peak_sustained_active")}
json.dump(res, open(out, "w"), indent=1)
tot = sum(v["time_s"] for v in kernels.values())
for n, v in sorted(kernels.items(), key=lambda kv: -kv[1]["time_s"])[:25]:
    print(f"{v['time_s'] * 1e3:9.3f} ms {100 * v['time_s'] / tot:5.1f}% x{v['launches']:4d} "
          f"{v['dram_bytes'] / 1e9:8.3f} GB  {n[:80]}")
