"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, total device time and share of the profiled run.
usage: python tools/launch_shares.py launches.csv out.json "source description" """
import csv, json, re, sys
from collections import OrderedDict

src, dst = sys.argv[1], sys.argv[2]
desc = sys.argv[3] if len(sys.argv) > 3 else ""
lines = [l for l in open(src) if l.startswith('"')]
rows = list(csv.DictReader(lines))
agg = OrderedDict()
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
    name = re.sub(r"^(void )?gmg::", "", name)
    us = float(r["Metric Value"].replace(",", "")) / (1e3 if r["Metric Unit"] == "ns" else 1.0)
    a = agg.setdefault(name, {"launches": 0, "total_us": 0.0})
    a["launches"] += 1
    a["total_us"] += us
tot = sum(a["total_us"] for a in agg.values())
out = {"source": desc, "total_us": round(tot, 1),
       "kernels": {k: {"launches": v["launches"], "total_us": round(v["total_us"], 1), "share": round(v["total_us"] / tot, 4)}
                   for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["total_us"])}}
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps({k: v["share"] for k, v in out["kernels"].items()}))
