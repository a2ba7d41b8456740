"""Write profiles/ncu_sweep_traffic.json (the bench's roofline.traffic) and a launch-share summary from a
tools/profile_r2.sh capture: DRAM bytes (read + write) and time of every sweep launch of one V-cycle (ncu
launch list, cold L2 per launch) and the --set full summary of the first captured sweep launches.
usage: python tools/write_traffic.py gpurun_out/prof_<tag> <tag>"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(d, tag):
    rows = list(csv.reader(l for l in open(f"{d}/launches.csv") if not l.startswith("==")))
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    per = defaultdict(dict)
    for r in rows[1:]:
        if len(r) >= len(hdr):
            per[(int(r[ix["ID"]]), r[ix["Kernel Name"]])][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "") or 0)
    keys = sorted(per)
    hist = [i for i, (_, n) in enumerate(keys) if n.startswith("k_norm_hist")]
    if len(hist) < 3:   # fused history (one rank, one domain): the norm reductions delimit the cycles
        hist = [i for i, (_, n) in enumerate(keys) if n.startswith("k_norm_sum")]
    cyc = keys[hist[-3] + 1:hist[-2] + 1]
    sw = [per[k] for k in cyc if "k_sweep" in k[1]]
    by = [m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in sw]
    tot_t = sum(m["gpu__time_duration.sum"] for m in per.values() if True) and sum(per[k]["gpu__time_duration.sum"] for k in cyc)
    cls = defaultdict(float)
    for k in cyc:
        cls[k[1].split("(")[0].split("<")[0].replace("void ", "")] += per[k]["gpu__time_duration.sum"]
    out = {"kernel": "k_sweep<3, LPC, FF> (W' formulation: neighbour record W' 40 B: [n][4] (rho, m) + [n] rho E, own (X, c) 48 B)",
           "captured": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, "
                       f"bench.py --profile-only (config 4), every sweep launch of one V-cycle, cold L2 per launch; "
                       f"tools/profile_r2.sh {tag}",
           "sweep_launches_per_vcycle": len(sw),
           "dram_bytes_per_launch": sum(by) / len(by),
           "sweep_us_per_launch_cold": sum(m["gpu__time_duration.sum"] for m in sw) / len(sw) / 1e3,
           "launch_shares_cold": {k: v / tot_t for k, v in sorted(cls.items(), key=lambda x: -x[1])},
           "vcycle_us_cold_serialised": tot_t / 1e3}
    json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_sweep_traffic.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
