"""Summarise ncu outputs of tools/profile_r2.sh (dev tool).
usage: python tools/ncu_summary.py gpurun_out/prof_<tag>"""
import csv
import json
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    per = defaultdict(dict)
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        k = (int(r[ix["ID"]]), r[ix["Kernel Name"]])
        v = r[ix["Metric Value"]].replace(",", "")
        per[k][r[ix["Metric Name"]]] = float(v) if v else 0.0
    return per


def main(d):
    per = launches(f"{d}/launches.csv")
    # one V-cycle = the launches between two history launches (k_norm_hist; on one rank and one domain the
    # norm reduction k_norm_sum writes the history entry itself)
    keys = sorted(per)
    hist = [i for i, (_, n) in enumerate(keys) if n.startswith("k_norm_hist")]
    if len(hist) < 3:   # fused history (one rank, one domain): the norm reductions delimit the cycles
        hist = [i for i, (_, n) in enumerate(keys) if n.startswith("k_norm_sum")]
    a, b = (hist[-3] + 1, hist[-2] + 1) if len(hist) >= 3 else (0, len(keys))
    cyc = keys[a:b]
    cls = defaultdict(lambda: [0.0, 0, 0.0])
    for k in cyc:
        m = per[k]
        name = k[1].split("<")[0].split("(")[0]
        c = cls[name]
        c[0] += m.get("gpu__time_duration.sum", 0.0)
        c[1] += 1
        c[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(c[0] for c in cls.values())
    out = {"launches_in_cycle": len(cyc), "total_us": tot / 1e3,
           "classes": {n: {"us": c[0] / 1e3, "launches": c[1], "share": c[0] / tot,
                           "dram_MB": c[2] / 1e6, "dram_TBps": c[2] / c[0] / 1e3 if c[0] else None}
                       for n, c in sorted(cls.items(), key=lambda x: -x[1][0])}}
    sw = cls.get("k_sweep")
    if sw:
        out["sweep_dram_bytes_per_launch"] = sw[2] / sw[1]
        out["sweep_us_per_launch"] = sw[0] / sw[1] / 1e3
    print(json.dumps(out, indent=1))
    # full-set raw summary
    try:
        rows = list(csv.reader(open(f"{d}/sweep_full_raw.csv")))
        hdr = rows[0]
        want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "lts__t_sector_hit_rate.pct", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
                "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
                "launch__grid_size", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "lts__t_sectors_srcunit_tex_op_read.sum"]
        idx = [hdr.index(w) for w in want if w in hdr]
        print("\t".join(hdr[i][:28] for i in idx))
        for r in rows[2:]:
            print("\t".join(r[i][:28] for i in idx))
    except Exception as e:
        print("raw:", e)


if __name__ == "__main__":
    main(sys.argv[1])
