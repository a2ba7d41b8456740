"""Summarise an ncu --csv metrics capture of the NEXT-1 kernels (k_ho_*) into
profiles/r02/ho_ncu.json (round 1: profiles/r01/; the round-2 capture is kept as
profiles/r02/ho_ncu_executed_v33.json): per kernel time, DRAM bytes, FP64 thread
instructions and flops (2 dfma + dmul + dadd); for k_ho_flux the FP64 flops
per Gauss point that bench.py's next1 roofline uses.

    ncu --clock-control none -k regex:k_ho_ -c 4 --csv --metrics <list below> \
        python tools/ho_bench.py --profile-only > gpurun_out/ho_ncu.csv
    python tools/ho_ncu.py gpurun_out/ho_ncu.csv <gauss_points>
"""
import csv
import json
import os
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]


def main(path, gauss_points):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    I = {h: i for i, h in enumerate(hdr)}
    ker = {}
    for r in rows:
        name = r[I["Kernel Name"]].split("(")[0]
        v = r[I["Metric Value"]].replace(",", "")
        try:
            ker.setdefault(name, {})[r[I["Metric Name"]]] = float(v)
        except ValueError:
            pass
    out = {"source": "ncu --clock-control none (cold, serialised), one launch each, config 4 (1 M cells)",
           "kernels": {}}
    for name, m in ker.items():
        fl = 2 * m.get(METRICS[3], 0) + m.get(METRICS[4], 0) + m.get(METRICS[5], 0)
        t = m.get(METRICS[0], 0) * 1e-9
        out["kernels"][name] = {"us": t * 1e6, "dram_MB": (m.get(METRICS[1], 0) + m.get(METRICS[2], 0)) / 1e6,
                                "fp64_gflop": fl / 1e9, "fp64_tflops_cold": fl / t / 1e12 if t else None,
                                "fp64_pipe_active_pct": m.get(METRICS[6]), "warps_active_pct": m.get(METRICS[7]),
                                "registers": m.get(METRICS[8])}
        if "k_ho_flux" in name:
            out["flux_fp64_flops_per_gauss_point"] = fl / gauss_points
    os.makedirs("profiles/r02", exist_ok=True)
    json.dump(out, open("profiles/r02/ho_ncu.json", "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
