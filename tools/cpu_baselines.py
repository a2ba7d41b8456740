"""The oracle as the CPU baseline on configs 1-4: its timing build (oracle.use_timing_build:
-O3 -march=native, OpenMP within a color, bit-identical to the parity build) with 1 thread and with every host
core, sweep cell-updates/s (Algorithm 2's count, the oracle runs every phase) and V-cycles/s over a bounded
number of V-cycles per config.  Run on the GPU box's host:  python tools/cpu_baselines.py > out.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from synth import configs, state  # noqa: E402


def main():
    cores = os.cpu_count() or 1
    model = "unknown"
    try:
        model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    out = {"host_cores": cores, "cpu": model, "configs": {}}
    for k, cycles in ((1, 20), (2, 5), (3, 2), (4, 1)):
        m = configs.config(k)
        fs = configs.FREESTREAM[k]
        W = state.bow_shock(m, *fs) if k in (3, 4) else state.gaussian_bump(m, *fs) if k == 1 else state.uniform(m, *fs)
        Winf = state.winf(*fs)
        H = oracle.build_hierarchy(m, 3, 0.5)
        cu = sum(e["level"].n for e in H[1:]) * 2 * 6
        row = {"cells": m.n_cells, "sweep_cell_updates_per_vcycle": cu, "vcycles_timed": cycles}
        for threads in (1, cores):
            oracle.use_timing_build(threads)
            oracle.vcycle(H, W, Winf, oracle.Options(), 1)          # warm-up (page-in, thread pool)
            t0 = time.perf_counter()
            oracle.vcycle(H, W, Winf, oracle.Options(), cycles)
            dt = (time.perf_counter() - t0) / cycles
            row[f"threads_{threads}"] = {"s_per_vcycle": dt, "cell_updates_per_s": cu / dt, "vcycles_per_s": 1 / dt}
        oracle.use_parity_build()
        out["configs"][f"config{k}"] = row
        print(json.dumps({k: row}), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
