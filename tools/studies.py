"""§8(f) NEXT-2 sensitivity studies on the GPU hot path (run under gpurun).

Reproduces the *structure* of the paper's §6 studies (PAPER.md:797-817,
853-874, 1101-1105) with the first-order operator of this build: residual
history of the 3-level V-cycle vs
  * MC-LU-SGS sweep count (paper: 4-6 optimal),
  * implicit CFL (paper: CFL >= 10 suffices),
  * relaxation: DF-adaptive (paper), DF off (alpha = 1; paper: "explodes" at
    Ma 2 / M6), fixed beta (traditional relaxation P:526-532),
and the explicit 1-level iteration (the "GPU explicit" column of Table 5) for
the GMG speed-up ratio.  Impulsive free-stream start.  Writes JSON.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_06347_b200 import gmg  # noqa: E402
from synth import configs, state  # noqa: E402


def run(m, W, Winf, n_cycles, n_levels=3, chunk=25, **kw):
    s = gmg.Solver(m, n_levels=n_levels, **kw)
    s.set_state(W, Winf)
    hist = []
    ok = True
    t0 = time.perf_counter()
    done = 0
    while done < n_cycles:
        k = min(chunk, n_cycles - done)
        try:
            h = s.vcycle(k)
        except gmg.GmgError as e:
            ok = False
            hist.append(float("nan"))
            break
        hist.extend(h[:-1, 0].tolist())
        done += k
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if ok:
        hist.append(float(h[-1, 0]))
    s.close()
    r0 = hist[0]
    rel = [x / r0 for x in hist]
    drop = None
    for k, x in enumerate(rel):
        if x <= 1e-3:
            drop = k
            break
    return {"ok": ok, "cycles": done, "final_rel": rel[-1], "min_rel": float(np.nanmin(rel)),
            "cycles_to_1e-3": drop, "ms_per_cycle": 1e3 * dt / max(done, 1),
            "hist": [rel[k] for k in range(0, len(rel), max(1, len(rel) // 50))]}


def main():
    out = {}
    cases = {
        "config2_naca_M0.5": (2, 600),
        "config3_cylinder_M8": (3, 600),
        "config4_sphere_M8": (4, 200),
    }
    for name, (k, ncyc) in cases.items():
        m = configs.config(k)
        fs = configs.FREESTREAM[k]
        W = state.uniform(m, *fs)
        Winf = state.winf(*fs)
        res = {}
        res["explicit_1level"] = run(m, W, Winf, ncyc * 10 if k != 4 else ncyc * 5, n_levels=1)
        for ns in ([1, 2, 4, 6, 8] if k != 4 else [2, 6]):
            res[f"sweeps{ns}"] = run(m, W, Winf, ncyc, n_sweeps=ns)
        for cfl in ([2.0, 5.0, 10.0, 20.0, 50.0, 100.0] if k != 4 else [10.0, 50.0]):
            res[f"cfl{cfl:g}"] = run(m, W, Winf, ncyc, cfl_imp=cfl)
        res["df_off"] = run(m, W, Winf, ncyc, df_mode=2)
        for b in ([0.25, 0.5, 0.75] if k != 4 else [0.5]):
            res[f"beta{b:g}"] = run(m, W, Winf, ncyc, df_mode=3, beta=b)
        out[name] = {"cells": m.n_cells, "runs": res}
        print(name, {kk: (v["ok"], round(v["final_rel"], 6) if v["ok"] else None, v["cycles_to_1e-3"],
                          round(v["ms_per_cycle"], 3)) for kk, v in res.items()}, flush=True)
    path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/studies.json"
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
