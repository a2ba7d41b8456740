"""Time-to-solution of the GPU multigrid vs the GPU explicit iteration on the
same mesh -- the structure of the paper's Table 5 ("GPU
explicit" vs "GPU multigrid" wall times), with this build's first-order KFVS
operator on every level, or (--operator cgks3, NEXT-4) the third-order
compact GKS fine operator of NEXT-1 on the fine level of both arms.

Both arms: impulsive free-stream start, CUDA-graph-replayed iterations on one
B200, wall time (device synchronised) until the fine residual (density
component, L2) drops below `target` x r0, or the iteration cap.  Explicit =
the 1-level hierarchy: the fine explicit update W -= (CFL_exp V/Sigma)/V R
every iteration (the V-cycle's pre-smoother alone).  Writes JSON."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_06347_b200 import gmg  # noqa: E402
from synth import configs, state  # noqa: E402


def solve(m, W, Winf, n_levels, cap, chunk, levels, fine_operator=0, p2min=0):
    """iterate to `cap` (or until the deepest level is reached); iterations and
    wall time (constant per iteration, graph replays) to each residual level"""
    kw = {"ho_p2min": p2min} if fine_operator else {}
    s = gmg.Solver(m, n_levels=n_levels, fine_operator=fine_operator, **kw)
    s.set_state(W, Winf)
    s.vcycle(1)                      # graph capture + warm-up, not timed
    s.set_state(W, Winf)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    done, r0 = 0, None
    hist = []
    while done < cap:
        h = s.vcycle(chunk)
        if r0 is None:
            r0 = float(h[0, 0])
        hist.extend((h[:-1, 0] / r0).tolist())
        done += chunk
        if min(hist) <= min(levels):
            break
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    s.close()
    per = dt / done
    out = {"iterations": done, "wall_s": dt, "ms_per_iteration": 1e3 * per, "final_rel": hist[-1]}
    for lv in levels:
        k = next((i for i, x in enumerate(hist) if x <= lv), None)
        out[f"to_{lv:g}"] = None if k is None else {"iterations": k, "wall_s": k * per}
    return out


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--operator", default="first", choices=["first", "cgks3"])
    ap.add_argument("--c3b", action="store_true", help="cgks3 with reading C3b (ho_p2min = d + 2)")
    args = ap.parse_args()
    fo = 1 if args.operator == "cgks3" else 0
    out = {"fine_operator": args.operator, "reading": "C3b" if args.c3b else "C3"}
    cases = [
        # name, mesh config, free stream, initial state, target, caps
        ("config2_naca_M0.5", 2, configs.FREESTREAM[2], "uniform", 1e-3, 2000, 400000),
        ("config4_sphere_M0.5", 4, (1.0, (0.5, 0.0, 0.0), 1.0 / 1.4), "uniform", 1e-3, 2000, 100000),
        ("config3_cylinder_M0.5", 3, (1.0, (0.5, 0.0), 1.0 / 1.4), "uniform", 1e-3, 2000, 200000),
    ]
    if fo:
        # NEXT-4 with the third-order CGKS fine operator (NEXT-1): "GPU explicit" is the 1-level
        # iteration of the same operator, as the paper's Table 5 compares
        cases = [
            ("config2_naca_M0.5", 2, configs.FREESTREAM[2], "uniform", 1e-3, 2000, 100000),
            ("config3_cylinder_M0.5", 3, (1.0, (0.5, 0.0), 1.0 / 1.4), "uniform", 1e-3, 1000, 40000),
        ]
    levels = (1e-1, 1e-2, 1e-3)
    if fo and args.c3b:
        # C3b converges the config-2 V-cycle: deeper levels; the M 0.5 cylinder's wake is unsteady
        cases = [("config2_naca_M0.5", 2, configs.FREESTREAM[2], "uniform", 1e-6, 6000, 400000)]
        levels = (1e-1, 1e-2, 1e-3, 1e-4, 1e-6)
    for name, k, fs, init, target, cap_gmg, cap_exp in cases:
        m = configs.config(k)
        W, Winf = state.uniform(m, *fs), state.winf(*fs)
        p2 = m.dim + 2 if args.c3b else 0
        g = solve(m, W, Winf, 3, cap_gmg, 50, levels, fo, p2)
        e = solve(m, W, Winf, 1, cap_exp, 2000, levels, fo, p2)
        sp = {}
        for lv in levels:
            a, b = g[f"to_{lv:g}"], e[f"to_{lv:g}"]
            if a and b and a["wall_s"] > 0:
                sp[f"{lv:g}"] = {"wall_time_ratio": b["wall_s"] / a["wall_s"],
                                 "iteration_ratio": b["iterations"] / max(a["iterations"], 1)}
        out[name] = {"cells": int(m.vol.size), "gpu_multigrid": g, "gpu_explicit": e,
                     "explicit_over_multigrid": sp}
        print(json.dumps({name: {"cells": out[name]["cells"], "speedups": sp}}), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/table5%s%s.json" % ("_cgks3" if fo else "", "_c3b" if args.c3b else ""), "w"),
              indent=1)


if __name__ == "__main__":
    main()
