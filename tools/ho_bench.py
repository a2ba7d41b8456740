"""NEXT-1 timing: the V-cycle with the third-order compact GKS fine operator
(fine_operator = 1) on a bench workload (default config 4, 1 M cells), next to
the first-order fine operator on the same mesh and state.  Per-kernel times
from CUDA events per launch (gmg_profile_vcycle).  One JSON line.

    python tools/ho_bench.py [--config 4] [--steps 20] [--profile-only]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--profile-only", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2509_06347_b200 import _build
    _build.build()
    from paper_2509_06347_b200 import gmg
    from bench import workload
    m, W, Winf = workload(args.config)
    out = {"config": args.config, "cells": m.n_cells, "faces": m.n_faces}
    for fo in ([1] if args.profile_only else [1, 0]):
        t0 = time.perf_counter()
        s = gmg.Solver(m, n_levels=3, device=0, fine_operator=fo, ho_geometry=fo == 1, setup_device=1)
        t_setup = time.perf_counter() - t0
        s.set_state(W, Winf)
        for _ in range(args.warmup):
            s.vcycle(1)
        s.set_state(W, Winf)
        if fo == 1:
            s.set_ho_state()
        if args.profile_only:
            s.vcycle(1)
            torch.cuda.synchronize()
            print(json.dumps({"profile_only": True}))
            return
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = torch.cuda.current_stream()
        e0.record(st)
        hist = s.vcycle(args.steps)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        s.set_state(W, Winf)
        if fo == 1:
            s.set_ho_state()
        pms, pcnt, pby = s.profile_vcycle(5)
        tot = float(pms.sum())
        key = "cgks3" if fo == 1 else "first_order"
        out[key] = {"ms_per_vcycle": ms, "setup_s": t_setup, "finite": bool(np.all(np.isfinite(hist))),
                    "hist_first_last": [hist[0].tolist(), hist[-1].tolist()],
                    "kernels": {gmg.K_NAMES[k]: {"ms_per_cycle": float(pms[k]) / 5,
                                                 "launches_per_cycle": int(pcnt[k]) // 5,
                                                 "share": float(pms[k]) / tot if tot else None,
                                                 "GB/s": float(pby[k] / (pms[k] * 1e-3) / 1e9) if pms[k] > 0 else None}
                                for k in range(gmg.K_COUNT) if pcnt[k] > 0}}
        if fo == 1:
            nf_gp = int(np.count_nonzero(m.gw))
            out[key]["gauss_points"] = nf_gp
            fl = out[key]["kernels"].get("ho_flux")
            if fl:
                fl["us_per_launch"] = fl["ms_per_cycle"] * 1e3 / max(fl["launches_per_cycle"], 1)
                fl["gauss_points_per_s"] = nf_gp / (fl["us_per_launch"] * 1e-6)
            _, fl_flags = s.ho_recon()
            out[key]["p2_cells"] = int(np.count_nonzero(fl_flags & 1))
        s.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
