"""NEXT-1 convergence probe: residual history of the third-order-operator
V-cycle on config 2 (NACA0012, M 0.5, impulsive start) for a few settings of
the readings the paper defers (C5 WENO epsilon / linear weights, C9 collision
time).  One JSON line per setting: the density residual / r0 every 100 cycles.

    python tools/ho_conv.py [config] [cycles] [p1|cfl]
    python tools/ho_conv.py bump"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_06347_b200 import gmg  # noqa: E402
from synth import configs, state  # noqa: E402


def bump():
    """convected density bump on uniform meshes (64 x 64 quads / random-diagonal triangles, all far field,
    M 0.54): explicit 1-level iteration vs the 3-level V-cycle, both with the third-order operator"""
    for mname, m in [("quad64", configs.quad_grid(64, 64)), ("tri64", configs.tri_square(64, 64, seed=1))]:
        fs = (1.0, (0.5, 0.2), 1.0 / 1.4)
        W, Winf = state.gaussian_bump(m, *fs), state.winf(*fs)
        for nl, n, kw in [(1, 3000, dict(ho_gam0=1e-12)), (1, 3000, dict()), (1, 3000, dict(ho_gam0=1.0)),
                          (3, 600, dict()), (3, 600, dict(fine_operator=0))]:
            kw2 = dict(kw)
            fo = kw2.pop("fine_operator", 1)
            s = gmg.Solver(m, n_levels=nl, fine_operator=fo, **kw2)
            s.set_state(W, Winf)
            h = s.vcycle(n)
            r = h[:, 0] / h[0, 0]
            print(json.dumps({"mesh": mname, "levels": nl, "setting": kw, "iterations": n,
                              "rho_res_every_tenth": [float("%.3g" % x) for x in r[::n // 10]]}), flush=True)
            s.close()


def wall():
    """config 2 with the Euler-level no-slip ghost (as configured) vs a slip (inviscid) wall: is the plateau of
    the third-order operator a property of an inviscid flow with a no-slip ghost?"""
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    for kind in ("noslip", "slip"):
        m = configs.config(2)
        if kind == "slip":
            m.patch_kind = m.patch_kind.copy()
            m.patch_kind[0] = configs.SLIP
        fs = configs.FREESTREAM[2]
        W, Winf = state.uniform(m, *fs), state.winf(*fs)
        for fo in (1, 0):
            s = gmg.Solver(m, n_levels=3, fine_operator=fo)
            s.set_state(W, Winf)
            try:
                h = s.vcycle(n)
                r = h[:, 0] / h[0, 0]
                print(json.dumps({"wall": kind, "fine_operator": fo, "rho_res_every100": [float("%.3g" % x) for x in r[::100]],
                                  "min": float(r.min()), "final": float(r[-1])}), flush=True)
            except gmg.GmgError as e:
                print(json.dumps({"wall": kind, "fine_operator": fo, "error": str(e)[:80]}), flush=True)
            s.close()


def grids():
    """which O-grid property carries the third-order plateau: wall spacing, triangle layers, far-field radius"""
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    for kw in (dict(), dict(first=1e-2), dict(first=1e-3), dict(n_tri=0), dict(first=1e-2, n_tri=0),
               dict(n_quad=24, n_tri=8, ni=128), dict(r_out=5.0)):
        m = configs.naca_ogrid(**kw)
        fs = configs.FREESTREAM[2]
        W, Winf = state.uniform(m, *fs), state.winf(*fs)
        s = gmg.Solver(m, n_levels=3, fine_operator=1)
        s.set_state(W, Winf)
        try:
            h = s.vcycle(n)
            r = h[:, 0] / h[0, 0]
            print(json.dumps({"grid": kw, "cells": m.n_cells, "rho_res_every200": [float("%.3g" % x) for x in r[::200]],
                              "min": float(r.min()), "final": float(r[-1])}), flush=True)
        except gmg.GmgError as e:
            print(json.dumps({"grid": kw, "error": str(e)[:80]}), flush=True)
        s.close()


def knobs():
    """the default config-2 grid under the deferred-reading knobs: collision-time pressure term (C9 c2), WENO-Z
    epsilon (C5), linear weight (C5)"""
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    m = configs.config(2)
    fs = configs.FREESTREAM[2]
    W, Winf = state.uniform(m, *fs), state.winf(*fs)
    for kw in (dict(ho_c2=0.0), dict(ho_eps=1e-10), dict(ho_eps=1e-8), dict(ho_c2=0.0, ho_eps=1e-10),
               dict(ho_gam0=0.99), dict(ho_gam0=0.8), dict(cfl_exp=0.3)):
        s = gmg.Solver(m, n_levels=3, fine_operator=1, **kw)
        s.set_state(W, Winf)
        try:
            h = s.vcycle(n)
            r = h[:, 0] / h[0, 0]
            print(json.dumps({"setting": kw, "rho_res_every200": [float("%.3g" % x) for x in r[::200]],
                              "min": float(r.min()), "final": float(r[-1])}), flush=True)
        except gmg.GmgError as e:
            print(json.dumps({"setting": kw, "error": str(e)[:80]}), flush=True)
        s.close()


def long(n_total, **kw):
    """config 2, third-order operator, n_total V-cycles in chunks of 2000 (the history buffer holds 4096)"""
    m = configs.config(2)
    fs = configs.FREESTREAM[2]
    W, Winf = state.uniform(m, *fs), state.winf(*fs)
    s = gmg.Solver(m, n_levels=3, fine_operator=1, **kw)
    s.set_state(W, Winf)
    r0, out = None, []
    try:
        for _ in range(n_total // 2000):
            h = s.vcycle(2000)
            r0 = h[0, 0] if r0 is None else r0
            out += [float("%.3g" % (x / r0)) for x in h[:-1:250, 0]]
        print(json.dumps({"setting": kw, "rho_res_every250": out, "final": float(h[-1, 0] / r0)}), flush=True)
    except gmg.GmgError as e:
        print(json.dumps({"setting": kw, "error": str(e)[:80]}), flush=True)
    s.close()


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "long":   # long <cycles> [key=int ...]
        return long(int(sys.argv[2]), **{k: int(v) for k, v in (a.split("=") for a in sys.argv[3:])})
    if len(sys.argv) > 1 and sys.argv[1] == "knobs":
        return knobs()
    if len(sys.argv) > 1 and sys.argv[1] == "grids":
        return grids()
    if len(sys.argv) > 1 and sys.argv[1] == "bump":
        return bump()
    if len(sys.argv) > 1 and sys.argv[1] == "wall":
        return wall()
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    m = configs.config(k)
    fs = configs.FREESTREAM[k] if k == 2 else (1.0, (0.5, 0.0), 1.0 / 1.4)
    W, Winf = state.uniform(m, *fs), state.winf(*fs)
    sets = [dict(), dict(ho_eps=1e-6), dict(ho_gam0=1.0), dict(ho_c1=0.01), dict(ho_c1=0.2), dict(fine_operator=0)]
    mode = sys.argv[3] if len(sys.argv) > 3 else ""
    if mode == "p1":       # Green-Gauss only (gamma_0 -> 0) and intermediate linear weights
        sets = [dict(ho_gam0=1e-12), dict(ho_gam0=0.5), dict(ho_gam0=0.8)]
    elif mode == "cfl":    # explicit CFL of the fine pre-smoother
        sets = [dict(cfl_exp=0.2), dict(cfl_exp=0.1), dict(cfl_exp=0.2, ho_gam0=1.0), dict(cfl_exp=0.1, ho_gam0=1.0),
                dict(cfl_exp=0.2, ho_eps=1e-6)]
    for kw in sets:
        kw2 = dict(kw)
        fo = kw2.pop("fine_operator", 1)
        s = gmg.Solver(m, n_levels=3, fine_operator=fo, **kw2)
        s.set_state(W, Winf)
        try:
            h = s.vcycle(n)
        except gmg.GmgError as e:
            print(json.dumps({"config": k, "setting": kw, "error": str(e)[:80]}), flush=True)
            s.close()
            continue
        r = h[:, 0] / h[0, 0]
        print(json.dumps({"config": k, "setting": kw, "rho_res_every100": [float("%.3g" % x) for x in r[::100]],
                          "min": float(r.min())}), flush=True)
        s.close()


if __name__ == "__main__":
    main()
