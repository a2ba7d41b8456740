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


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "bump":
        return bump()
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
