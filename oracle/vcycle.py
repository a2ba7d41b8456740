"""Oracle hierarchy build + V-cycle orchestration.

TEST INFRASTRUCTURE (see oracle/__init__.py).  All arithmetic is in
gmg_oracle.c; this module calls the C steps in the order O8 states and
holds no floating-point work besides the history norms and the forcing
difference F = Res* - R(W0), written out as numpy expressions.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import (Level, agglomerate, coarse_build, color, diag, explicit_update,
               prolong, residual, restrict, smooth)


@dataclass
class Options:
    """Defaults: S:495, S:583, P:690-692, P:800 (six sweeps)."""
    gamma: float = 1.4
    cfl_imp: float = 10.0
    cfl_exp: float = 0.5
    n_sweeps: int = 6
    n_levels: int = 3
    pre_smooth: int = 1
    post_smooth: int = 0
    skew_limit: float = 0.5
    r_factor: float = 1.0
    fine_smoother: int = 0      # 0 explicit (paper), 1 MC-LU-SGS
    df_mode: int = 0            # 0 first-order helper, 1 user alpha, 2 alpha == 1, 3 fixed beta relaxation
    beta: float = 0.5           # df_mode 3: "traditional" fixed relaxation factor (reading B3)
    fine_operator: int = 0      # 0 first-order KFVS residual, 1 third-order CGKS (NEXT-1)
    c1: float = 0.05            # C9 collision time tau = c1 dt + c2 dt |pl-pr|/(pl+pr)
    c2: float = 1.0
    gam0: float = 0.95          # C5 linear weight of the large stencil
    p2min: int = 0              # C3 / C3b: interior neighbours p2 needs (0: d + 1)


def perm_from_color(col):
    """Renumbering: stable sort by (color, natural id) (O2)."""
    return np.lexsort((np.arange(col.shape[0]), col)).astype(np.int64)


def build_hierarchy(mesh, n_levels=3, theta=0.5, part=None):
    """Levels with their Algorithm-1 coloring and the fine->coarse parent.
    Stops early (stall) when a level merges nothing."""
    lv = Level.from_mesh(mesh) if not isinstance(mesh, Level) else mesh
    levels = []
    cur_part = None if part is None else np.ascontiguousarray(part, dtype=np.int32)
    while True:
        col, nc = color(lv)
        entry = {"level": lv, "color": col, "ncolor": nc, "parent": None, "part": cur_part}
        levels.append(entry)
        if len(levels) >= n_levels:
            break
        parent, ncoarse, merges = agglomerate(lv, theta, cur_part)
        if merges == 0:
            break
        entry["parent"] = parent
        lv = coarse_build(lv, parent, ncoarse)
        if cur_part is not None:
            cp = np.zeros(ncoarse, dtype=np.int32)
            cp[parent] = cur_part
            cur_part = cp
    return levels


def _norms(R):
    return np.sqrt((R * R).sum(axis=1))


def vcycle(levels, W0, Winf, opt: Options, n_cycles=1, user_alpha=None, trace=None, mesh=None, ho_state=None):
    """O8: n_cycles 3-level V-cycles (pre = 1, post = 0).  Returns the fine
    state and the history [n_cycles+1][nv] of per-component residual L2
    norms at each cycle start plus one final entry (reading A26).

    opt.fine_operator = 1 (NEXT-1, reading C14): the fine residual is the
    third-order CGKS operator of cgks3.c on `mesh` (a synth.Mesh with m2 /
    gp / gw); `ho_state` = {"G": [nv][d][n], "alpha": [n]} carries the
    cell-averaged slopes and the DF between calls (updated in place; default
    G = 0, alpha = 1, reading C1)."""
    if opt.pre_smooth != 1 or opt.post_smooth != 0:
        raise ValueError("oracle implements the paper's pre=1, post=0 (P:690)")
    if opt.fine_operator == 1:
        return _vcycle_cgks3(levels, W0, Winf, opt, n_cycles, mesh, ho_state)
    g, om = opt.gamma, opt.r_factor
    L = [e["level"] for e in levels]
    nl = len(L)
    W = np.array(W0, dtype=np.float64, copy=True)
    hist = []

    def fine_alpha(a):
        if opt.df_mode == 1:
            return np.asarray(user_alpha, dtype=np.float64)
        if opt.df_mode == 2:
            return np.ones_like(a)
        return a

    def relax(a):
        # the factor that blends the implicit and explicit operators in the
        # smoother: the DF alpha (Eq.(DF-relaxation-hybrid)), or a fixed
        # beta for the traditional relaxation of P:526-532 (reading B3)
        return np.full_like(a, opt.beta) if opt.df_mode == 3 else a

    for cyc in range(n_cycles):
        R0, a0, S0, rf0 = residual(L[0], W, Winf, g, om)
        a0 = fine_alpha(a0)
        hist.append(_norms(R0))
        # fine pre-smoothing
        if opt.fine_smoother == 0:
            W = explicit_update(W, S0, R0, opt.cfl_exp)
        else:
            D0 = diag(S0, relax(a0), opt.cfl_imp, opt.cfl_exp)
            dW = smooth(L[0], W, R0, relax(a0), D0, rf0, levels[0]["color"], levels[0]["ncolor"], opt.n_sweeps, g)
            W = W + dW
        if nl == 1:
            continue
        R0, a0, _, _ = residual(L[0], W, Winf, g, om)          # reading A10
        a0 = fine_alpha(a0)
        Wl = [W]
        W0l = [None]
        al = [a0]
        Rt_prev = R0
        for l in range(1, nl):
            par = levels[l - 1]["parent"]
            W0c, Rs, ac = restrict(par, L[l].n, L[l - 1].vol, L[l].vol, Wl[l - 1], Rt_prev, al[l - 1])
            Rc, _, Sc, rfc = residual(L[l], W0c, Winf, g, om)
            F = Rs - Rc
            Dl = diag(Sc, relax(ac), opt.cfl_imp, opt.cfl_exp)
            dW = smooth(L[l], W0c, Rs, relax(ac), Dl, rfc, levels[l]["color"], levels[l]["ncolor"], opt.n_sweeps, g)
            Wc = W0c + dW
            if trace is not None:
                trace.append({"level": l, "W0": W0c, "Rs": Rs, "alpha": ac, "dW": dW, "F": F})
            Wl.append(Wc)
            W0l.append(W0c)
            al.append(ac)
            if l < nl - 1:
                Rl, _, _, _ = residual(L[l], Wc, Winf, g, om)
                Rt_prev = Rl + F                                  # reading A8 / A11
        for l in range(nl - 1, 0, -1):
            Wl[l - 1] = prolong(levels[l - 1]["parent"], al[l - 1], Wl[l], W0l[l], Wl[l - 1])
        W = Wl[0]
    R0, _, _, _ = residual(L[0], W, Winf, g, om)
    hist.append(_norms(R0))
    return W, np.array(hist)


def _vcycle_cgks3(levels, W0, Winf, opt: Options, n_cycles, mesh, ho_state):
    """Reading C14: cycle start -> CGKS3 evaluation at (W, G, alpha) (history,
    explicit update Eq.(smo) with Dt_i = CFL_exp V_i / Sigma_i, new slopes and
    DF); a second evaluation at the updated state gives the restricted
    residual and the DF of restriction / prolongation, which is also the DF
    carried to the next p1 (its slopes are not used).  Coarse levels as O8."""
    from . import cgks3
    if opt.fine_smoother != 0 or opt.df_mode != 0:
        raise ValueError("the CGKS3 fine operator runs with the explicit fine smoother and DF mode 0")
    g, om = opt.gamma, opt.r_factor
    o3 = cgks3.Opt3(gamma=g, cfl_exp=opt.cfl_exp, c1=opt.c1, c2=opt.c2, gam0=opt.gam0, p2min=opt.p2min)
    M3 = cgks3.Mesh3(mesh)
    L = [e["level"] for e in levels]
    nl = len(L)
    d, n = mesh.dim, mesh.n_cells
    if ho_state is None:
        ho_state = {}
    G = ho_state.get("G")
    G = np.zeros((d + 2, d, n)) if G is None else np.array(G, dtype=np.float64)
    alpha = ho_state.get("alpha")
    alpha = np.ones(n) if alpha is None else np.array(alpha, dtype=np.float64)
    W = np.array(W0, dtype=np.float64, copy=True)
    hist = []
    for cyc in range(n_cycles):
        R0, Gn, a1, S0, _, _ = cgks3.residual(M3, W, G, alpha, Winf, o3)
        hist.append(_norms(R0))
        W = explicit_update(W, S0, R0, opt.cfl_exp)
        G, alpha = Gn, a1
        if nl == 1:
            continue
        R0, _, a0, _, _, _ = cgks3.residual(M3, W, G, alpha, Winf, o3)
        alpha = a0
        Wl, W0l, al = [W], [None], [a0]
        Rt_prev = R0
        for l in range(1, nl):
            par = levels[l - 1]["parent"]
            W0c, Rs, ac = restrict(par, L[l].n, L[l - 1].vol, L[l].vol, Wl[l - 1], Rt_prev, al[l - 1])
            Rc, _, Sc, rfc = residual(L[l], W0c, Winf, g, om)
            F = Rs - Rc
            Dl = diag(Sc, ac, opt.cfl_imp, opt.cfl_exp)
            dW = smooth(L[l], W0c, Rs, ac, Dl, rfc, levels[l]["color"], levels[l]["ncolor"], opt.n_sweeps, g)
            Wc = W0c + dW
            Wl.append(Wc)
            W0l.append(W0c)
            al.append(ac)
            if l < nl - 1:
                Rl, _, _, _ = residual(L[l], Wc, Winf, g, om)
                Rt_prev = Rl + F
        for l in range(nl - 1, 0, -1):
            Wl[l - 1] = prolong(levels[l - 1]["parent"], al[l - 1], Wl[l], W0l[l], Wl[l - 1])
        W = Wl[0]
    R0, _, _, _, _, _ = cgks3.residual(M3, W, G, alpha, Winf, o3)
    hist.append(_norms(R0))
    ho_state["G"], ho_state["alpha"] = G, alpha
    return W, np.array(hist)
