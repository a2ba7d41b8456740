"""Oracle wrappers for the third-order compact GKS fine operator (NEXT-1;
DESIGN.md §12, readings C1-C14).  TEST INFRASTRUCTURE (see oracle/__init__.py):
the arithmetic is in cgks3.c; these are ctypes marshalling helpers only."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _f64, _p, lib

P_ = C.c_void_p


class Orc3Mesh(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_patches", C.c_int), ("G", C.c_int), ("n", C.c_int64), ("nf", C.c_int64),
                ("vol", P_), ("ctr", P_), ("m2", P_), ("left", P_), ("right", P_), ("avec", P_), ("gp", P_),
                ("gw", P_), ("patch_kind", P_)]


class Orc3Opt(C.Structure):
    _fields_ = [("gamma", C.c_double), ("cfl_exp", C.c_double), ("c1", C.c_double), ("c2", C.c_double),
                ("gam0", C.c_double), ("eps", C.c_double), ("p2min", C.c_int)]


@dataclass
class Opt3:
    """Readings C5, C8, C9."""
    gamma: float = 1.4
    cfl_exp: float = 0.5
    c1: float = 0.05
    c2: float = 1.0
    gam0: float = 0.95
    eps: float = 1e-14
    p2min: int = 0             # C3: p2 needs >= p2min interior neighbours (0: d + 1); C3b: d + 2

    def c(self):
        return Orc3Opt(self.gamma, self.cfl_exp, self.c1, self.c2, self.gam0, self.eps, self.p2min)


def _lib3():
    L = lib()
    if not getattr(L, "_c3", False):
        L.orc3_gks_local.restype = None
        L.orc3_gks_local.argtypes = [C.c_int, C.c_double, P_, P_, P_, P_, C.c_double, C.c_double, P_, P_]
        L.orc3_gks_flux.restype = None
        L.orc3_gks_flux.argtypes = [C.c_int, C.c_double, P_, P_, P_, P_, P_, C.c_double, C.c_double, P_, P_]
        L.orc3_p2.restype = C.c_int
        L.orc3_p2.argtypes = [C.POINTER(Orc3Mesh), P_, C.c_int, C.c_int64, P_, P_, P_]
        L.orc3_recon.restype = C.c_int64
        L.orc3_recon.argtypes = [C.POINTER(Orc3Mesh), C.POINTER(Orc3Opt), P_, P_, P_, P_, P_, P_]
        L.orc3_residual.restype = C.c_int64
        L.orc3_residual.argtypes = [C.POINTER(Orc3Mesh), C.POINTER(Orc3Opt), P_, P_, P_, P_, P_, P_, P_, P_, P_]
        L._c3 = True
    return L


class Mesh3:
    """The fine level with its high-order geometry (synth.Mesh m2 / gp / gw)."""

    def __init__(self, m):
        self.dim = m.dim
        self.vol, self.ctr, self.m2 = _f64(m.vol), _f64(m.ctr), _f64(m.m2)
        self.left = np.ascontiguousarray(m.left, dtype=np.int64)
        self.right = np.ascontiguousarray(m.right, dtype=np.int64)
        self.avec, self.gp, self.gw = _f64(m.avec), _f64(m.gp), _f64(m.gw)
        self.patch_kind = np.ascontiguousarray(m.patch_kind, dtype=np.int32)
        self.G = self.gw.shape[0]
        self._s = Orc3Mesh(self.dim, len(self.patch_kind), self.G, self.vol.shape[0], self.left.shape[0],
                           _p(self.vol), _p(self.ctr), _p(self.m2), _p(self.left), _p(self.right), _p(self.avec),
                           _p(self.gp), _p(self.gw), _p(self.patch_kind))

    @property
    def n(self):
        return self.vol.shape[0]


def gks_local(dim, gamma, Wl, dWl, Wr, dWr, dt, tau):
    """Flux (time-integrated, per unit area) and Gauss-point state in the local
    frame; dW [d][nv] derivatives along the local axes."""
    F, Wt = np.zeros(dim + 2), np.zeros(dim + 2)
    a = [_f64(x) for x in (Wl, dWl, Wr, dWr)]
    _lib3().orc3_gks_local(dim, gamma, *(_p(x) for x in a), dt, tau, _p(F), _p(Wt))
    return F, Wt


def gks_flux(dim, gamma, Wl, dWl, Wr, dWr, n, dt, tau):
    """Global frame: dW [d][nv] with dW[c][q] = dW_q/dx_c; n unit normal l -> r."""
    F, Wt = np.zeros(dim + 2), np.zeros(dim + 2)
    a = [_f64(x) for x in (Wl, dWl, Wr, dWr, n)]
    _lib3().orc3_gks_flux(dim, gamma, *(_p(x) for x in a), dt, tau, _p(F), _p(Wt))
    return F, Wt


def p2(M: Mesh3, cell, nbrs, Qbar, Qgrad):
    """p2 coefficients (lin[d], quad[nq]) of one component, or None (C3)."""
    nb = np.ascontiguousarray(nbrs, dtype=np.int64)
    a = np.zeros(9)
    Qbar, Qgrad = _f64(Qbar), _f64(Qgrad)
    ok = _lib3().orc3_p2(C.byref(M._s), _p(nb), len(nb), cell, _p(Qbar), _p(Qgrad), _p(a))
    d = M.dim
    return a[:d + d * (d + 1) // 2] if ok else None


def residual(M: Mesh3, W, G, alpha, Winf, opt: Opt3 = None):
    """One evaluation of the third-order operator: R [nv][n] (time-averaged
    flux sum), Gnew [nv][d][n], alpha [n], Sigma [n], flags [n], n_fallback."""
    opt = opt or Opt3()
    d, n = M.dim, M.n
    nv = d + 2
    W, G, alpha, Winf = _f64(W), _f64(G), _f64(alpha), _f64(Winf)
    R = np.zeros((nv, n))
    Gn = np.zeros((nv, d, n))
    a = np.zeros(n)
    S = np.zeros(n)
    fl = np.zeros(n, dtype=np.int32)
    o = opt.c()
    nfall = _lib3().orc3_residual(C.byref(M._s), C.byref(o), _p(W), _p(G), _p(alpha), _p(Winf), _p(R), _p(Gn),
                                  _p(a), _p(S), _p(fl))
    return R, Gn, a, S, fl, int(nfall)


def recon(M: Mesh3, W, G, alpha, Winf, opt: Opt3 = None):
    """Final per-cell polynomials poly [n][nv][1+d+nq] (c0, lin, quad about the
    centroid), flags [n] (bit 0 p2 used), 0 (positivity is per Gauss point, C6b)."""
    opt = opt or Opt3()
    d, n = M.dim, M.n
    nv, nc = d + 2, 1 + d + d * (d + 1) // 2
    W, G, alpha, Winf = _f64(W), _f64(G), _f64(alpha), _f64(Winf)
    poly = np.zeros((n, nv, nc))
    fl = np.zeros(n, dtype=np.int32)
    o = opt.c()
    nfall = _lib3().orc3_recon(C.byref(M._s), C.byref(o), _p(W), _p(G), _p(alpha), _p(Winf), _p(poly), _p(fl))
    return poly, fl, int(nfall)
