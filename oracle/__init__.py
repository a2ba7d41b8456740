"""CPU oracle for the GMG / MC-LU-SGS hot path (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with
the CUDA product path (paper_2509_06347_b200/) and never imports it.

The arithmetic lives in gmg_oracle.c (plain C, fp64, natural order,
-O2 -ffp-contract=off); this package only builds/loads it and orchestrates the
V-cycle (oracle/vcycle.py) in the order of SURVEY.md §8(c) O8.

Residual histories over many V-cycles have no printed values to pin against
(the paper's convergence curves are images without data):
they are pinned through their constituent steps and by invariants only -- the
free-stream fixed point and frame equivariance (a 90-degree rotation or a
reflection of mesh and velocities reproduces the 40-cycle 2D and 25-cycle 3D
histories with the momentum norms permuted, tests/test_oracle_pins.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gmg_oracle.c")
_SRC3 = os.path.join(_HERE, "cgks3.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """The parity build: -O2 -ffp-contract=off, sequential (the OpenMP pragmas are ignored)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC),
                                                                          os.path.getmtime(_SRC3)):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-o", _LIB, _SRC, _SRC3, "-lm"])
    return _LIB


def build_timing() -> str:
    """The timing build (bench.py's CPU baseline only): the same sources with
    -O3 -march=native -fopenmp -ffp-contract=off, compiled on THIS host (the
    -march=native code is host specific) into the temp directory, keyed by the
    sources and the CPU model.  Same results bit for bit as the parity build
    (tests/test_oracle_timing.py)."""
    import hashlib
    import tempfile
    h = hashlib.sha1()
    for f in (_SRC, _SRC3):
        h.update(open(f, "rb").read())
    try:
        h.update(open("/proc/cpuinfo", "rb").read().split(b"\n\n")[0])
    except OSError:
        pass
    out = os.path.join(tempfile.gettempdir(), f"liboracle_timing_{h.hexdigest()[:16]}.so")
    if not os.path.exists(out):
        tmp = out + f".{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=native", "-fopenmp", "-std=gnu11", "-ffp-contract=off",
                               "-fno-fast-math", "-fPIC", "-shared", "-o", tmp, _SRC, _SRC3, "-lm"])
        os.replace(tmp, out)
    return out


_parity_lib = None


def use_timing_build(threads: int):
    """Route the wrappers below to the timing build with `threads` OpenMP threads."""
    global _lib, _parity_lib
    if _parity_lib is None:
        _parity_lib = lib()
    L = C.CDLL(build_timing())
    _declare(L)
    L.omp_set_num_threads.argtypes = [C.c_int]
    L.omp_set_num_threads(int(threads))
    _lib = L


def use_parity_build():
    global _lib
    if _parity_lib is not None:
        _lib = _parity_lib


class OrcLevel(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_patches", C.c_int), ("n", C.c_int64), ("nf", C.c_int64),
                ("vol", C.c_void_p), ("ctr", C.c_void_p), ("left", C.c_void_p), ("right", C.c_void_p),
                ("avec", C.c_void_p), ("fctr", C.c_void_p), ("ngauss", C.c_void_p), ("patch_kind", C.c_void_p)]


class OrcLevelOut(C.Structure):
    _fields_ = [("vol", C.c_void_p), ("ctr", C.c_void_p), ("left", C.c_void_p), ("right", C.c_void_p),
                ("avec", C.c_void_p), ("fctr", C.c_void_p), ("ngauss", C.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        _declare(L)
        _lib = L
    return _lib


def _declare(L):
    if True:
        P = C.c_void_p
        L.orc_color.restype = C.c_int
        L.orc_color.argtypes = [C.c_int64, C.c_int64, P, P, P]
        L.orc_face_hash.restype = C.c_uint64
        L.orc_face_hash.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_skewness.restype = C.c_double
        L.orc_skewness.argtypes = [C.c_int, C.c_double, P, P, P]
        L.orc_agglomerate.restype = C.c_int64
        L.orc_agglomerate.argtypes = [C.POINTER(OrcLevel), C.c_double, P, P, P]
        L.orc_coarse_build.restype = C.c_int64
        L.orc_coarse_build.argtypes = [C.POINTER(OrcLevel), P, C.c_int64, C.POINTER(OrcLevelOut)]
        L.orc_kfvs_flux.restype = None
        L.orc_kfvs_flux.argtypes = [C.c_int, C.c_double, P, P, P, P]
        L.orc_df_face.restype = C.c_double
        L.orc_df_face.argtypes = [C.c_int, C.c_double, P, P, P]
        L.orc_spectral_radius.restype = C.c_double
        L.orc_spectral_radius.argtypes = [C.c_int, C.c_double, C.c_double, P, P, P]
        L.orc_euler_flux.restype = None
        L.orc_euler_flux.argtypes = [C.c_int, C.c_double, P, P, P]
        L.orc_residual.restype = None
        L.orc_residual.argtypes = [C.POINTER(OrcLevel), C.c_double, C.c_double, P, P, P, P, P, P]
        L.orc_diag.restype = None
        L.orc_diag.argtypes = [C.c_int64, P, P, C.c_double, C.c_double, P]
        L.orc_smooth.restype = None
        L.orc_smooth.argtypes = [C.POINTER(OrcLevel), C.c_double, P, P, P, P, P, P, C.c_int, C.c_int, P]
        L.orc_explicit_update.restype = None
        L.orc_explicit_update.argtypes = [C.c_int64, C.c_int, C.c_double, P, P, P]
        L.orc_restrict.restype = None
        L.orc_restrict.argtypes = [C.c_int64, C.c_int64, C.c_int, P, P, P, P, P, P, P, P, P]
        L.orc_prolong.restype = None
        L.orc_prolong.argtypes = [C.c_int64, C.c_int64, C.c_int, P, P, P, P, P]


def _p(a):
    return a.ctypes.data if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Level:
    """A mesh level in natural order (same fields as synth.Mesh)."""

    def __init__(self, dim, vol, ctr, left, right, avec, fctr, ngauss, patch_kind):
        self.dim = int(dim)
        self.vol = _f64(vol)
        self.ctr = _f64(ctr).reshape(dim, -1)
        self.left = np.ascontiguousarray(left, dtype=np.int64)
        self.right = np.ascontiguousarray(right, dtype=np.int64)
        self.avec = _f64(avec).reshape(dim, -1)
        self.fctr = _f64(fctr).reshape(dim, -1)
        self.ngauss = np.ascontiguousarray(ngauss, dtype=np.int8)
        self.patch_kind = np.ascontiguousarray(patch_kind, dtype=np.int32)
        self._s = OrcLevel(self.dim, len(self.patch_kind), self.vol.shape[0], self.left.shape[0],
                           _p(self.vol), _p(self.ctr), _p(self.left), _p(self.right), _p(self.avec),
                           _p(self.fctr), _p(self.ngauss), _p(self.patch_kind))

    @classmethod
    def from_mesh(cls, m):
        return cls(m.dim, m.vol, m.ctr, m.left, m.right, m.avec, m.fctr, m.ngauss, m.patch_kind)

    @property
    def n(self):
        return self.vol.shape[0]

    @property
    def nf(self):
        return self.left.shape[0]

    @property
    def nv(self):
        return self.dim + 2

    n_cells = n
    n_faces = nf

    def ref(self):
        return C.byref(self._s)


# ---------------------------------------------------------------------------
# thin wrappers (no arithmetic here)
# ---------------------------------------------------------------------------
def color(level: Level):
    col = np.zeros(level.n, dtype=np.int32)
    nc = lib().orc_color(level.n, level.nf, _p(level.left), _p(level.right), _p(col))
    return col, int(nc)


def face_hash(l, r, nf):
    return int(lib().orc_face_hash(l, r, nf))


def skewness(dim, sigma, A, x, Cv):
    A, x, Cv = _f64(A), _f64(x), _f64(Cv)
    return float(lib().orc_skewness(dim, sigma, _p(A), _p(x), _p(Cv)))


def agglomerate(level: Level, theta: float, part=None):
    parent = np.zeros(level.n, dtype=np.int64)
    nc = np.zeros(1, dtype=np.int64)
    pa = None if part is None else np.ascontiguousarray(part, dtype=np.int32)
    merges = lib().orc_agglomerate(level.ref(), theta, _p(pa), _p(parent), _p(nc))
    return parent, int(nc[0]), int(merges)


def coarse_build(level: Level, parent, nc) -> Level:
    parent = np.ascontiguousarray(parent, dtype=np.int64)
    nfc = lib().orc_coarse_build(level.ref(), _p(parent), nc, None)
    d = level.dim
    vol = np.zeros(nc)
    ctr = np.zeros((d, nc))
    left = np.zeros(nfc, dtype=np.int64)
    right = np.zeros(nfc, dtype=np.int64)
    avec = np.zeros((d, nfc))
    fctr = np.zeros((d, nfc))
    ng = np.zeros(nfc, dtype=np.int8)
    out = OrcLevelOut(_p(vol), _p(ctr), _p(left), _p(right), _p(avec), _p(fctr), _p(ng))
    lib().orc_coarse_build(level.ref(), _p(parent), nc, C.byref(out))
    return Level(d, vol, ctr, left, right, avec, fctr, ng, level.patch_kind)


def kfvs_flux(dim, gamma, WL, WR, n):
    F = np.zeros(dim + 2)
    WL, WR, n = _f64(WL), _f64(WR), _f64(n)
    lib().orc_kfvs_flux(dim, gamma, _p(WL), _p(WR), _p(n), _p(F))
    return F


def df_face(dim, gamma, WL, WR, n):
    WL, WR, n = _f64(WL), _f64(WR), _f64(n)
    return float(lib().orc_df_face(dim, gamma, _p(WL), _p(WR), _p(n)))


def spectral_radius(dim, gamma, omega, WL, WR, n):
    WL, WR, n = _f64(WL), _f64(WR), _f64(n)
    return float(lib().orc_spectral_radius(dim, gamma, omega, _p(WL), _p(WR), _p(n)))


def euler_flux(dim, gamma, W, n):
    T = np.zeros(dim + 2)
    W, n = _f64(W), _f64(n)
    lib().orc_euler_flux(dim, gamma, _p(W), _p(n), _p(T))
    return T


def residual(level: Level, W, Winf, gamma=1.4, omega=1.0):
    W = _f64(W)
    n, nv = level.n, level.nv
    R = np.zeros((nv, n))
    alpha = np.zeros(n)
    Sigma = np.zeros(n)
    rf = np.zeros(level.nf)
    Winf = _f64(Winf)
    lib().orc_residual(level.ref(), gamma, omega, _p(W), _p(Winf), _p(R), _p(alpha), _p(Sigma), _p(rf))
    return R, alpha, Sigma, rf


def diag(Sigma, alpha, cfl_imp, cfl_exp):
    Sigma, alpha = _f64(Sigma), _f64(alpha)
    D = np.zeros_like(Sigma)
    lib().orc_diag(Sigma.shape[0], _p(Sigma), _p(alpha), cfl_imp, cfl_exp, _p(D))
    return D


def smooth(level: Level, W, Rt, alpha, D, rf, col, ncolor, n_sweeps, gamma=1.4):
    dW = np.zeros((level.nv, level.n))
    W, Rt, alpha, D, rf = _f64(W), _f64(Rt), _f64(alpha), _f64(D), _f64(rf)
    col = np.ascontiguousarray(col, dtype=np.int32)
    lib().orc_smooth(level.ref(), gamma, _p(W), _p(Rt), _p(alpha), _p(D), _p(rf), _p(col), int(ncolor),
                     int(n_sweeps), _p(dW))
    return dW


def explicit_update(W, Sigma, R, cfl_exp):
    W = _f64(W).copy()
    Sigma, R = _f64(Sigma), _f64(R)
    lib().orc_explicit_update(W.shape[1], W.shape[0], cfl_exp, _p(Sigma), _p(R), _p(W))
    return W


def restrict(parent, nc, vol_f, vol_c, Wf, Rf, af):
    Wf, Rf = _f64(Wf), _f64(Rf)
    nv, nfine = Wf.shape
    W0c = np.zeros((nv, nc))
    Rc = np.zeros((nv, nc))
    ac = np.zeros(nc)
    parent = np.ascontiguousarray(parent, dtype=np.int64)
    vol_f, vol_c, af = _f64(vol_f), _f64(vol_c), _f64(af)
    lib().orc_restrict(nfine, nc, nv, _p(parent), _p(vol_f), _p(vol_c), _p(Wf), _p(Rf), _p(af), _p(W0c), _p(Rc),
                       _p(ac))
    return W0c, Rc, ac


def prolong(parent, alpha_f, Wc, W0c, Wf):
    Wf = _f64(Wf).copy()
    nv, nfine = Wf.shape
    parent = np.ascontiguousarray(parent, dtype=np.int64)
    alpha_f, Wc, W0c = _f64(alpha_f), _f64(Wc), _f64(W0c)
    lib().orc_prolong(nfine, Wc.shape[1], nv, _p(parent), _p(alpha_f), _p(Wc), _p(W0c), _p(Wf))
    return Wf


from .vcycle import Options, build_hierarchy, vcycle, perm_from_color  # noqa: E402,F401
