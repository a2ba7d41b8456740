"""Thin ctypes binding of libgmg (include/gmg.h) -- argument marshalling only.

Every step of the hot path runs in libgmg's sm_100a kernels; this module
never computes anything and has no CPU fallback: if libgmg.so is missing or
no CUDA device is present, the compute calls raise.

Names mirror the C ABI (gmg_create, gmg_load_mesh, ...); `Solver` bundles
them with a torch-allocated device workspace and torch's current stream
(PyTorch is used for device memory and streams only).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIBPATH = os.path.join(_HERE, "libgmg.so")

GMG_OK, GMG_EINVAL, GMG_ETOPO, GMG_ECOLOR, GMG_ESTALL, GMG_ENOMEM, GMG_ECUDA, GMG_ENCCL, GMG_ENONFINITE, GMG_ESTATE = range(10)
STATUS = ["GMG_OK", "GMG_EINVAL", "GMG_ETOPO", "GMG_ECOLOR", "GMG_ESTALL", "GMG_ENOMEM", "GMG_ECUDA", "GMG_ENCCL",
          "GMG_ENONFINITE", "GMG_ESTATE"]
K_FACE, K_GATHER, K_SWEEP, K_RESTRICT, K_PROLONG, K_NORM, K_HO_RECON, K_HO_FLUX, K_HALO, K_COUNT = range(10)
K_NAMES = ["face", "gather", "sweep", "restrict", "prolong", "norm", "ho_recon", "ho_flux", "halo"]
# gmg_get_level_field fields (include/gmg.h)
FIELD_W, FIELD_W0, FIELD_DW, FIELD_RS, FIELD_F, FIELD_RT, FIELD_ALPHA = range(7)

# every symbol include/gmg.h declares
ABI_SYMBOLS = ["gmg_set_state_owned_async", "gmg_get_state_owned_async", "gmg_set_state_async", "gmg_vcycle_async", "gmg_get_state_async", "gmg_sync",
               "gmg_load_ho_geometry", "gmg_set_ho_state", "gmg_get_ho_state", "gmg_ho_residual", "gmg_ho_recon",
               "gmg_default_options", "gmg_create", "gmg_load_mesh", "gmg_set_coloring", "gmg_build_hierarchy",
               "gmg_get_level_info", "gmg_get_maps", "gmg_get_level_geometry", "gmg_workspace_bytes",
               "gmg_set_workspace", "gmg_set_state", "gmg_set_level_state", "gmg_get_state", "gmg_set_alpha",
               "gmg_residual", "gmg_set_level_inputs", "gmg_smooth", "gmg_vcycle", "gmg_profile_vcycle",
               "gmg_time_smooth", "gmg_vcycle_launches", "gmg_vcycle_visits", "gmg_get_level_field", "gmg_partition_rcb", "gmg_get_halo", "gmg_p2p_layout",
               "gmg_p2p_import", "gmg_get_p2p_targets", "gmg_p2p_emulate_smooth", "gmg_last_error", "gmg_destroy"]


class GmgError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS[status] if 0 <= status < len(STATUS) else status}: {msg}")
        self.status = status


class Options(C.Structure):
    _fields_ = [("dim", C.c_int), ("gamma", C.c_double), ("cfl_imp", C.c_double), ("cfl_exp", C.c_double),
                ("n_sweeps", C.c_int), ("n_levels", C.c_int), ("pre_smooth", C.c_int), ("post_smooth", C.c_int),
                ("skew_limit", C.c_double), ("r_factor", C.c_double), ("fine_smoother", C.c_int),
                ("df_mode", C.c_int), ("rank", C.c_int), ("nranks", C.c_int), ("nccl_id", C.c_void_p),
                ("device", C.c_int), ("stream", C.c_void_p), ("beta", C.c_double), ("local_domains", C.c_int),
                ("setup_device", C.c_int), ("fine_operator", C.c_int), ("ho_c1", C.c_double), ("ho_c2", C.c_double),
                ("ho_gam0", C.c_double), ("ho_eps", C.c_double), ("skip_repeat", C.c_int), ("p2p", C.c_int),
                ("overlap", C.c_int), ("l2_persist_mb", C.c_int), ("sweep_lanes", C.c_int), ("pdl", C.c_int),
                ("ho_p2min", C.c_int)]


_lib = None


def lib():
    """Load libgmg.so (build it first with paper_2509_06347_b200._build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIBPATH):
            raise ImportError(f"{LIBPATH} missing: run `python -m paper_2509_06347_b200._build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIBPATH)
        P, I64, I, D = C.c_void_p, C.c_int64, C.c_int, C.c_double
        sig = {
            "gmg_default_options": (None, [C.POINTER(Options)]),
            "gmg_create": (I, [C.POINTER(Options), C.POINTER(P)]),
            "gmg_load_mesh": (I, [P, I64, P, P, I64, P, P, P, P, P, I, P, P]),
            "gmg_set_coloring": (I, [P, I, P]),
            "gmg_build_hierarchy": (I, [P, I, C.POINTER(I)]),
            "gmg_get_level_info": (I, [P, I, C.POINTER(I64), C.POINTER(I), C.POINTER(I64)]),
            "gmg_get_maps": (I, [P, I, P, P, P]),
            "gmg_get_level_geometry": (I, [P, I, P, P, P, P, P, P, P]),
            "gmg_workspace_bytes": (C.c_size_t, [P]),
            "gmg_set_workspace": (I, [P, P, C.c_size_t]),
            "gmg_set_state": (I, [P, P, P]),
            "gmg_set_level_state": (I, [P, I, P]),
            "gmg_get_state": (I, [P, I, P]),
            "gmg_set_alpha": (I, [P, P]),
            "gmg_residual": (I, [P, I, P, P, P]),
            "gmg_set_level_inputs": (I, [P, I, P, P]),
            "gmg_smooth": (I, [P, I, I, P]),
            "gmg_vcycle": (I, [P, I, P]),
            "gmg_profile_vcycle": (I, [P, I, P, P, P]),
            "gmg_time_smooth": (I, [P, I, I, I, P, P, P]),
            "gmg_vcycle_launches": (I64, [P]),
            "gmg_vcycle_visits": (I64, [P]),
            "gmg_get_level_field": (I, [P, I, I, P]),
            "gmg_partition_rcb": (I, [I64, I, P, I, P]),
            "gmg_get_halo": (I, [P, I, I, P, P, P, P, P, P, P, P, P, P, P, P]),
            "gmg_p2p_layout": (I, [P, P]),
            "gmg_p2p_import": (I, [P, P, P, P]),
            "gmg_get_p2p_targets": (I, [P, I, I, P, P, P, P]),
            "gmg_p2p_emulate_smooth": (I, [P, I, I, P]),
            "gmg_set_state_owned_async": (I, [P, P, P]),
            "gmg_get_state_owned_async": (I, [P, P]),
            "gmg_set_state_async": (I, [P, P, P]),
            "gmg_vcycle_async": (I, [P, I]),
            "gmg_get_state_async": (I, [P, P]),
            "gmg_sync": (I, [P]),
            "gmg_load_ho_geometry": (I, [P, P, I, P, P]),
            "gmg_set_ho_state": (I, [P, P, P]),
            "gmg_get_ho_state": (I, [P, P, P]),
            "gmg_ho_residual": (I, [P, P, P, P, P]),
            "gmg_ho_recon": (I, [P, P, P]),
            "gmg_last_error": (C.c_char_p, [P]),
            "gmg_destroy": (None, [P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ptr(a, count=None):
    """Raw pointer of a float64-or-index buffer.  With `count` (the doubles the
    call reads or writes) the buffer must be float64, contiguous and at least
    that large: a mismatched buffer would otherwise be read or written out of
    bounds by the library."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if count is not None:
            import torch
            if a.dtype != torch.float64 or not a.is_contiguous() or a.numel() < count:
                raise ValueError(f"need a contiguous float64 tensor of >= {count} elements, got {a.dtype} "
                                 f"{tuple(a.shape)} contiguous={a.is_contiguous()}")
        return a.data_ptr()
    if count is not None and (a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"] or a.size < count):
        raise ValueError(f"need a C-contiguous float64 array of >= {count} elements, got {a.dtype} {a.shape}")
    return a.ctypes.data


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# C-ABI names (marshalling only)
# ---------------------------------------------------------------------------
def gmg_default_options(**kw) -> Options:
    o = Options()
    lib().gmg_default_options(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def _check(ctx, st, allow=()):
    if st != GMG_OK and st not in allow:
        msg = lib().gmg_last_error(ctx)
        raise GmgError(st, msg.decode() if msg else "")
    return st


_NV = {}   # context handle -> nv (for the buffer-size checks of the wrappers)


def _nv(ctx):
    return _NV.get(ctx.value if hasattr(ctx, "value") else ctx, 1)


def gmg_create(opt: Options):
    h = C.c_void_p()
    st = lib().gmg_create(C.byref(opt), C.byref(h))
    if st != GMG_OK:
        raise GmgError(st, "gmg_create: invalid options")
    _NV[h.value] = opt.dim + 2
    return h


def gmg_load_mesh(ctx, mesh, part=None):
    keep = [_f64(mesh.vol), _f64(mesh.ctr), np.ascontiguousarray(mesh.left, np.int64),
            np.ascontiguousarray(mesh.right, np.int64), _f64(mesh.avec), _f64(mesh.fctr),
            np.ascontiguousarray(mesh.ngauss, np.int8), np.ascontiguousarray(mesh.patch_kind, np.int32),
            None if part is None else np.ascontiguousarray(part, np.int32)]
    vol, ctr, left, right, avec, fctr, ng, pk, pa = keep
    return _check(ctx, lib().gmg_load_mesh(ctx, vol.shape[0], _ptr(vol), _ptr(ctr), left.shape[0], _ptr(left),
                                           _ptr(right), _ptr(avec), _ptr(fctr), _ptr(ng), pk.shape[0], _ptr(pk),
                                           _ptr(pa)))


def gmg_set_coloring(ctx, level, color):
    c = None if color is None else np.ascontiguousarray(color, np.int32)
    return _check(ctx, lib().gmg_set_coloring(ctx, level, _ptr(c)))


def gmg_build_hierarchy(ctx, n_levels):
    nb = C.c_int(0)
    st = _check(ctx, lib().gmg_build_hierarchy(ctx, n_levels, C.byref(nb)), allow=(GMG_ESTALL,))
    return nb.value, st


def gmg_get_level_info(ctx, level):
    n, nc, nf = C.c_int64(), C.c_int(), C.c_int64()
    _check(ctx, lib().gmg_get_level_info(ctx, level, C.byref(n), C.byref(nc), C.byref(nf)))
    return n.value, nc.value, nf.value


def gmg_get_maps(ctx, level):
    n, _, _ = gmg_get_level_info(ctx, level)
    color = np.zeros(n, np.int32)
    perm = np.zeros(n, np.int64)
    parent = np.zeros(n, np.int64)
    _check(ctx, lib().gmg_get_maps(ctx, level, _ptr(color), _ptr(perm), _ptr(parent)))
    return color, perm, parent


def gmg_get_level_geometry(ctx, level, dim):
    n, _, nf = gmg_get_level_info(ctx, level)
    out = dict(vol=np.zeros(n), ctr=np.zeros((dim, n)), left=np.zeros(nf, np.int64), right=np.zeros(nf, np.int64),
               avec=np.zeros((dim, nf)), fctr=np.zeros((dim, nf)), ngauss=np.zeros(nf, np.int8))
    _check(ctx, lib().gmg_get_level_geometry(ctx, level, *(_ptr(out[k]) for k in
                                                           ("vol", "ctr", "left", "right", "avec", "fctr", "ngauss"))))
    return out


def gmg_workspace_bytes(ctx):
    return int(lib().gmg_workspace_bytes(ctx))


def gmg_set_workspace(ctx, dptr, nbytes):
    return _check(ctx, lib().gmg_set_workspace(ctx, dptr, nbytes))


def gmg_set_state(ctx, W, W_inf):
    Wk = W if hasattr(W, "data_ptr") else _f64(W)
    wi = _f64(W_inf)
    n, _, _ = gmg_get_level_info(ctx, 0)
    return _check(ctx, lib().gmg_set_state(ctx, _ptr(Wk, _nv(ctx) * n), _ptr(wi, _nv(ctx))))


def gmg_set_level_state(ctx, level, W):
    Wk = W if hasattr(W, "data_ptr") else _f64(W)
    n, _, _ = gmg_get_level_info(ctx, level)
    return _check(ctx, lib().gmg_set_level_state(ctx, level, _ptr(Wk, _nv(ctx) * n)))


def gmg_get_state(ctx, level, out):
    n, _, _ = gmg_get_level_info(ctx, level)
    return _check(ctx, lib().gmg_get_state(ctx, level, _ptr(out, _nv(ctx) * n)))


def gmg_get_level_field(ctx, level, field, out):
    n, _, _ = gmg_get_level_info(ctx, level)
    return _check(ctx, lib().gmg_get_level_field(ctx, level, field, _ptr(out, (1 if field == FIELD_ALPHA else _nv(ctx)) * n)))


def gmg_set_alpha(ctx, alpha):
    a = alpha if hasattr(alpha, "data_ptr") else _f64(alpha)
    return _check(ctx, lib().gmg_set_alpha(ctx, _ptr(a)))


def gmg_residual(ctx, level, R_out=None, alpha_out=None, sigma_out=None):
    return _check(ctx, lib().gmg_residual(ctx, level, _ptr(R_out), _ptr(alpha_out), _ptr(sigma_out)))


def gmg_set_level_inputs(ctx, level, Rt=None, alpha=None):
    R = None if Rt is None else (Rt if hasattr(Rt, "data_ptr") else _f64(Rt))
    a = None if alpha is None else (alpha if hasattr(alpha, "data_ptr") else _f64(alpha))
    return _check(ctx, lib().gmg_set_level_inputs(ctx, level, _ptr(R), _ptr(a)))


def gmg_smooth(ctx, level, n_sweeps, dW_out=None):
    return _check(ctx, lib().gmg_smooth(ctx, level, n_sweeps, _ptr(dW_out)))


def gmg_vcycle(ctx, n_cycles, res_hist=None):
    return _check(ctx, lib().gmg_vcycle(ctx, n_cycles, _ptr(res_hist)))


def gmg_profile_vcycle(ctx, n_cycles):
    ms = np.zeros(K_COUNT)
    cnt = np.zeros(K_COUNT, np.int64)
    by = np.zeros(K_COUNT)
    _check(ctx, lib().gmg_profile_vcycle(ctx, n_cycles, _ptr(ms), _ptr(cnt), _ptr(by)))
    return ms, cnt, by


def gmg_time_smooth(ctx, level, n_sweeps, reps):
    ms, cu, by = C.c_double(), C.c_double(), C.c_double()
    _check(ctx, lib().gmg_time_smooth(ctx, level, n_sweeps, reps, C.byref(ms), C.byref(cu), C.byref(by)))
    return ms.value, cu.value, by.value


def gmg_vcycle_launches(ctx):
    return int(lib().gmg_vcycle_launches(ctx))


def gmg_vcycle_visits(ctx):
    return int(lib().gmg_vcycle_visits(ctx))


def gmg_partition_rcb(ctr, nparts):
    """a5: recursive coordinate bisection of centroids [dim][n] -> part[n]."""
    ctr = _f64(ctr)
    dim, n = ctr.shape
    part = np.zeros(n, np.int32)
    st = lib().gmg_partition_rcb(n, dim, _ptr(ctr), nparts, _ptr(part))
    if st != GMG_OK:
        raise GmgError(st, "gmg_partition_rcb")
    return part


def gmg_get_halo(ctx, level, dom=0):
    """Halo plan of a local domain (natural ids); see include/gmg.h."""
    no, ng, npr, ns, nr = C.c_int64(), C.c_int64(), C.c_int(), C.c_int64(), C.c_int64()
    _check(ctx, lib().gmg_get_halo(ctx, level, dom, C.byref(no), C.byref(ng), C.byref(npr), C.byref(ns), C.byref(nr),
                                   None, None, None, None, None, None, None))
    _, nc, _ = gmg_get_level_info(ctx, level)
    out = dict(owned=np.zeros(no.value, np.int64), ghost=np.zeros(ng.value, np.int64),
               peers=np.zeros(npr.value, np.int32), send=np.zeros(ns.value, np.int64),
               send_off=np.zeros(nc * npr.value + 1, np.int64), recv=np.zeros(nr.value, np.int64),
               recv_off=np.zeros(nc * npr.value + 1, np.int64))
    _check(ctx, lib().gmg_get_halo(ctx, level, dom, None, None, None, None, None,
                                   *(_ptr(out[k]) for k in ("owned", "ghost", "peers", "send", "send_off", "recv",
                                                            "recv_off"))))
    out["n_colors"] = nc
    return out


def gmg_p2p_layout(ctx, n_levels):
    out = np.zeros(n_levels + 1, np.int64)
    _check(ctx, lib().gmg_p2p_layout(ctx, _ptr(out)))
    return out


def gmg_p2p_import(ctx, handles, base_off, layouts):
    """handles: nranks x 64-byte cudaIpcMemHandle_t; base_off: [nranks] int64;
    layouts: [nranks][n_levels + 1] int64 (each rank's gmg_p2p_layout)."""
    hb = np.frombuffer(b"".join(bytes(h).ljust(64, b"\0")[:64] for h in handles), np.uint8).copy()
    bo = np.ascontiguousarray(base_off, np.int64)
    ly = np.ascontiguousarray(layouts, np.int64)
    _check(ctx, lib().gmg_p2p_import(ctx, _ptr(hb), _ptr(bo), _ptr(ly)))


def gmg_get_p2p_targets(ctx, level, dom=0):
    """Fused-halo targets of a domain (see include/gmg.h): (off, peer_slot, ghost_local)."""
    nt = C.c_int64()
    _check(ctx, lib().gmg_get_p2p_targets(ctx, level, dom, C.byref(nt), None, None, None))
    h = gmg_get_halo(ctx, level, dom)
    off = np.zeros(len(h["owned"]) + 1, np.int32)
    k = np.zeros(nt.value, np.int32)
    g = np.zeros(nt.value, np.int32)
    _check(ctx, lib().gmg_get_p2p_targets(ctx, level, dom, None, _ptr(off), _ptr(k), _ptr(g)))
    return off, k, g


def gmg_p2p_emulate_smooth(ctx, level, n_sweeps, nv, n):
    """Test only: all local domains' smoothing step in one cooperative launch (see include/gmg.h)."""
    dW = np.zeros((nv, n))
    _check(ctx, lib().gmg_p2p_emulate_smooth(ctx, level, n_sweeps, _ptr(dW)))
    return dW


def gmg_set_state_async(ctx, W, W_inf):
    """W: pinned host tensor / device tensor / array that stays alive until gmg_sync"""
    Wi = _f64(W_inf)
    n, _, _ = gmg_get_level_info(ctx, 0)
    _check(ctx, lib().gmg_set_state_async(ctx, _ptr(W, _nv(ctx) * n), _ptr(Wi, _nv(ctx))))


def gmg_set_state_owned_async(ctx, W_owned, W_inf):
    """W_owned[nv][n_own]: this rank's owned cells in gmg_get_halo(level 0) "owned" order"""
    Wi = _f64(W_inf)
    _check(ctx, lib().gmg_set_state_owned_async(ctx, _ptr(W_owned), _ptr(Wi)))


def gmg_get_state_owned_async(ctx, W_owned_out):
    _check(ctx, lib().gmg_get_state_owned_async(ctx, _ptr(W_owned_out)))


def gmg_vcycle_async(ctx, n_cycles):
    _check(ctx, lib().gmg_vcycle_async(ctx, int(n_cycles)))


def gmg_get_state_async(ctx, W_out):
    n, _, _ = gmg_get_level_info(ctx, 0)
    _check(ctx, lib().gmg_get_state_async(ctx, _ptr(W_out, _nv(ctx) * n)))


def gmg_sync(ctx):
    _check(ctx, lib().gmg_sync(ctx))


def gmg_load_ho_geometry(ctx, mesh):
    m2, gp, gw = _f64(mesh.m2), _f64(mesh.gp), _f64(mesh.gw)
    _check(ctx, lib().gmg_load_ho_geometry(ctx, _ptr(m2), int(gw.shape[0]), _ptr(gp), _ptr(gw)))


def gmg_set_ho_state(ctx, G=None, alpha=None):
    G = None if G is None else _f64(G)
    alpha = None if alpha is None else _f64(alpha)
    _check(ctx, lib().gmg_set_ho_state(ctx, _ptr(G), _ptr(alpha)))


def gmg_get_ho_state(ctx, G_out=None, alpha_out=None):
    _check(ctx, lib().gmg_get_ho_state(ctx, _ptr(G_out), _ptr(alpha_out)))


def gmg_ho_residual(ctx, R_out=None, G_out=None, alpha_out=None, sigma_out=None):
    _check(ctx, lib().gmg_ho_residual(ctx, _ptr(R_out), _ptr(G_out), _ptr(alpha_out), _ptr(sigma_out)))


def gmg_ho_recon(ctx, poly_out=None, flags_out=None):
    _check(ctx, lib().gmg_ho_recon(ctx, _ptr(poly_out), _ptr(flags_out)))


def gmg_last_error(ctx):
    m = lib().gmg_last_error(ctx)
    return m.decode() if m else ""


def gmg_destroy(ctx):
    _NV.pop(ctx.value if hasattr(ctx, "value") else ctx, None)
    lib().gmg_destroy(ctx)


# ---------------------------------------------------------------------------
# convenience wrapper: torch workspace + stream
# ---------------------------------------------------------------------------
class Solver:
    """One rank's GMG solver on one CUDA device.

    mesh: synth.Mesh-like (vol, ctr, left, right, avec, fctr, ngauss,
    patch_kind, dim).  kw: gmg_options fields (cfl_imp, n_sweeps, ...).
    """

    def __init__(self, mesh, n_levels=3, device=0, color0=None, build_only=False, part=None, nccl_id=None,
                 ho_geometry=False, **kw):
        self.dim = int(mesh.dim)
        self.nv = self.dim + 2
        self.opt = gmg_default_options(dim=self.dim, n_levels=n_levels, device=device, **kw)
        self._nccl_id = None
        if nccl_id is not None:
            self._nccl_id = C.create_string_buffer(bytes(nccl_id), 128)
            self.opt.nccl_id = C.cast(self._nccl_id, C.c_void_p)
        self._torch = None
        if not build_only:
            import torch
            if not torch.cuda.is_available():
                raise RuntimeError("libgmg needs a CUDA device (no CPU fallback)")
            self._torch = torch
            self.device = torch.device("cuda", device)
            self.opt.stream = torch.cuda.current_stream(self.device).cuda_stream
        self.ctx = gmg_create(self.opt)
        gmg_load_mesh(self.ctx, mesh, part)
        if self.opt.fine_operator == 1 or ho_geometry:
            gmg_load_ho_geometry(self.ctx, mesh)
        if color0 is not None:
            gmg_set_coloring(self.ctx, 0, color0)
        self.n_levels, self.build_status = gmg_build_hierarchy(self.ctx, n_levels)
        self.sizes = [gmg_get_level_info(self.ctx, l) for l in range(self.n_levels)]
        self.ws = None
        if not build_only:
            nb = gmg_workspace_bytes(self.ctx)
            self.ws = self._torch.empty(nb, dtype=self._torch.uint8, device=self.device)
            gmg_set_workspace(self.ctx, self.ws.data_ptr(), nb)
            if self.opt.nranks > 1 and self.opt.p2p == 1:
                self._p2p_exchange()

    def _p2p_exchange(self):
        """Fused P2P halo between ranks: share every rank's workspace through
        CUDA IPC (the caching allocator's block handle + this workspace's
        offset in it) and its record / flag layout, then map the peers'."""
        import torch.distributed as dist
        info = self.ws.untyped_storage()._share_cuda_()
        handle, off = bytes(info[1]), int(info[3])
        lay = gmg_p2p_layout(self.ctx, self.n_levels)
        allv = [None] * self.opt.nranks
        dist.all_gather_object(allv, (handle, off, lay.tolist()))
        gmg_p2p_import(self.ctx, [a[0] for a in allv], [a[1] for a in allv], [a[2] for a in allv])

    def n_cells(self, level=0):
        return self.sizes[level][0]

    def n_colors(self, level=0):
        return self.sizes[level][1]

    def maps(self, level=0):
        return gmg_get_maps(self.ctx, level)

    def geometry(self, level=0):
        return gmg_get_level_geometry(self.ctx, level, self.dim)

    def set_state(self, W, W_inf):
        gmg_set_state(self.ctx, W, W_inf)

    def set_level_state(self, level, W):
        gmg_set_level_state(self.ctx, level, W)

    def get_state(self, level=0):
        out = np.zeros((self.nv, self.n_cells(level)))
        gmg_get_state(self.ctx, level, out)
        return out

    def set_alpha(self, alpha):
        gmg_set_alpha(self.ctx, alpha)

    def residual(self, level=0):
        n = self.n_cells(level)
        R, a, s = np.zeros((self.nv, n)), np.zeros(n), np.zeros(n)
        gmg_residual(self.ctx, level, R, a, s)
        return R, a, s

    def set_level_inputs(self, level, Rt=None, alpha=None):
        gmg_set_level_inputs(self.ctx, level, Rt, alpha)

    def smooth(self, level, n_sweeps):
        dW = np.zeros((self.nv, self.n_cells(level)))
        gmg_smooth(self.ctx, level, n_sweeps, dW)
        return dW

    def vcycle(self, n_cycles=1):
        hist = np.zeros((n_cycles + 1, self.nv))
        gmg_vcycle(self.ctx, n_cycles, hist)
        return hist

    def profile_vcycle(self, n_cycles=1):
        return gmg_profile_vcycle(self.ctx, n_cycles)

    def time_smooth(self, level, n_sweeps, reps):
        return gmg_time_smooth(self.ctx, level, n_sweeps, reps)

    def vcycle_launches(self):
        return gmg_vcycle_launches(self.ctx)

    def vcycle_visits(self):
        return gmg_vcycle_visits(self.ctx)

    def level_field(self, level, field):
        out = np.zeros((1 if field == FIELD_ALPHA else self.nv, self.n_cells(level)))
        gmg_get_level_field(self.ctx, level, field, out)
        return out[0] if field == FIELD_ALPHA else out

    # NEXT-1 (fine_operator = 1 or ho_geometry = True)
    def set_ho_state(self, G=None, alpha=None):
        gmg_set_ho_state(self.ctx, G, alpha)

    def get_ho_state(self):
        n = self.n_cells(0)
        G, a = np.zeros((self.nv, self.dim, n)), np.zeros(n)
        gmg_get_ho_state(self.ctx, G, a)
        return G, a

    def ho_residual(self):
        n = self.n_cells(0)
        R, G, a, s = np.zeros((self.nv, n)), np.zeros((self.nv, self.dim, n)), np.zeros(n), np.zeros(n)
        gmg_ho_residual(self.ctx, R, G, a, s)
        return R, G, a, s

    def ho_recon(self):
        n = self.n_cells(0)
        nc = 1 + self.dim + self.dim * (self.dim + 1) // 2
        poly = np.zeros((self.nv * nc, n))
        fl = np.zeros(n, dtype=np.int32)
        gmg_ho_recon(self.ctx, poly, fl)
        return np.ascontiguousarray(poly.T.reshape(n, self.nv, nc)), fl

    def halo(self, level=0, dom=0):
        return gmg_get_halo(self.ctx, level, dom)

    def close(self):
        if self.ctx:
            gmg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
