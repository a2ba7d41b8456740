"""Element-wise comparison helpers of the GPU parity tests (no method arithmetic).

The bar (BASELINE.json north_star): FP64 fields within 1e-10,
measured per component as max_i |gpu_i - ref_i| / max_i |ref_i| (so a wrong
element is not hidden by a global norm dominated by the free stream).
"""
import numpy as np

TOL = 1e-10


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def elem(a, b, scale=None):
    """max over components q of max_i |a[q,i] - b[q,i]| / max_i |scale[q,i]|
    (scale defaults to b)."""
    a = np.atleast_2d(np.asarray(a, dtype=np.float64))
    b = np.atleast_2d(np.asarray(b, dtype=np.float64))
    s = np.abs(np.atleast_2d(b if scale is None else scale)).max(axis=1)
    s[s == 0] = 1.0
    return float(np.max(np.abs(a - b).max(axis=1) / s))


def check_levels(G, s, entries, n_levels, tol=TOL, first=None):
    """Coarse levels of the last V-cycle (oracle trace entries) against the
    library's level fields, element by element: restricted state W0
    (P:643-647), restricted residual Res* (P:648-652), DF alpha (min over the
    children, A15), forcing F = Res* - R(W0) (absolute error scale
    of its operands, Res*), the smoothing increment dW and the coarse state
    W0 + dW.  Returns the worst ratio per field.

    first: the FIRST cycle's trace entries of a long run.  Then every field is
    measured against max(|ref|, |first-cycle ref|) per component -- the
    normalised-absolute reading SURVEY §8(c) fixes for histories (|r_gpu(k) -
    r_orc(k)| <= 1e-10 r(0)): once a run has converged, Res*, F and dW are
    rounding-level quantities and their relative error says nothing."""
    worst = {}
    f0 = {t["level"]: t for t in first} if first else {}
    for t in entries:
        l = t["level"]
        got = {
            "W0": (s.level_field(l, G.FIELD_W0), t["W0"], None),
            "Rs": (s.level_field(l, G.FIELD_RS), t["Rs"], None),
            "alpha": (s.level_field(l, G.FIELD_ALPHA), t["alpha"], np.ones_like(t["alpha"])),
            "dW": (s.level_field(l, G.FIELD_DW), t["dW"], None),
            "W": (s.get_state(l), t["W0"] + t["dW"], None),
        }
        if l < n_levels - 1:
            got["F"] = (s.level_field(l, G.FIELD_F), t["F"], t["Rs"])
        for k, (a, b, sc) in got.items():
            if l in f0 and k != "alpha":
                t0 = f0[l]
                b0 = {"W0": t0["W0"], "Rs": t0["Rs"], "dW": t0["dW"], "W": t0["W0"] + t0["dW"], "F": t0["Rs"]}[k]
                base = np.abs(np.atleast_2d(b if sc is None else sc))
                sc = np.maximum(base.max(axis=1, keepdims=True), np.abs(np.atleast_2d(b0)).max(axis=1, keepdims=True))
            e = elem(a, b, sc)
            worst[f"L{l}.{k}"] = e
            assert e <= tol, f"level {l} {k}: {e:.3e}"
    return worst
