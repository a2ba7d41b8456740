"""Pins of the NEXT-1 oracle (oracle/cgks3.c, DESIGN.md §12 readings C1-C14)
against things other than itself: a brute-force velocity-space + time
quadrature of the paper's distribution function (Eqs. (dis1), (dis2), (co),
(compatibility2)), closed forms (free stream = Euler flux),
invariants (side swap, rotation, free-stream preservation, discrete
conservation) and exactness of the reconstruction on polynomial fields
(P:312-352)."""
import numpy as np
import pytest
from scipy.special import gamma as Gamma

import oracle
from oracle import cgks3
from synth import configs, state

GAM = 1.4


def _K(dim):
    return (5 - 3 * GAM) / (GAM - 1) if dim == 3 else (4 - 2 * GAM) / (GAM - 1)


def _rand_state(rng, dim, rho=1.0, p=1.0, u=0.5):
    r = rho * (1 + 0.2 * rng.random())
    v = u * (2 * rng.random(dim) - 1)
    pr = p * (1 + 0.2 * rng.random())
    W = np.zeros(dim + 2)
    W[0] = r
    W[1:1 + dim] = r * v
    W[-1] = pr / (GAM - 1) + 0.5 * r * (v @ v)
    return W


# ---------------------------------------------------------------------------
# brute force: the paper's f(x=0, t, u, xi) integrated numerically
# ---------------------------------------------------------------------------
class _Quad:
    """Gauss-Legendre tensor grid over velocity space, u1 split at 0; the
    internal variable enters through s = |xi|^2 with <s^m> =
    Gamma(K/2 + m) / Gamma(K/2) / lambda^m (chi-square moments)."""

    def __init__(self, dim, L=14.0, n1=72, nt=64):
        x, w = np.polynomial.legendre.leggauss(n1)
        pos = 0.5 * L * (x + 1)
        wp = 0.5 * L * w
        u1 = np.concatenate([-pos[::-1], pos])
        w1 = np.concatenate([wp[::-1], wp])
        xt, wt = np.polynomial.legendre.leggauss(nt)
        ut = L * xt
        wtt = L * wt
        axes = [u1] + [ut] * (dim - 1)
        ws = [w1] + [wtt] * (dim - 1)
        grids = np.meshgrid(*axes, indexing="ij")
        self.u = [g.ravel() for g in grids]
        W = ws[0][:, None] * ws[1][None, :]
        if dim == 3:
            W = W[:, :, None] * ws[2][None, None, :]
        self.w = W.ravel()
        self.dim = dim

    def maxwell(self, W):
        d = self.dim
        rho = W[0]
        U = W[1:1 + d] / rho
        p = (GAM - 1) * (W[-1] - 0.5 * rho * U @ U)
        lam = rho / (2 * p)
        r2 = sum((self.u[k] - U[k]) ** 2 for k in range(d))
        g = (lam / np.pi) ** (d / 2) * np.exp(-lam * r2)
        s_mom = [Gamma(_K(d) / 2 + m) / Gamma(_K(d) / 2) / lam ** m for m in range(4)]
        return dict(rho=rho, U=U, lam=lam, g=g, s=s_mom)

    def psi(self):
        """psi_a as (coefficient of s^0, of s^1) on the grid."""
        d = self.dim
        one = np.ones_like(self.u[0])
        zero = np.zeros_like(one)
        out = [(one, zero)] + [(self.u[k], zero) for k in range(d)]
        out.append((0.5 * sum(self.u[k] ** 2 for k in range(d)), 0.5 * one))
        return out

    def mom(self, M, f, rng="full"):
        """(1/rho) int f g over u (and s): f = (c0, c1, c2) coefficients of s^m."""
        mask = 1.0
        if rng == "pos":
            mask = (self.u[0] > 0).astype(float)
        elif rng == "neg":
            mask = (self.u[0] < 0).astype(float)
        tot = 0.0
        for m, c in enumerate(f):
            tot += M["s"][m] * np.sum(self.w * mask * M["g"] * c)
        return tot


def _pmul(a, b):
    """product of s-polynomials (lists of grid arrays)."""
    out = [0.0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] = out[i + j] + x * y
    return out


def _slope_poly(Q, s):
    """s . psi as an s-polynomial."""
    ps = Q.psi()
    return [sum(s[a] * ps[a][0] for a in range(len(s))), sum(s[a] * ps[a][1] for a in range(len(s)))]


def _micro(Q, M, b):
    ps = Q.psi()
    nv = len(ps)
    A = np.array([[Q.mom(M, _pmul(ps[a], ps[c])) for c in range(nv)] for a in range(nv)])
    return np.linalg.solve(A, b)


def _adotu(Q, a):
    tot = [0.0, 0.0]
    for e in range(Q.dim):
        sp = _slope_poly(Q, a[e])
        tot = [tot[0] + sp[0] * Q.u[e], tot[1] + sp[1] * Q.u[e]]
    return tot


def _Acoef(Q, M, a):
    ps = Q.psi()
    au = _adotu(Q, a)
    b = np.array([-Q.mom(M, _pmul(au, ps[q])) for q in range(len(ps))])
    return _micro(Q, M, b)


def brute_gks(dim, Wl, dWl, Wr, dWr, dt, tau, Q=None):
    Q = Q or _Quad(dim)
    ps = Q.psi()
    nv = dim + 2
    Ml, Mr = Q.maxwell(Wl), Q.maxwell(Wr)
    al = [_micro(Q, Ml, dWl[e] / Ml["rho"]) for e in range(dim)]
    ar = [_micro(Q, Mr, dWr[e] / Mr["rho"]) for e in range(dim)]
    Al, Ar = _Acoef(Q, Ml, al), _Acoef(Q, Mr, ar)
    Wc = np.array([Ml["rho"] * Q.mom(Ml, ps[q], "pos") + Mr["rho"] * Q.mom(Mr, ps[q], "neg") for q in range(nv)])
    Mc = Q.maxwell(Wc)
    ac = []
    for e in range(dim):
        sl, sr = _slope_poly(Q, al[e]), _slope_poly(Q, ar[e])
        b = np.array([(Ml["rho"] * Q.mom(Ml, _pmul(sl, ps[q]), "pos") + Mr["rho"] * Q.mom(Mr, _pmul(sr, ps[q]), "neg"))
                      for q in range(nv)]) / Mc["rho"]
        ac.append(_micro(Q, Mc, b))
    Ac = _Acoef(Q, Mc, ac)
    acu, Acp = _adotu(Q, ac), _slope_poly(Q, Ac)
    alu, Alp = _adotu(Q, al), _slope_poly(Q, Al)
    aru, Arp = _adotu(Q, ar), _slope_poly(Q, Ar)

    def fmoments(t, weight):
        """int weight * psi * f(t) as (1/1) absolute moments (Eq.(dis1)+(dis2))."""
        ex = np.exp(-t / tau)
        C1, C2, C3 = 1 - ex, (t + tau) * ex - tau, t - tau + tau * ex
        out = np.zeros(nv)
        for q in range(nv):
            base = _pmul(ps[q], weight)
            eq = [C1 * base[0], C1 * base[1]]
            ta = _pmul(base, acu)
            tA = _pmul(base, Acp)
            val = Mc["rho"] * (Q.mom(Mc, eq) + C2 * Q.mom(Mc, ta) + C3 * Q.mom(Mc, tA))
            for M, au, Ap, rg in ((Ml, alu, Alp, "pos"), (Mr, aru, Arp, "neg")):
                bracket = [1.0 - tau * (au[0] + Ap[0]) - t * au[0], -tau * (au[1] + Ap[1]) - t * au[1]]
                val += M["rho"] * ex * Q.mom(M, _pmul(base, bracket), rg)
            out[q] = val
        return out

    one = [np.ones_like(Q.u[0]), np.zeros_like(Q.u[0])]
    u1 = [Q.u[0], np.zeros_like(Q.u[0])]
    xt, wt = np.polynomial.legendre.leggauss(24)
    ts = 0.5 * dt * (xt + 1)
    F = sum(0.5 * dt * w * fmoments(t, u1) for t, w in zip(ts, wt))
    Wt = fmoments(dt, one)
    return F, Wt


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("seed", [0, 1])
def test_gks_local_matches_bruteforce_quadrature(dim, seed):
    rng = np.random.default_rng(seed)
    Wl, Wr = _rand_state(rng, dim), _rand_state(rng, dim, rho=0.8, p=0.7)
    dWl = 0.3 * rng.standard_normal((dim, dim + 2))
    dWr = 0.3 * rng.standard_normal((dim, dim + 2))
    dt, tau = 0.05, 0.02
    F, Wt = cgks3.gks_local(dim, GAM, Wl, dWl, Wr, dWr, dt, tau)
    Fb, Wb = brute_gks(dim, Wl, dWl, Wr, dWr, dt, tau)
    assert np.max(np.abs(F - Fb)) <= 1e-9 * np.max(np.abs(Fb)), (F, Fb)
    assert np.max(np.abs(Wt - Wb)) <= 1e-9 * np.max(np.abs(Wb)), (Wt, Wb)


@pytest.mark.parametrize("dim", [2, 3])
def test_gks_free_stream_is_euler_flux(dim):
    """equal uniform states, no slopes: f = g, F = dt T(W; n), W(dt) = W."""
    rng = np.random.default_rng(5)
    for _ in range(5):
        W = _rand_state(rng, dim, u=2.0)
        n = rng.standard_normal(dim)
        n /= np.linalg.norm(n)
        z = np.zeros((dim, dim + 2))
        F, Wt = cgks3.gks_flux(dim, GAM, W, z, W, z, n, 0.3, 0.01)
        T = oracle.euler_flux(dim, GAM, W, n)
        assert np.allclose(F, 0.3 * T, rtol=1e-13, atol=1e-13)
        assert np.allclose(Wt, W, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("dim", [2, 3])
def test_gks_side_swap_and_rotation(dim):
    rng = np.random.default_rng(7)
    Wl, Wr = _rand_state(rng, dim), _rand_state(rng, dim, rho=0.7)
    dWl, dWr = 0.2 * rng.standard_normal((dim, dim + 2)), 0.2 * rng.standard_normal((dim, dim + 2))
    n = rng.standard_normal(dim)
    n /= np.linalg.norm(n)
    F, Wt = cgks3.gks_flux(dim, GAM, Wl, dWl, Wr, dWr, n, 0.04, 0.01)
    F2, Wt2 = cgks3.gks_flux(dim, GAM, Wr, dWr, Wl, dWl, -n, 0.04, 0.01)
    assert np.allclose(F, -F2, rtol=1e-12, atol=1e-14)
    assert np.allclose(Wt, Wt2, rtol=1e-12, atol=1e-14)
    # rotation Q: momenta and gradient directions rotate, scalars do not
    Qm, _ = np.linalg.qr(rng.standard_normal((dim, dim)))

    def rotW(W):
        o = W.copy()
        o[1:1 + dim] = Qm @ W[1:1 + dim]
        return o

    def rotG(G):               # G[c][q] = dW_q / dx_c
        H = np.array([rotW(G[c]) for c in range(dim)])
        return Qm @ H
    F3, Wt3 = cgks3.gks_flux(dim, GAM, rotW(Wl), rotG(dWl), rotW(Wr), rotG(dWr), Qm @ n, 0.04, 0.01)
    assert np.allclose(F3, rotW(F), rtol=1e-12, atol=1e-14)
    assert np.allclose(Wt3, rotW(Wt), rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------------------
# reconstruction
# ---------------------------------------------------------------------------
def _meshes():
    return [configs.tri_square(6, 6, seed=3), configs.quad_grid(5, 4),
            configs.box3d(3, 3, 3, 1, seed=2), configs.box3d(3, 2, 2, 0, seed=4)]


def _quad_field(m, rng):
    """q(x) = c + b.x + x^T H x: exact cell averages and averaged gradients."""
    d = m.dim
    c = rng.standard_normal()
    b = rng.standard_normal(d)
    H = rng.standard_normal((d, d))
    H = 0.5 * (H + H.T)
    iu = np.triu_indices(d)
    M2 = np.zeros((m.n_cells, d, d))
    M2[:, iu[0], iu[1]] = m.m2.T
    M2[:, iu[1], iu[0]] = m.m2.T
    x = m.ctr.T
    avg = c + x @ b + np.einsum("ia,ab,ib->i", x, H, x) + np.einsum("ab,iab->i", H, M2)
    grad = (b[None, :] + 2 * x @ H).T      # [d][n]
    return avg, grad, b, H


def _nbrs(m, i):
    f = np.nonzero((m.left == i) | (m.right == i))[0]
    out = []
    for ff in f:
        if m.right[ff] < 0:
            continue
        out.append(m.right[ff] if m.left[ff] == i else m.left[ff])
    return out


@pytest.mark.parametrize("k", range(4))
def test_p2_exact_for_quadratic_fields(k):
    """the constrained least squares reproduces a quadratic exactly
    (its averages are met exactly, its averaged slopes with zero residual)."""
    m = _meshes()[k]
    M = cgks3.Mesh3(m)
    rng = np.random.default_rng(k)
    avg, grad, b, H = _quad_field(m, rng)
    d = m.dim
    checked = 0
    for i in range(m.n_cells):
        nb = _nbrs(m, i)
        a = cgks3.p2(M, i, nb, avg, grad)
        if len(nb) < d + 1:
            assert a is None
            continue
        assert a is not None
        x = m.ctr[:, i]
        lin = b + 2 * H @ x
        quad = [H[p, q] * (1 if p == q else 2) for p in range(d) for q in range(p, d)]
        assert np.allclose(a, np.concatenate([lin, quad]), rtol=1e-9, atol=1e-9), (i, a)
        checked += 1
    assert checked >= 10


@pytest.mark.parametrize("k", range(4))
def test_recon_reproduces_quadratic_when_smooth_weights(k):
    """With gamma_0 = 1 (large stencil only, weights = linear) the final
    polynomial of an interior cell is p2: quadratic data come back exactly."""
    m = _meshes()[k]
    M = cgks3.Mesh3(m)
    rng = np.random.default_rng(10 + k)
    d, n = m.dim, m.n_cells
    nv = d + 2
    W = np.zeros((nv, n))
    G = np.zeros((nv, d, n))
    Hs = []
    for q in range(nv):
        avg, grad, b, H = _quad_field(m, rng)
        W[q] = avg * 0.01 + (5.0 if q in (0, nv - 1) else 0.0)
        G[q] = grad * 0.01
        Hs.append((b * 0.01, H * 0.01))
    Winf = W[:, 0].copy()
    poly, fl, nfall = cgks3.recon(M, W, G, np.ones(n), Winf, cgks3.Opt3(gam0=1.0))
    assert nfall == 0
    for i in range(n):
        if not (fl[i] & 1):
            continue
        x = m.ctr[:, i]
        for q in range(nv):
            b, H = Hs[q]
            lin = b + 2 * H @ x
            quad = [H[p, r] * (1 if p == r else 2) for p in range(d) for r in range(p, d)]
            assert np.allclose(poly[i, q, 1:], np.concatenate([lin, quad]), rtol=1e-8, atol=1e-10)


def test_green_gauss_exact_for_linear_on_uniform_grid():
    """with gamma_0 -> 0 (sub-stencil only) an interior cell of a
    uniform quad grid gets the exact gradient of a linear field."""
    m = configs.quad_grid(6, 6)
    M = cgks3.Mesh3(m)
    n = m.n_cells
    b = np.array([0.3, -0.2])
    W = np.zeros((4, n))
    W[0] = 1.0 + m.ctr.T @ b
    W[3] = 3.0
    Winf = W[:, 0].copy()
    poly, fl, _ = cgks3.recon(M, W, np.zeros((4, 2, n)), np.ones(n), Winf, cgks3.Opt3(gam0=1e-300))
    interior = [i for i in range(n) if len(_nbrs(m, i)) == 4]
    for i in interior:
        assert np.allclose(poly[i, 0, 1:3], b, rtol=1e-12, atol=1e-13)
        assert np.allclose(poly[i, 0, 3:], 0.0)


@pytest.mark.parametrize("gam0", [0.95, 0.5])
def test_weno_combination_consistent_for_linear_data(gam0):
    """C5: p = w0 (p2 - g1 p1) / g0 + w1 p1 reproduces a field that
    BOTH candidates represent exactly, whatever the nonlinear weights: linear
    averages with consistent slopes on a uniform quad grid (p2 exact for
    quadratics, Green-Gauss exact for linear data at interior cells) come back
    exactly at every interior p2 cell for any linear weight gamma_0."""
    m = configs.quad_grid(6, 6)
    M = cgks3.Mesh3(m)
    n = m.n_cells
    b = np.array([0.3, -0.2])
    W = np.zeros((4, n))
    W[0] = 1.0 + m.ctr.T @ b
    W[3] = 3.0
    G = np.zeros((4, 2, n))
    G[0] = b[:, None]
    Winf = W[:, 0].copy()
    poly, fl, _ = cgks3.recon(M, W, G, np.ones(n), Winf, cgks3.Opt3(gam0=gam0))
    interior = [i for i in range(n) if len(_nbrs(m, i)) == 4 and (fl[i] & 1)]
    assert interior
    for i in interior:
        assert np.allclose(poly[i, 0, 1:3], b, rtol=1e-12, atol=1e-13)
        assert np.allclose(poly[i, 0, 3:], 0.0, atol=1e-13)


def test_weno_weights_favour_the_smooth_sub_stencil():
    """C5: averages of a linear field (p1 smooth) with wildly wrong neighbour
    slopes (p2 rough): the large-stencil weight collapses, the final
    polynomial is close to p1 (quadratic part far below p2's)."""
    m = configs.quad_grid(8, 8)
    M = cgks3.Mesh3(m)
    n = m.n_cells
    b = np.array([0.3, -0.2])
    W = np.zeros((4, n))
    W[0] = 10.0 + m.ctr.T @ b
    W[3] = 300.0
    rng = np.random.default_rng(3)
    G = np.zeros((4, 2, n))
    G[0] = 50.0 * rng.standard_normal((2, n))
    Winf = W[:, 0].copy()
    poly_s, _, _ = cgks3.recon(M, W, G, np.ones(n), Winf, cgks3.Opt3())
    poly_l, _, _ = cgks3.recon(M, W, G, np.ones(n), Winf, cgks3.Opt3(gam0=1.0))
    interior = [i for i in range(n) if len(_nbrs(m, i)) == 4]
    ratio = [np.max(np.abs(poly_s[i, 0, 3:])) / np.max(np.abs(poly_l[i, 0, 3:])) for i in interior]
    assert np.mean(np.array(ratio) < 0.1) >= 0.7, ratio


# ---------------------------------------------------------------------------
# whole operator
# ---------------------------------------------------------------------------
def _farfield_meshes():
    F = configs.FARFIELD
    return [configs.tri_square(6, 6, seed=1), configs.quad_grid(5, 5),
            configs.box3d(4, 4, 3, 1, seed=1, patch_kinds=(F,)), configs.box3d(2, 3, 3, 0, seed=3, patch_kinds=(F,))]


@pytest.mark.parametrize("k", range(4))
def test_residual_free_stream_preserved(k):
    m = _farfield_meshes()[k]
    M = cgks3.Mesh3(m)
    d = m.dim
    vel = (0.6, 0.2, -0.1)[:d]
    W = state.uniform(m, 1.0, vel, 0.7)
    Winf = state.winf(1.0, vel, 0.7)
    R, Gn, a, S, fl, nf = cgks3.residual(M, W, np.zeros((d + 2, d, m.n_cells)), np.ones(m.n_cells), Winf)
    assert nf == 0
    assert np.max(np.abs(R)) < 1e-13 * np.max(S)
    assert np.max(np.abs(Gn)) < 1e-12
    assert np.allclose(a, 1.0)


@pytest.mark.parametrize("k", range(4))
def test_residual_discrete_conservation(k):
    """interior fluxes telescope: with a perturbation away from the farfield
    boundary, sum_i R_i = sum of free-stream boundary fluxes = 0 (closure)."""
    m = _farfield_meshes()[k]
    M = cgks3.Mesh3(m)
    d, n = m.dim, m.n_cells
    vel = (0.6, 0.2, -0.1)[:d]
    W = state.uniform(m, 1.0, vel, 0.7)
    Winf = state.winf(1.0, vel, 0.7)
    rng = np.random.default_rng(k)
    bnd = set(m.left[m.right < 0].tolist())
    inner = np.array([i for i in range(n) if i not in bnd and all(j not in bnd for j in _nbrs(m, i))])
    if inner.size == 0:
        pytest.skip("no cell away from the boundary")
    W[:, inner] *= 1 + 0.05 * rng.random((1, inner.size))
    G = np.zeros((d + 2, d, n))
    R, Gn, a, S, fl, nf = cgks3.residual(M, W, G, np.ones(n), Winf)
    assert np.max(np.abs(R.sum(axis=1))) < 1e-12 * np.max(np.abs(R)), R.sum(axis=1)


def test_p2min_reading_c3b(orc):
    """Reading C3b: with p2min = d + 2 a cell uses p2 only with at
    least d + 2 interior neighbours -- on a triangulated square no cell does (3
    faces each), on a quad grid the interior cells still do; where p2 is off
    the polynomial is the p1 (Green-Gauss x DF) one, identical to the default
    run's p1 cells."""
    from oracle import cgks3
    for m, expect_p2 in ((configs.tri_square(6, 6, seed=2), False), (configs.quad_grid(6, 6), True)):
        W = state.perturbed(m, 1.0, [0.5, 0.1], 0.7, eps=0.05, seed=1)
        Winf = state.winf(1.0, [0.5, 0.1], 0.7)
        G0 = np.zeros((4, 2, m.n_cells))
        a0 = np.ones(m.n_cells)
        M = cgks3.Mesh3(m)
        p_def, f_def, _ = cgks3.recon(M, W, G0, a0, Winf)
        p_b, f_b, _ = cgks3.recon(M, W, G0, a0, Winf, cgks3.Opt3(p2min=4))
        assert bool((f_b & 1).any()) == expect_p2
        assert bool((f_def & 1).any())
        same = (f_b & 1) == (f_def & 1)
        assert np.array_equal(p_b[same], p_def[same])
        gone = (f_def & 1) & ~(f_b & 1)
        assert np.all(p_b[gone.astype(bool)][:, :, 3:] == 0.0)     # no quadratic terms where p2 is off
