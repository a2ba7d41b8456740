"""Round-2 pins of the oracle steps the round-1 pins left open (CPU only).

Each test names the passage it pins and the plausible mistake it catches;
tests/test_oracle_mutants.py applies those mistakes to a copy of the oracle
and checks that the named test turns red.  Nothing here calls the CUDA path.

* FAS forcing (readings A8/A11): forcing identity and
  steady-state consistency -- a flipped or dropped F fails the latter.
* DF cell product alpha_i = prod_f alpha_f^{M_f} with mixed M_f (P:356-358,
  A16) -- a dropped exponent or a min instead of a product fails.
* DF tangential-Mach term |Ma_t^l - Ma_t^r|^2 (A17) -- an
  unsquared or magnitude-only term fails.
* Sigma_i over ALL faces, boundary faces included (A6), hand-computed
  on single boundary cells -- an interior-only sum fails.
* Linear-flux reduction of the MC-SGS smoother to symmetric Gauss-Seidel with
  scipy.sparse triangular solves (SURVEY §8(c) sweep pin (vi)).
* Eq.(smo) explicit step with reading A9 (W -= CFL_exp/Sigma R), worked.
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular

from synth import configs, state
from synth.mesh import EXTRAP, FARFIELD, SLIP, NOSLIP

G = 1.4


def _W(rho, u, p, gamma=G):
    return state.prim_to_cons(np.array(rho), np.asarray(u, dtype=float), np.array(p), gamma=gamma)


# ------------------------------------------------------------ FAS forcing
def _steady_naca(orc):
    """A converged non-uniform fine state: flow around a small NACA0012
    O-grid (no-slip ghost wall, farfield M 0.5), 400 V-cycles drive the fine
    residual to machine level (≈1e-14 from 2e-2)."""
    m = configs.naca_ogrid(ni=32, n_quad=6, n_tri=2, r_out=5.0)
    H = orc.build_hierarchy(m, 3, 0.5)
    fs = configs.FREESTREAM[2]
    W = state.uniform(m, *fs)
    Winf = state.winf(*fs)
    Ws, hist = orc.vcycle(H, W, Winf, orc.Options(), 400)
    return m, H, Ws, Winf, hist


@pytest.fixture(scope="module")
def steady(orc):
    return _steady_naca(orc)


def test_forcing_identity(orc, steady):
    """S:570 / P:664: immediately after the forcing is formed,
    R_2h(W0) + F = Res*_2h (to rounding of one subtraction), on both coarse
    levels, at a generic (non-converged) state."""
    m, H, _, Winf, _ = steady
    W = state.perturbed(m, 1.0, [0.5, 0.0], 1 / 1.4, eps=0.05, seed=3)
    trace = []
    orc.vcycle(H, W, Winf, orc.Options(), 1, trace=trace)
    assert [t["level"] for t in trace] == [1, 2]
    for t in trace:
        lv = H[t["level"]]["level"]
        Rc, _, _, _ = orc.residual(lv, t["W0"], Winf)
        scale = np.abs(t["Rs"]).max()
        assert np.abs(Rc + t["F"] - t["Rs"]).max() <= 4e-16 * max(scale, np.abs(Rc).max())
        # F is not trivially zero: the coarse operator does not reproduce Res*
        assert np.abs(t["F"]).max() > 1e-3 * scale


def test_fas_steady_state_consistency(orc, steady):
    """S:573 (readings A8, A11): at a converged fine solution
    (residual tol = ||R_0(W*)||_2 ≈ 1e-14) one V-cycle changes the fine state
    by <= 10 tol.  With F's sign flipped, F dropped on level 2, or Res*
    replaced by R_2h(W0) as the coarse right-hand side, the coarse levels see
    R_2h(W0) != 0 and the change is O(1e-2) (tests/test_oracle_mutants.py)."""
    m, H, Ws, Winf, hist = steady
    R, _, _, _ = orc.residual(H[0]["level"], Ws, Winf)
    tol = np.linalg.norm(R)
    assert tol < 1e-12 and hist[0, 0] > 1e-3           # converged from a real transient
    assert np.abs(Ws - state.uniform(m, *configs.FREESTREAM[2])).max() > 0.1   # non-trivial
    # the coarse operator at the restricted state is far from zero: F matters
    trace = []
    W1, _ = orc.vcycle(H, Ws, Winf, orc.Options(), 1, trace=trace)
    assert all(np.abs(t["F"]).max() > 1e-4 for t in trace)
    assert np.abs(W1 - Ws).max() <= 10 * tol


# ------------------------------------------------------------ DF cell product
def test_df_cell_product_mixed_gauss_points(orc):
    """P:356-358 alpha_i = prod_p prod_k alpha_{p,k} (A16: first-order states,
    one alpha_f per face, M_f Gauss points: 3 per triangle, 4 per quad).
    One prism cell at p = 2 among cells at p = 1, all at rest: every face of
    that cell has D = |1|/2 + |1|/1 = 3/2 -> alpha_f = 1/(1 + 9/4) =
    4/13; boundary faces are extrapolation ghosts (alpha_f = 1).  So
    alpha_k = (4/13)^(sum of M_f over its interior faces) and each neighbour
    j gets (4/13)^(M_f of the shared face): exponents 3 and 4 both occur."""
    m = configs.box3d(2, 2, 2, 2, seed=1, patch_kinds=(EXTRAP,))
    lv = orc.Level.from_mesh(m)
    n = m.n_cells
    p = np.ones(n)
    # a prism with both triangle and quad interior faces
    k = None
    for c in range(n):
        fs = [f for f in range(m.n_faces) if m.right[f] >= 0 and c in (m.left[f], m.right[f])]
        if {3, 4} <= {int(m.ngauss[f]) for f in fs}:
            k, faces_k = c, fs
            break
    assert k is not None
    p[k] = 2.0
    W = np.stack([_W(1.0, [0.0, 0.0, 0.0], pi) for pi in p], axis=1)
    _, alpha, _, _ = orc.residual(lv, W, W[:, 0])
    base = 4.0 / 13.0
    expo = sum(int(m.ngauss[f]) for f in faces_k)
    assert abs(alpha[k] - base ** expo) <= 1e-14 * base ** expo
    seen_M = set()
    for f in faces_k:
        j = m.right[f] if m.left[f] == k else m.left[f]
        M = int(m.ngauss[f])
        seen_M.add(M)
        assert abs(alpha[j] - base ** M) <= 1e-14 * base ** M, (j, M)
    assert seen_M == {3, 4}
    others = np.setdiff1d(np.arange(n), [k] + [m.right[f] if m.left[f] == k else m.left[f] for f in faces_k])
    assert np.all(alpha[others] == 1.0)


# ------------------------------------------------------------ DF tangential Mach
def test_df_tangential_mach_term(orc):
    """P:360-365, reading A17: D includes |Ma_t^l - Ma_t^r|^2, the squared
    norm of the vector difference of the tangential Mach numbers
    (Ma_t = (u - (u.n) n)/a).  Equal p and rho:
      2D  dMa_t = 2                 -> D = 4      -> alpha = 1/17
      3D  Ma_t = +e_y / -e_y        -> |dMa_t|^2 = 4 -> 1/17 (a magnitude-only
          reading (|Ma_t^l| - |Ma_t^r|)^2 would give 0 -> alpha = 1)
      3D  oblique n, dMa_n = 1, |dMa_t| = 2 -> D = 5 -> 1/26."""
    a = math.sqrt(G)                       # rho = p... a = sqrt(gamma p / rho) with p = rho = 1
    al = orc.df_face(2, G, _W(1.0, [0.0, 2 * a], 1.0), _W(1.0, [0.0, 0.0], 1.0), [1.0, 0.0])
    assert abs(al - 1.0 / 17.0) <= 1e-15
    al = orc.df_face(3, G, _W(1.0, [0.0, a, 0.0], 1.0), _W(1.0, [0.0, -a, 0.0], 1.0), [1.0, 0.0, 0.0])
    assert abs(al - 1.0 / 17.0) <= 1e-15
    n = np.array([0.6, 0.8, 0.0])
    t = np.array([-0.8, 0.6, 0.0])
    uL = a * n + 2 * a * t
    al = orc.df_face(3, G, _W(1.0, uL, 1.0), _W(1.0, [0.0, 0.0, 0.0], 1.0), n)
    assert abs(al - 1.0 / 26.0) <= 1e-14
    # a tangential component along the third axis too (both tangential directions enter)
    uL = a * np.array([0.0, 1.0, 1.0])
    al = orc.df_face(3, G, _W(1.0, uL, 1.0), _W(1.0, [0.0, 0.0, 0.0], 1.0), [1.0, 0.0, 0.0])
    assert abs(al - 1.0 / 5.0) <= 1e-15


# ------------------------------------------------------------ Sigma over all faces
def test_sigma_single_boundary_cell_hand_computed(orc):
    """Reading A6 (closure P:454 needs every face): Sigma_i = sum over ALL
    faces of S_f r_f, r_f = |u.n| + a of the average of the cell and its
    ghost (A5).  Unit square, 4 unit faces with normals +-x, +-y:
    * far field with W_inf = W: r = |u.n| + a -> Sigma = 2|u_x| + 2|u_y| + 4a;
    * slip walls: the average has zero normal momentum and a larger pressure
      p_x = (g-1)(E - m_y^2/(2 rho)) on the x faces (p_y likewise)
      -> Sigma = 2 a(p_x) + 2 a(p_y)."""
    rho, u, p = 1.3, np.array([0.4, -0.7]), 0.9
    W = _W(rho, u, p)
    a = math.sqrt(G * p / rho)
    m = configs.quad_grid(1, 1)
    _, _, S, _ = orc.residual(orc.Level.from_mesh(m), W[:, None], W)
    assert abs(S[0] - (2 * abs(u[0]) + 2 * abs(u[1]) + 4 * a)) <= 1e-14 * S[0]
    m = configs.quad_grid(1, 1, patch_kinds=(SLIP,))
    _, _, S, _ = orc.residual(orc.Level.from_mesh(m), W[:, None], W)
    E = W[3]
    px = (G - 1) * (E - 0.5 * (rho * u[1]) ** 2 / rho)
    py = (G - 1) * (E - 0.5 * (rho * u[0]) ** 2 / rho)
    expect = 2 * math.sqrt(G * px / rho) + 2 * math.sqrt(G * py / rho)
    assert abs(S[0] - expect) <= 1e-14 * expect
    # no-slip ghost (-m): the average is at rest with p = (g-1)E -> r = a(E)
    m = configs.quad_grid(1, 1, patch_kinds=(NOSLIP,))
    _, _, S, _ = orc.residual(orc.Level.from_mesh(m), W[:, None], W)
    expect = 4 * math.sqrt(G * (G - 1) * E / rho)
    assert abs(S[0] - expect) <= 1e-14 * expect


def test_sigma_mixed_cell_two_squares(orc):
    """The unit square split into two 1/2 x 1 cells: each has 3 boundary
    faces and 1 interior face (two x-faces of length 1, two y-faces of length
    1/2); the same state everywhere and W_inf = W gives
    Sigma = 2(|u_x| + a) + (|u_y| + a) for both cells (an interior-only sum
    would give |u_x| + a)."""
    rho, u, p = 0.8, np.array([-0.3, 0.5]), 1.1
    W = _W(rho, u, p)
    a = math.sqrt(G * p / rho)
    m = configs.two_cells()
    _, _, S, _ = orc.residual(orc.Level.from_mesh(m), np.repeat(W[:, None], 2, axis=1), W)
    expect = 2 * (abs(u[0]) + a) + (abs(u[1]) + a)
    assert np.all(np.abs(S - expect) <= 1e-14 * expect)


# ------------------------------------------------------------ linear-flux reduction
@pytest.mark.parametrize("mk", ["tri", "box"])
def test_linear_flux_sweep_is_symmetric_gauss_seidel(orc, mk):
    """SURVEY §8(c) sweep pin (vi).  With gamma = 1 the pressure vanishes
    identically, so for a state with rho, m fixed (dW has zero mass and
    momentum parts) and E = 0 the Euler flux difference is exactly linear in
    the energy increment: T(W_j+dW_j; n)_E - T(W_j; n)_E = (u_j.n) dE_j.  The
    MC-SGS step (Eq.(gpu-forward-relaxation)/(gpu-backward-relaxation)
    P:536-551, Algorithm 2, reading A7) then IS symmetric
    Gauss-Seidel on A x = -b with
        A_ii = D_i,  A_ij = 1/2 alpha_i S_f ((u_j . n_ij) - r_f),  b = Rt_E,
    in color-permuted order: forward (D+L) x' = -b - U x, backward
    (D+U) x'' = -b - L x'.  The reference solves with scipy.sparse
    triangular solves on a matrix assembled here from the mesh geometry."""
    m = configs.tri_square(6, 5, seed=7) if mk == "tri" else configs.box3d(2, 2, 2, 1, seed=3)
    d, n = m.dim, m.n_cells
    rng = np.random.default_rng(11)
    rho = rng.uniform(0.5, 2.0, n)
    vel = rng.normal(size=(d, n))
    W = np.zeros((d + 2, n))
    W[0] = rho
    W[1:d + 1] = rho * vel
    Rt = np.zeros((d + 2, n))
    b = rng.normal(size=n)
    Rt[d + 1] = b
    alpha = rng.uniform(0.05, 1.0, n)
    Dg = rng.uniform(4.0, 8.0, n)
    rf = rng.uniform(0.5, 1.5, m.n_faces)
    lv = orc.Level.from_mesh(m)
    col, nc = orc.color(lv)
    n_sweeps = 3
    dW = orc.smooth(lv, W, Rt, alpha, Dg, rf, col, nc, n_sweeps, gamma=1.0)
    assert np.all(dW[:d + 1] == 0.0)
    # assemble A in color-permuted order
    order = np.lexsort((np.arange(n), col))
    pos = np.empty(n, dtype=np.int64)
    pos[order] = np.arange(n)
    rows, cols, vals = [], [], []
    for f in range(m.n_faces):
        l, r = m.left[f], m.right[f]
        if r < 0:
            continue
        A = m.avec[:, f]
        S = np.linalg.norm(A)
        nn = A / S
        for i, j, sg in ((l, r, 1.0), (r, l, -1.0)):
            rows.append(pos[i])
            cols.append(pos[j])
            vals.append(0.5 * alpha[i] * S * (vel[:, j] @ (sg * nn) - rf[f]))
    Off = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    Lo, Up = sp.tril(Off, -1).tocsr(), sp.triu(Off, 1).tocsr()
    Dm = sp.diags(Dg[order])
    assert abs(Off - Lo - Up).max() == 0.0          # no same-color coupling on the diagonal
    rhs = -b[order]
    x = np.zeros(n)
    for _ in range(n_sweeps):
        x = spsolve_triangular((Dm + Lo).tocsr(), rhs - Up @ x, lower=True)
        x = spsolve_triangular((Dm + Up).tocsr(), rhs - Lo @ x, lower=False)
    ref = np.empty(n)
    ref[order] = x
    assert np.abs(dW[d + 1] - ref).max() <= 1e-13 * np.abs(ref).max()


# ------------------------------------------------------------ Eq.(smo), reading A9
def test_explicit_step_worked_example(orc):
    """Eq.(smo) P:638-641 with reading A9: W^{n+1} = W^n - (Dt/V) R with the
    local time step Dt = CFL_exp V / Sigma (A3): W = 1, Sigma = 4, R = 2,
    CFL_exp = 0.5 -> 1 - 0.5/4*2 = 0.75 (P:640 printed V/Dt would give -15)."""
    W = np.full((4, 1), 1.0)
    R = np.full((4, 1), 2.0)
    Wn = orc.explicit_update(W, np.array([4.0]), R, 0.5)
    assert np.all(Wn == 0.75)
