"""GPU parity of the NEXT-1 third-order compact GKS fine operator (ho.cu,
fine_operator = 1) against the oracle (oracle/cgks3.c), through the C ABI:
the reconstruction (polynomials, p2 flags bit-exact), the Gauss-point positivity fallback, one
evaluation (R, evolved slopes, DF, Sigma) and whole V-cycles (state,
slopes, DF, residual history).  Tolerance: the north-star 1e-10 relative L2
for FP64 states and histories."""
import numpy as np
import pytest

import oracle
from oracle import cgks3
from synth import configs, state

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def _cases():
    F, S, N, E = configs.FARFIELD, configs.SLIP, configs.NOSLIP, configs.EXTRAP
    return {
        "tri2d": (configs.tri_square(12, 12, seed=3), (1.0, (0.5, 0.2), 0.8)),
        "quad2d": (configs.quad_grid(10, 8, patch_kinds=(F, S, E, N)), (1.0, (0.4, -0.1), 0.7)),
        "box3d_prism": (configs.box3d(6, 5, 4, 2, seed=1), (1.0, (0.6, 0.2, -0.1), 0.7)),
        "box3d_tet": (configs.box3d(5, 5, 5, 0, seed=2, patch_kinds=(F, S, E, F)), (1.0, (0.3, -0.4, 0.2), 0.9)),
    }


def _state(m, fs, seed, eps=0.08):
    W = state.perturbed(m, *fs, eps=eps, seed=seed)
    rng = np.random.default_rng(seed + 100)
    d, n = m.dim, m.n_cells
    G = 0.3 * rng.standard_normal((d + 2, d, n))
    alpha = 0.5 + 0.5 * rng.random(n)
    return W, state.winf(*fs), G, alpha


def _solver(m, **kw):
    from paper_2509_06347_b200 import Solver
    return Solver(m, fine_operator=1, **kw)


@pytest.mark.parametrize("name", list(_cases()))
def test_recon_matches_oracle(name):
    m, fs = _cases()[name]
    W, Winf, G, alpha = _state(m, fs, 1)
    s = _solver(m, n_levels=1)
    s.set_state(W, Winf)
    s.set_ho_state(G, alpha)
    poly, fl = s.ho_recon()
    s.close()
    po, flo, nfall = cgks3.recon(cgks3.Mesh3(m), W, G, alpha, Winf)
    assert np.array_equal(fl, flo)
    assert (flo & 1).sum() > 0
    assert _rel(poly, po) <= TOL, _rel(poly, po)


@pytest.mark.parametrize("name", list(_cases()))
def test_one_evaluation_matches_oracle(name):
    m, fs = _cases()[name]
    W, Winf, G, alpha = _state(m, fs, 2)
    s = _solver(m, n_levels=1)
    s.set_state(W, Winf)
    s.set_ho_state(G, alpha)
    R, Gn, a, S = s.ho_residual()
    G2, a2 = s.get_ho_state()
    s.close()
    Ro, Gno, ao, So, _, _ = cgks3.residual(cgks3.Mesh3(m), W, G, alpha, Winf)
    assert _rel(S, So) <= 1e-13
    assert _rel(R, Ro) <= TOL, _rel(R, Ro)
    assert _rel(Gn, Gno) <= TOL, _rel(Gn, Gno)
    assert _rel(a, ao) <= TOL, _rel(a, ao)
    assert np.array_equal(G2, G) and np.array_equal(a2, alpha)      # no state change


@pytest.mark.parametrize("name", ["quad2d", "box3d_prism"])
def test_positivity_fallback_matches_oracle(name):
    """C6b: rough slopes drive some Gauss-point states inadmissible; both sides
    fall back at exactly those points (same fp64 decision)."""
    m, fs = _cases()[name]
    W, Winf, G, alpha = _state(m, (fs[0], fs[1], 0.02), 5, eps=0.3)    # low pressure, rough slopes
    G = 40.0 * G
    Ro, Gno, ao, So, _, nfall = cgks3.residual(cgks3.Mesh3(m), W, G, alpha, Winf)
    assert nfall > 0
    s = _solver(m, n_levels=1)
    s.set_state(W, Winf)
    s.set_ho_state(G, alpha)
    R, Gn, a, S = s.ho_residual()
    s.close()
    assert _rel(R, Ro) <= TOL, _rel(R, Ro)
    assert _rel(Gn, Gno) <= TOL
    assert _rel(a, ao) <= TOL


@pytest.mark.parametrize("name", list(_cases()))
def test_vcycles_match_oracle(name):
    m, fs = _cases()[name]
    W, Winf, _, _ = _state(m, fs, 3)
    nc = 4
    s = _solver(m, n_levels=3)
    s.set_state(W, Winf)
    hist = s.vcycle(nc)
    Wg = s.get_state(0)
    Gg, ag = s.get_ho_state()
    s.close()
    H = oracle.build_hierarchy(m, 3, 0.5)
    hs = {}
    Wo, ho = oracle.vcycle(H, W, Winf, oracle.Options(fine_operator=1), nc, mesh=m, ho_state=hs)
    assert _rel(Wg, Wo) <= TOL, _rel(Wg, Wo)
    assert _rel(Gg, hs["G"]) <= TOL, _rel(Gg, hs["G"])
    assert _rel(ag, hs["alpha"]) <= TOL
    herr = np.max(np.abs(hist - ho) / ho[0][None, :])
    assert herr <= TOL, herr


def test_vcycles_continue_from_carried_state():
    """slopes and DF persist across gmg_vcycle calls exactly as in one call."""
    m, fs = _cases()["box3d_prism"]
    W, Winf, _, _ = _state(m, fs, 4)
    s = _solver(m, n_levels=3)
    s.set_state(W, Winf)
    s.vcycle(2)
    h2 = s.vcycle(2)
    W4 = s.get_state(0)
    s.set_state(W, Winf)
    s.set_ho_state()
    s.vcycle(4)
    assert np.array_equal(s.get_state(0), W4)
    s.close()
    assert np.all(np.isfinite(h2))


def test_free_stream_preserved_on_device():
    F = configs.FARFIELD
    m = configs.box3d(6, 5, 4, 2, seed=5, patch_kinds=(F,))
    fs = (1.0, (0.6, 0.2, -0.1), 0.7)
    s = _solver(m, n_levels=3)
    s.set_state(state.uniform(m, *fs), state.winf(*fs))
    hist = s.vcycle(3)
    W = s.get_state(0)
    G, a = s.get_ho_state()
    s.close()
    assert np.max(np.abs(W - state.uniform(m, *fs))) < 1e-13
    assert np.max(np.abs(G)) < 1e-12 and np.allclose(a, 1.0)
    assert np.max(hist) < 1e-12


@pytest.mark.slow
def test_config2_sized_vcycle_matches_oracle():
    """a larger 2D case in the launch configuration of a real run (tens of
    thousands of Gauss points, many resident waves)."""
    m = configs.naca_ogrid(ni=96, n_quad=24, n_tri=8)
    fs = (1.0, (0.5, 0.0), 1.0 / 1.4)
    W = state.uniform(m, *fs)
    Winf = state.winf(*fs)
    s = _solver(m, n_levels=3)
    s.set_state(W, Winf)
    hist = s.vcycle(2)
    Wg = s.get_state(0)
    s.close()
    H = oracle.build_hierarchy(m, 3, 0.5)
    Wo, ho = oracle.vcycle(H, W, Winf, oracle.Options(fine_operator=1), 2, mesh=m, ho_state={})
    assert _rel(Wg, Wo) <= TOL
    assert np.max(np.abs(hist - ho) / ho[0][None, :]) <= TOL


@pytest.fixture(scope="module")
def config4():
    return configs.config(4)


@pytest.mark.slow
def test_config4_full_size_p2_sampled_against_oracle(config4):
    """bench-size launch (1 M cells): with gamma_0 = 1 the device polynomial is
    p2 (C5), which the oracle computes cell by cell (orc3_p2 needs only the
    cell's stencil) -- compared on 2 000 sampled cells."""
    m = config4
    fs = configs.FREESTREAM[4]
    W = state.bow_shock(m, *fs)
    rng = np.random.default_rng(11)
    d, n = m.dim, m.n_cells
    G = 0.05 * rng.standard_normal((d + 2, d, n))
    s = _solver(m, n_levels=3, ho_gam0=1.0, setup_device=1)
    s.set_state(W, state.winf(*fs))
    s.set_ho_state(G, np.ones(n))
    poly, fl = s.ho_recon()
    s.close()
    M = cgks3.Mesh3(m)
    cells = rng.choice(n, 2000, replace=False)
    inn = np.nonzero(m.right >= 0)[0]
    owner = np.concatenate([m.left, m.right[inn]])
    face = np.concatenate([np.arange(m.n_faces), inn])
    order = np.lexsort((face, owner))
    owner, face = owner[order], face[order]
    start = np.searchsorted(owner, np.arange(n + 1))
    checked = 0
    for i in cells:
        f = face[start[i]:start[i + 1]]                      # ascending face id (the oracle's order)
        nb = [int(m.right[x] if m.left[x] == i else m.left[x]) for x in f if m.right[x] >= 0]
        for q in range(d + 2):
            a = cgks3.p2(M, int(i), nb, W[q], G[q])
            if a is None:
                assert not (fl[i] & 1)
                continue
            assert fl[i] & 1
            scale = np.abs(a).max() + 1e-300
            assert np.max(np.abs(poly[i, q, 1:] - a)) <= 1e-10 * max(scale, 1.0), (i, q)
            c0 = W[q, i] - float(np.dot(a[d:], m.m2[:, i]))
            assert abs(poly[i, q, 0] - c0) <= 1e-12 * max(abs(c0), 1.0)
            checked += 1
    assert checked > 5000


@pytest.mark.slow
def test_config4_full_size_free_stream(config4):
    """bench-size launch: with every patch far field, a uniform free stream is
    preserved exactly by the third-order V-cycle (R = 0, slopes 0, DF 1)."""
    import copy
    m = copy.copy(config4)
    m.patch_kind = np.zeros_like(config4.patch_kind)
    fs = configs.FREESTREAM[4]
    W = state.uniform(m, *fs)
    s = _solver(m, n_levels=3, setup_device=1)
    s.set_state(W, state.winf(*fs))
    hist = s.vcycle(2)
    Wg = s.get_state(0)
    G, a = s.get_ho_state()
    s.close()
    assert np.max(np.abs(Wg - W)) <= 1e-12 * np.max(np.abs(W))
    assert np.max(np.abs(G)) <= 1e-8 and np.allclose(a, 1.0)
    assert np.max(hist) <= 1e-9 * max(1.0, float(np.abs(W).max()))


@pytest.mark.parametrize("name", ["tri2d", "box3d_prism", "box3d_tet"])
@pytest.mark.parametrize("P", [2, 3])
def test_partitioned_vcycles_match_oracle(name, P, monkeypatch):
    """the third-order fine operator on P sub-domains (gmg_options.local_domains,
    the partitioned path's layouts, halo plans and exchange points; ghosts'
    W, slopes, polynomials and Dt by halo) against the oracle on the same
    partition-constrained hierarchy."""
    from paper_2509_06347_b200 import gmg
    m, fs = _cases()[name]
    W, Winf, _, _ = _state(m, fs, 6)
    part = gmg.gmg_partition_rcb(m.ctr, P)
    s = _solver(m, n_levels=3, part=part, local_domains=P)
    s.set_state(W, Winf)
    hist = s.vcycle(3)
    Wg = s.get_state(0)
    Gg, ag = s.get_ho_state()
    s.close()
    H = oracle.build_hierarchy(m, 3, 0.5, part=part)
    hs = {}
    Wo, ho = oracle.vcycle(H, W, Winf, oracle.Options(fine_operator=1), 3, mesh=m, ho_state=hs)
    assert _rel(Wg, Wo) <= TOL, _rel(Wg, Wo)
    assert _rel(Gg, hs["G"]) <= TOL
    assert _rel(ag, hs["alpha"]) <= TOL
    assert np.max(np.abs(hist - ho) / ho[0][None, :]) <= TOL


@pytest.mark.parametrize("P", [2, 4])
def test_partitioned_one_evaluation_matches_oracle(P):
    from paper_2509_06347_b200 import gmg
    m, fs = _cases()["box3d_prism"]
    W, Winf, G, alpha = _state(m, fs, 7)
    part = gmg.gmg_partition_rcb(m.ctr, P)
    s = _solver(m, n_levels=1, part=part, local_domains=P)
    s.set_state(W, Winf)
    s.set_ho_state(G, alpha)
    R, Gn, a, S = s.ho_residual()
    poly, fl = s.ho_recon()
    s.close()
    Ro, Gno, ao, So, _, _ = cgks3.residual(cgks3.Mesh3(m), W, G, alpha, Winf)
    po, flo, _ = cgks3.recon(cgks3.Mesh3(m), W, G, alpha, Winf)
    assert np.array_equal(fl, flo)
    assert _rel(poly, po) <= TOL
    assert _rel(R, Ro) <= TOL and _rel(Gn, Gno) <= TOL and _rel(a, ao) <= TOL


@pytest.mark.parametrize("name", ["tri2d", "box3d_prism"])
def test_explicit_cgks3_iteration_matches_oracle(name):
    """NEXT-4's explicit arm (the "GPU explicit" row of Table 5):
    the one-level cycle with the third-order operator IS one explicit CGKS3
    iteration (Eq.(smo), readings C12/C14, no coarse correction).  40
    iterations on the device vs the oracle: state, slopes, DF and residual
    history, element by element."""
    from tests.parity import elem
    m, fs = _cases()[name]
    W, Winf, _, _ = _state(m, fs, 7)
    s = _solver(m, n_levels=1)
    s.set_state(W, Winf)
    hist = s.vcycle(40)
    Wg = s.get_state(0)
    Gg, ag = s.get_ho_state()
    s.close()
    H = oracle.build_hierarchy(m, 1, 0.5)
    hs = {}
    Wo, ho = oracle.vcycle(H, W, Winf, oracle.Options(fine_operator=1, n_levels=1), 40, mesh=m, ho_state=hs)
    assert elem(Wg, Wo) <= TOL
    assert elem(Gg.reshape(-1, m.n_cells), hs["G"].reshape(-1, m.n_cells)) <= TOL
    assert elem(ag, hs["alpha"], np.ones_like(ag)) <= TOL
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])


def test_p2min_reading_c3b_matches_oracle():
    """Reading C3b (gmg_options.ho_p2min = d + 2: simplices keep p1):
    on a hybrid quad / triangle O-grid the p2 flags (quads only) are bit-exact
    and 4 V-cycles match the oracle run with the same reading."""
    from tests.parity import elem
    m = configs.naca_ogrid(ni=48, n_quad=8, n_tri=4)
    fs = configs.FREESTREAM[2]
    W, Winf = state.perturbed(m, *fs, eps=0.05, seed=5), state.winf(*fs)
    s = _solver(m, n_levels=3, ho_p2min=4)
    s.set_state(W, Winf)
    poly, fl = s.ho_recon()
    hist = s.vcycle(4)
    Wg = s.get_state(0)
    s.close()
    _, flo, _ = cgks3.recon(cgks3.Mesh3(m), W, np.zeros((4, 2, m.n_cells)), np.ones(m.n_cells), Winf,
                            cgks3.Opt3(p2min=4))
    assert np.array_equal(fl & 1, flo & 1)
    nint = np.zeros(m.n_cells, int)
    for f in range(m.n_faces):
        if m.right[f] >= 0:
            nint[m.left[f]] += 1
            nint[m.right[f]] += 1
    assert np.all((flo & 1) <= (nint >= 4))           # no cell with fewer than 4 interior neighbours uses p2
    H = oracle.build_hierarchy(m, 3, 0.5)
    Wo, ho = oracle.vcycle(H, W, Winf, oracle.Options(fine_operator=1, p2min=4), 4, mesh=m, ho_state={})
    assert elem(Wg, Wo) <= TOL
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])
