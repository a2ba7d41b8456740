"""GPU parity of the partitioned path: P sub-domains driven
in one process on one GPU (gmg_options.local_domains = P) -- the same
layouts, halo plans, pack/unpack kernels and exchange points as the NCCL
path, with device copies as the transport -- against the oracle run on the
same partition-constrained hierarchy."""
import numpy as np
import pytest

from synth import configs, state
from tests.parity import TOL, check_levels, elem, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_06347_b200 import _build, gmg
    _build.build()
    gmg.lib()
    return gmg


def _case(name):
    if name == "config1":
        m = configs.config(1)
        fs = configs.FREESTREAM[1]
        return m, state.winf(*fs), state.gaussian_bump(m, *fs, jump=True)
    if name == "box":
        m = configs.box3d(6, 5, 4, 2, seed=3)
        fs = (1.0, (0.6, 0.2, -0.1), 0.7)
        return m, state.winf(*fs), state.perturbed(m, *fs, eps=0.1, seed=4)
    m = configs.sphere_shell(8, 4, 4)
    fs = configs.FREESTREAM[4]
    return m, state.winf(*fs), state.bow_shock(m, *fs)


@pytest.mark.parametrize("mode", ["serial", "overlap", "p2p"])
@pytest.mark.parametrize("name", ["config1", "box", "sphere"])
@pytest.mark.parametrize("P", [2, 3, 4])
def test_partitioned_vcycle_parity(G, orc, name, P, mode, monkeypatch):
    # serial: pack / transport / unpack after every color; overlap: boundary
    # cells first, exchange on a side stream while the interior is swept (the
    # NCCL default); p2p: the fused halo -- the sweep epilogue stores the
    # increments into the peers' ghost records and publishes its phase count
    m, Winf, W = _case(name)
    part = G.gmg_partition_rcb(m.ctr, P)
    s = G.Solver(m, n_levels=3, part=part, local_domains=P, overlap=1 if mode == "overlap" else 0,
                 p2p=1 if mode == "p2p" else 0)
    s.set_state(W, Winf)
    hist = s.vcycle(3)
    Wg = s.get_state(0)
    H = orc.build_hierarchy(m, 3, 0.5, part=part)
    trace = []
    Wo, ho = orc.vcycle(H, W, Winf, orc.Options(), 3, trace=trace)
    assert elem(Wg, Wo) <= TOL
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])
    # coarse levels of the last cycle, element by element: restricted W0, forcing, increments, states
    check_levels(G, s, trace[-2:], len(H))
    s.close()


def test_partitioned_fine_mclusgs_parity(G, orc):
    m, Winf, W = _case("box")
    part = G.gmg_partition_rcb(m.ctr, 3)
    s = G.Solver(m, n_levels=3, part=part, local_domains=3, fine_smoother=1)
    s.set_state(W, Winf)
    s.vcycle(2)
    H = orc.build_hierarchy(m, 3, 0.5, part=part)
    Wo, _ = orc.vcycle(H, W, Winf, orc.Options(fine_smoother=1), 2)
    assert rel(s.get_state(0), Wo) <= TOL
    s.close()


@pytest.mark.parametrize("P", [2, 4])
def test_partitioned_smooth_and_residual_parity(G, orc, P):
    m, Winf, W = _case("sphere")
    part = G.gmg_partition_rcb(m.ctr, P)
    s = G.Solver(m, n_levels=1, part=part, local_domains=P)
    s.set_state(W, Winf)
    lv = orc.Level.from_mesh(m)
    R, a, S, rf = orc.residual(lv, W, Winf)
    Rg, ag, Sg = s.residual(0)
    assert rel(Rg, R) <= 1e-12 and rel(Sg, S) <= 1e-13
    alpha = np.random.default_rng(9).uniform(0.05, 1.0, m.n_cells)
    s.set_level_inputs(0, R, alpha)
    dW = s.smooth(0, 6)
    col, nc = orc.color(lv)
    dWo = orc.smooth(lv, W, R, alpha, orc.diag(S, alpha, 10.0, 0.5), rf, col, nc, 6)
    assert rel(dW, dWo) <= TOL
    s.close()


def test_partition_one_domain_equals_unpartitioned(G):
    """P = 1 with a part[] array is the single-domain path."""
    m, Winf, W = _case("config1")
    a = G.Solver(m, n_levels=3)
    a.set_state(W, Winf)
    ha = a.vcycle(2)
    b = G.Solver(m, n_levels=3, part=np.zeros(m.n_cells, np.int32), local_domains=1)
    b.set_state(W, Winf)
    hb = b.vcycle(2)
    assert np.array_equal(a.get_state(0), b.get_state(0)) and np.array_equal(ha, hb)
    a.close()
    b.close()


@pytest.mark.parametrize("P", [2, 4])
def test_p2p_smooth_equals_exchange(G, monkeypatch, P):
    """gmg_smooth with the fused P2P halo gives the same increments as the
    pack / copy / unpack exchange (same arithmetic, only the transport differs)."""
    m, Winf, W = _case("sphere")
    part = G.gmg_partition_rcb(m.ctr, P)
    out = {}
    for mode in ("0", "1"):
        s = G.Solver(m, n_levels=3, part=part, local_domains=P, p2p=int(mode))
        s.set_state(W, Winf)
        s.vcycle(1)
        dW = s.smooth(1, 3)   # level 1's Rt = R(W) + F from the cycle
        assert np.all(np.isfinite(dW))
        out[mode] = (dW, s.get_state(0))
        s.close()
    assert np.array_equal(out["0"][0], out["1"][0])
    assert np.array_equal(out["0"][1], out["1"][1])


@pytest.mark.parametrize("mode", ["serial", "p2p"])
@pytest.mark.parametrize("kw", [dict(fine_smoother=1), dict(df_mode=2), dict(df_mode=3, beta=0.5)])
def test_partitioned_variants_parity(G, orc, mode, kw, monkeypatch):
    """MC-LU-SGS on the fine level, DF off and fixed-beta relaxation on the
    partitioned path (copy exchange and fused P2P halo) vs the oracle."""
    m, Winf, W = _case("box")
    part = G.gmg_partition_rcb(m.ctr, 3)
    s = G.Solver(m, n_levels=3, part=part, local_domains=3, p2p=1 if mode == "p2p" else 0, **kw)
    s.set_state(W, Winf)
    hist = s.vcycle(2)
    H = orc.build_hierarchy(m, 3, 0.5, part=part)
    Wo, ho = orc.vcycle(H, W, Winf, orc.Options(**kw), 2)
    assert rel(s.get_state(0), Wo) <= TOL
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])
    s.close()


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("level", [0, 1])
def test_p2p_protocol_under_concurrency(G, monkeypatch, P, level):
    """The fused-P2P-halo protocol with the domains running at the SAME time:
    one cooperative launch, one block group per domain, each waiting on its
    peers' phase counts (the single-GPU stand-in for ranks that wait on one
    another).  Same increments as the sequential launches (up to the
    summation order of the lanes per cell)."""
    m, Winf, W = _case("sphere")
    part = G.gmg_partition_rcb(m.ctr, P)
    s = G.Solver(m, n_levels=3, part=part, local_domains=P, p2p=1)
    s.set_state(W, Winf)
    s.vcycle(1)
    ref = s.smooth(level, 4)
    emu = G.gmg_p2p_emulate_smooth(s.ctx, level, 4, s.nv, s.n_cells(level))
    assert np.all(np.isfinite(emu))
    assert rel(emu, ref) <= 1e-12
    s.close()
