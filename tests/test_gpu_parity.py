"""GPU parity: libgmg's CUDA path (through the C ABI) vs the CPU oracle on
the same seeded inputs.  Tolerances: maps bit-exact
(tests/test_abi_host.py); FP64 increments, states, forcing and residuals
element by element, max_i |gpu_i - ref_i| <= 1e-10 max_i |ref_i| per component
(tests/parity.py; BASELINE.json north_star); residual histories
normalised-absolute |r_gpu(k) - r_orc(k)| <= 1e-10 r_orc(0).
"""
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
        W = state.gaussian_bump(m, *fs, jump=True)
    elif name == "box":
        m = configs.box3d(6, 5, 4, 2, seed=3)
        fs = (1.0, (0.6, 0.2, -0.1), 0.7)
        W = state.perturbed(m, *fs, eps=0.1, seed=4)
    elif name == "sphere_small":
        m = configs.sphere_shell(8, 4, 4)
        fs = configs.FREESTREAM[4]
        W = state.bow_shock(m, *fs)
    elif name == "naca_small":
        m = configs.naca_ogrid(ni=96, n_quad=12, n_tri=6)
        fs = configs.FREESTREAM[2]
        W = state.perturbed(m, *fs, eps=0.05, seed=1)
    elif name == "cyl_small":
        m = configs.cylinder_ogrid(ni=96, nr=40, n_tri=8)
        fs = configs.FREESTREAM[3]
        W = state.bow_shock(m, *fs)
    else:
        raise ValueError(name)
    return m, state.winf(*fs), W


CASES = ["config1", "box", "sphere_small", "naca_small", "cyl_small"]


@pytest.mark.parametrize("name", CASES)
def test_residual_parity(G, orc, name):
    m, Winf, W = _case(name)
    s = G.Solver(m, n_levels=1)
    s.set_state(W, Winf)
    R, a, sig = s.residual(0)
    Ro, ao, so, _ = orc.residual(orc.Level.from_mesh(m), W, Winf)
    assert elem(R, Ro) <= 1e-12
    assert elem(a, ao, np.ones_like(ao)) <= 1e-12
    assert elem(sig, so) <= 1e-13
    s.close()


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("n_sweeps", [1, 6])
def test_fine_smooth_parity(G, orc, name, n_sweeps):
    m, Winf, W = _case(name)
    s = G.Solver(m, n_levels=1)
    s.set_state(W, Winf)
    lv = orc.Level.from_mesh(m)
    R, a, S, rf = orc.residual(lv, W, Winf)
    alpha = np.random.default_rng(7).uniform(0.05, 1.0, m.n_cells)
    s.set_level_inputs(0, R, alpha)
    dW = s.smooth(0, n_sweeps)
    col, nc = orc.color(lv)
    D = orc.diag(S, alpha, 10.0, 0.5)
    dWo = orc.smooth(lv, W, R, alpha, D, rf, col, nc, n_sweeps)
    assert elem(dW, dWo) <= TOL
    s.close()


@pytest.mark.parametrize("name", ["config1", "box", "sphere_small"])
def test_coarse_smooth_parity(G, orc, name):
    m, Winf, W = _case(name)
    s = G.Solver(m, n_levels=3)
    s.set_state(W, Winf)
    H = orc.build_hierarchy(m, 3, 0.5)
    for l in (1, 2):
        lv = H[l]["level"]
        # a coarse state: restriction of the fine state
        Wl = W
        for k in range(l):
            Wl, _, _ = orc.restrict(H[k]["parent"], H[k + 1]["level"].n, H[k]["level"].vol, H[k + 1]["level"].vol,
                                    Wl, np.zeros_like(Wl), np.ones(Wl.shape[1]))
        s.set_level_state(l, Wl)
        R, a, S, rf = orc.residual(lv, Wl, Winf)
        alpha = np.random.default_rng(l).uniform(0.05, 1.0, lv.n)
        s.set_level_inputs(l, R, alpha)
        dW = s.smooth(l, 6)
        D = orc.diag(S, alpha, 10.0, 0.5)
        dWo = orc.smooth(lv, Wl, R, alpha, D, rf, H[l]["color"], H[l]["ncolor"], 6)
        assert elem(dW, dWo) <= TOL, f"level {l}"
    s.close()


def _vcycle_pair(G, orc, m, Winf, W, n_cycles, levels=True, **kw):
    """n_cycles V-cycles on both sides; with `levels` the coarse levels of the
    last cycle are compared element by element (tests/parity.check_levels)."""
    opt = orc.Options(**{k: v for k, v in kw.items() if k in orc.Options.__dataclass_fields__})
    fields = [f[0] for f in G.Options._fields_]
    s = G.Solver(m, n_levels=opt.n_levels, **{k: v for k, v in kw.items() if k in fields and k != "n_levels"})
    s.set_state(W, Winf)
    ua = kw.get("_alpha")
    if ua is not None:
        s.set_alpha(ua)
    hist = s.vcycle(n_cycles)
    Wg = s.get_state(0)
    H = orc.build_hierarchy(m, opt.n_levels, opt.skew_limit)
    trace = []
    Wo, ho = orc.vcycle(H, W, Winf, opt, n_cycles, user_alpha=ua, trace=trace)
    if levels and len(H) > 1:
        nc = len(H) - 1
        check_levels(G, s, trace[-nc:], len(H), first=trace[:nc] if n_cycles >= 50 else None)
    s.close()
    return Wg, hist, Wo, ho


@pytest.mark.parametrize("name", CASES)
def test_vcycle_parity_short(G, orc, name):
    m, Winf, W = _case(name)
    Wg, hist, Wo, ho = _vcycle_pair(G, orc, m, Winf, W, 3)
    assert elem(Wg, Wo) <= TOL
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])


def test_vcycle_parity_100_cycles_config1(G, orc):
    """Residual histories over 100 V-cycles (north_star parity bar)."""
    m, Winf, W = _case("config1")
    Wg, hist, Wo, ho = _vcycle_pair(G, orc, m, Winf, W, 100)
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])
    assert elem(Wg, Wo) <= TOL


def test_vcycle_parity_fine_mclusgs(G, orc):
    m, Winf, W = _case("box")
    Wg, hist, Wo, ho = _vcycle_pair(G, orc, m, Winf, W, 3, fine_smoother=1)
    assert elem(Wg, Wo) <= TOL
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])


@pytest.mark.parametrize("df_mode", [1, 2, 3])
def test_vcycle_parity_df_modes(G, orc, df_mode):
    m, Winf, W = _case("config1")
    ua = np.random.default_rng(3).uniform(0, 1, m.n_cells) if df_mode == 1 else None
    Wg, hist, Wo, ho = _vcycle_pair(G, orc, m, Winf, W, 3, df_mode=df_mode, _alpha=ua, beta=0.7)
    assert elem(Wg, Wo) <= TOL


def test_vcycle_parity_fixed_beta_3d(G, orc):
    m, Winf, W = _case("sphere_small")
    Wg, hist, Wo, ho = _vcycle_pair(G, orc, m, Winf, W, 3, df_mode=3, beta=0.3)
    assert elem(Wg, Wo) <= TOL
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])


def test_vcycle_two_levels(G, orc):
    m, Winf, W = _case("config1")
    Wg, hist, Wo, ho = _vcycle_pair(G, orc, m, Winf, W, 2, n_levels=2)
    assert elem(Wg, Wo) <= TOL


def test_freestream_fixed_point_gpu(G):
    m = configs.tri_square(16, 16, seed=2)
    W = state.uniform(m, 1.0, [0.5, 0.1], 0.7)
    s = G.Solver(m, n_levels=3)
    s.set_state(W, state.winf(1.0, [0.5, 0.1], 0.7))
    hist = s.vcycle(3)
    assert np.abs(s.get_state(0) - W).max() <= 1e-12 * np.abs(W).max()
    assert hist.max() < 1e-13
    s.close()


def test_alpha_zero_vcycle_is_explicit_step_gpu(G, orc):
    """P:705-711 + P:519 on the GPU: fine alpha = 0 -> V-cycle = explicit step."""
    m, Winf, W = _case("config1")
    s = G.Solver(m, n_levels=3, df_mode=1)
    s.set_state(W, Winf)
    s.set_alpha(np.zeros(m.n_cells))
    s.vcycle(1)
    R, a, S, _ = orc.residual(orc.Level.from_mesh(m), W, Winf)
    assert rel(s.get_state(0), orc.explicit_update(W, S, R, 0.5)) <= 1e-14
    s.close()


def test_nonfinite_detected(G):
    m, Winf, W = _case("config1")
    W = W.copy()
    W[0, 77] = np.nan
    s = G.Solver(m, n_levels=3)
    s.set_state(W, Winf)
    with pytest.raises(G.GmgError) as e:
        s.vcycle(1)
    assert e.value.status == G.GMG_ENONFINITE
    assert "level" in str(e.value) and "cell" in str(e.value)    # level and cell named
    s.close()


def test_torch_device_buffers(G):
    """Device pointers are accepted at the boundary (cudaMemcpyDefault)."""
    import torch
    m, Winf, W = _case("box")
    s = G.Solver(m, n_levels=2)
    Wd = torch.from_numpy(W).cuda()
    s.set_state(Wd, Winf)
    out = torch.zeros_like(Wd)
    G.gmg_get_state(s.ctx, 0, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), W)
    s.close()


@pytest.mark.parametrize("k", [2, 3])
def test_configs_2_3_full_size_vcycles(G, orc, k):
    """BASELINE configs[1] (NACA0012 O-grid, ~20k mixed cells, no-slip wall)
    and configs[2] (Mach-8 cylinder, 100k cells, bow-shock state, DF-adaptive
    relaxation) at full size: 5 V-cycles, state and history vs the oracle."""
    m = configs.config(k)
    fs = configs.FREESTREAM[k]
    W = state.bow_shock(m, *fs) if k == 3 else state.perturbed(m, *fs, eps=0.05, seed=2)
    Wg, hist, Wo, ho = _vcycle_pair(G, orc, m, state.winf(*fs), W, 5)
    assert elem(Wg, Wo) <= TOL
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])


@pytest.mark.slow
def test_config4_full_size_vcycles(G, orc):
    """BASELINE configs[3] (the bench workload, 1 M cells) at full size, in the
    bench's launch configuration: 10 V-cycles, history, final state and the
    last cycle's coarse levels element by element vs the oracle."""
    m = configs.config(4)
    fs = configs.FREESTREAM[4]
    W = state.bow_shock(m, *fs)
    Winf = state.winf(*fs)
    Wg, hist, Wo, ho = _vcycle_pair(G, orc, m, Winf, W, 10)
    assert elem(Wg, Wo) <= TOL
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])


@pytest.mark.parametrize("name", ["config1", "sphere_small", "cyl_small"])
def test_repeated_phase_skip_is_exact(G, name):
    """The same-color phase at each sweep turn (c_N then c_N, c_1 then c_1) is
    dropped by default (gmg_options.skip_repeat).  A cell's update never reads
    its own state and its other-colored neighbours do not change in between,
    so the repeated phase recomputes the same values: bit for bit at the
    backward -> forward turns; at the first forward -> backward turn the
    repeated phase evaluates the same sum in the W' form X - c sum T(W')
    instead of the first-forward form W - Rt/D - c sum [T(W') - T(W)]
    (DESIGN.md §6), equal up to rounding.  Running every phase of Algorithm 2
    must therefore agree to rounding (and execute more cell-updates)."""
    m, Winf, W = _case(name)
    out = {}
    for v in (0, 1):
        s = G.Solver(m, n_levels=3, skip_repeat=v)
        s.set_state(W, Winf)
        h = s.vcycle(3)
        Wv = s.get_state(0)
        coarse = [s.get_state(l) for l in (1, 2)]
        s.set_level_state(1, coarse[0])
        dW = s.smooth(1, 4)
        out[v] = (h, Wv, coarse, dW, s.vcycle_visits())
        s.close()
    a, b = out[0], out[1]
    assert np.all(np.abs(a[0] - b[0]) <= 1e-13 * a[0][0][None, :])
    assert elem(a[1], b[1]) <= 1e-13
    for x, y in zip(a[2], b[2]):
        assert elem(x, y) <= 1e-13
    assert elem(a[3], b[3]) <= 1e-12
    assert b[4] < a[4]                 # fewer cell-updates executed


@pytest.mark.parametrize("lanes", [1, 4])
def test_sweep_lanes_parity(G, orc, lanes):
    """1 and 4 lanes per cell (another summation order of a cell's slots)."""
    m, Winf, W = _case("sphere_small")
    Wg, hist, Wo, ho = _vcycle_pair(G, orc, m, Winf, W, 3, sweep_lanes=lanes)
    assert elem(Wg, Wo) <= TOL
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])


@pytest.mark.parametrize("name", ["cyl_small", "sphere_small"])
def test_per_cycle_correction_elementwise(G, orc, name):
    """The correction one V-cycle applies to the fine state, W_out - W_in, from
    the SAME input on both sides (the oracle's state of cycle k), element by
    element for 8 consecutive cycles of a bow-shock case (DF alpha spanning
    (0, 1], DF-limited prolongation)."""
    m, Winf, W = _case(name)
    H = orc.build_hierarchy(m, 3, 0.5)
    s = G.Solver(m, n_levels=3)
    Wk = W
    for k in range(8):
        s.set_state(Wk, Winf)
        s.vcycle(1)
        Wg = s.get_state(0)
        Wn, _ = orc.vcycle(H, Wk, Winf, orc.Options(), 1)
        assert elem(Wg - Wk, Wn - Wk) <= TOL, k
        Wk = Wn
    s.close()


@pytest.mark.slow
def test_config3_100_cycles(G, orc):
    """BASELINE configs[2] (Mach-8 cylinder, 100k cells, bow shock, DF-adaptive
    relaxation with alpha spanning (0, 1], DF-limited prolongation across the
    shock) over 100 V-cycles: residual history per component within
    1e-10 of r0, final state and the last cycle's coarse levels element by
    element."""
    m = configs.config(3)
    fs = configs.FREESTREAM[3]
    W = state.bow_shock(m, *fs)
    Wg, hist, Wo, ho = _vcycle_pair(G, orc, m, state.winf(*fs), W, 100)
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])
    assert elem(Wg, Wo) <= TOL


@pytest.mark.slow
def test_config2_long_history(G, orc):
    """BASELINE configs[1] (NACA0012, impulsive start) over 200 V-cycles: the
    residual history stays on the oracle's to 1e-10 of r0 per component and
    the final state to 1e-10 (no drift from reassociation over a long run)."""
    m = configs.config(2)
    fs = configs.FREESTREAM[2]
    Winf = state.winf(*fs)
    W = state.uniform(m, *fs)
    Wg, hist, Wo, ho = _vcycle_pair(G, orc, m, Winf, W, 200)
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])
    assert elem(Wg, Wo) <= TOL


def test_pipelined_host_io_equals_synchronous():
    """gmg_*_async (copy stream, double-buffered staging) give bit-identical
    results to the synchronous calls in the same order, step after step."""
    import torch
    from paper_2509_06347_b200 import gmg
    m = configs.box3d(6, 5, 4, 2, seed=3)
    fs = (1.0, (0.6, 0.2, -0.1), 0.7)
    Winf = state.winf(*fs)
    Ws = [np.ascontiguousarray(state.perturbed(m, *fs, eps=0.1, seed=k)) for k in range(4)]
    s = gmg.Solver(m, n_levels=3)
    ref = []
    for W in Ws:
        s.set_state(W, Winf)
        s.vcycle(2)
        ref.append(s.get_state(0))
    ins = [torch.from_numpy(W).pin_memory() for W in Ws]
    outs = [torch.empty_like(ins[0]).pin_memory() for _ in Ws]
    for k in range(len(Ws)):
        gmg.gmg_set_state_async(s.ctx, ins[k], Winf)
        gmg.gmg_vcycle_async(s.ctx, 2)
        gmg.gmg_get_state_async(s.ctx, outs[k])
    gmg.gmg_sync(s.ctx)
    s.close()
    for k in range(len(Ws)):
        assert np.array_equal(outs[k].numpy(), ref[k]), k


def test_owned_layout_host_io_equals_synchronous():
    """gmg_set/get_state_owned_async (the per-rank layout: owned cells in
    gmg_get_halo order, ghosts by the cycle's halo) on one domain equal the
    natural-order synchronous calls bit for bit."""
    import torch
    from paper_2509_06347_b200 import gmg
    m = configs.box3d(6, 5, 4, 2, seed=3)
    fs = (1.0, (0.6, 0.2, -0.1), 0.7)
    Winf = state.winf(*fs)
    Ws = [np.ascontiguousarray(state.perturbed(m, *fs, eps=0.1, seed=10 + k)) for k in range(3)]
    s = gmg.Solver(m, n_levels=3)
    ref = []
    for W in Ws:
        s.set_state(W, Winf)
        s.vcycle(2)
        ref.append(s.get_state(0))
    own = s.halo(0, 0)["owned"]
    ins = [torch.from_numpy(np.ascontiguousarray(W[:, own])).pin_memory() for W in Ws]
    outs = [torch.empty_like(ins[0]).pin_memory() for _ in Ws]
    for k in range(len(Ws)):
        gmg.gmg_set_state_owned_async(s.ctx, ins[k], Winf)
        gmg.gmg_vcycle_async(s.ctx, 2)
        gmg.gmg_get_state_owned_async(s.ctx, outs[k])
    gmg.gmg_sync(s.ctx)
    s.close()
    for k in range(len(Ws)):
        assert np.array_equal(outs[k].numpy(), ref[k][:, own]), k


def test_async_device_source_is_ordered_after_the_stream():
    """gmg_set_state_async with a DEVICE tensor produced on the compute stream
    (ADVICE r1): the library's copy stream must wait for that producer.  A long
    matmul is queued first, then the new state is written into the tensor on
    the same stream; the async V-cycle must see the new state (bit-identical
    to the synchronous calls on it), not the old one."""
    import torch
    from paper_2509_06347_b200 import gmg
    m = configs.box3d(6, 5, 4, 2, seed=3)
    fs = (1.0, (0.6, 0.2, -0.1), 0.7)
    Winf = state.winf(*fs)
    W1 = np.ascontiguousarray(state.perturbed(m, *fs, eps=0.1, seed=21))
    W2 = np.ascontiguousarray(state.perturbed(m, *fs, eps=0.1, seed=22))
    s = gmg.Solver(m, n_levels=3)
    s.set_state(W2, Winf)
    s.vcycle(1)
    ref = s.get_state(0)
    Wd = torch.from_numpy(W1).cuda()
    W2d = torch.from_numpy(W2).cuda()
    out = torch.empty_like(torch.from_numpy(W1)).pin_memory()
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.float64)
    torch.cuda.synchronize()
    for _ in range(4):
        a = a @ a / 4096.0                      # keeps the stream busy for a while
    Wd.copy_(W2d)                               # the producer, on the compute stream
    gmg.gmg_set_state_async(s.ctx, Wd, Winf)
    gmg.gmg_vcycle_async(s.ctx, 1)
    gmg.gmg_get_state_async(s.ctx, out)
    gmg.gmg_sync(s.ctx)
    s.close()
    assert np.array_equal(out.numpy(), ref)
