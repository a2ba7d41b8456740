"""GPU parity on the degenerate meshes the method has (DESIGN.md §4 "edge
cases"): a cell with no interior face (single triangle/quad/tet: every slot
list empty, the sweep reduces to dW = -Rt/D, the hierarchy stalls at one
level), two cells (one interior face, one color pair), a one-cell-thick
strip (every coarse level a chain, ragged last color), and a strip of odd
length (an unmerged cell left over by the agglomeration).  Each runs V-cycles
through the C ABI with both fine smoothers and is compared with the oracle at
the parity bar of tests/test_gpu_parity.py (relative L2 <= 1e-10, histories
<= 1e-10 of the first norm)."""
import numpy as np
import pytest

from synth import configs, state

pytestmark = pytest.mark.gpu
TOL = 1e-10

FS2 = (1.0, (0.5, 0.2), 0.8)
FS3 = (1.0, (0.6, 0.2, -0.1), 0.7)

MESHES = {
    "single_quad": lambda: (configs.single_cell(2), FS2),
    "single_tet": lambda: (configs.single_cell(3), FS3),
    "two_cells": lambda: (configs.two_cells(), FS2),
    "strip_16": lambda: (configs.quad_grid(16, 1), FS2),
    "strip_odd_tri": lambda: (configs.tri_square(7, 1, seed=2), FS2),
    "box_thin": lambda: (configs.box3d(5, 1, 1, 0, seed=1), FS3),
}


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def G():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_06347_b200 import _build, gmg
    _build.build()
    gmg.lib()
    return gmg


@pytest.mark.parametrize("fine_smoother", [0, 1], ids=["explicit", "mclusgs"])
@pytest.mark.parametrize("name", list(MESHES))
def test_degenerate_vcycle_parity(G, orc, name, fine_smoother):
    m, fs = MESHES[name]()
    W = state.perturbed(m, *fs, eps=0.1, seed=7)
    Winf = state.winf(*fs)
    opt = orc.Options(fine_smoother=fine_smoother)
    H = orc.build_hierarchy(m, opt.n_levels, opt.skew_limit)
    s = G.Solver(m, n_levels=3, fine_smoother=fine_smoother)
    assert s.n_levels == len(H)
    for l in range(len(H)):
        col, perm, parent = s.maps(l)
        assert np.array_equal(col, H[l]["color"])
        assert np.array_equal(perm, orc.perm_from_color(H[l]["color"]))
        if H[l]["parent"] is not None:
            assert np.array_equal(parent, H[l]["parent"])
    s.set_state(W, Winf)
    hist = s.vcycle(5)
    Wg = s.get_state(0)
    s.close()
    Wo, ho = orc.vcycle(H, W, Winf, opt, 5)
    assert rel(Wg, Wo) <= TOL
    assert np.all(np.abs(hist - ho) <= TOL * ho[0][None, :])
