"""The oracle's timing build (bench.py's CPU baseline: -O3 -march=native,
OpenMP within a color, built on the host) computes the same bits as the
parity build: its pragmas only parallelise independent iterations (cells of
one color, per-face flux evaluations, per-cell updates) and every sum keeps
its sequential order.  CPU only."""
import numpy as np
import pytest

from synth import configs, state


@pytest.mark.parametrize("which", ["config1", "box", "sphere_small"])
def test_timing_build_bit_identical(orc, which):
    if which == "config1":
        m = configs.config(1)
        fs = configs.FREESTREAM[1]
        W = state.gaussian_bump(m, *fs, jump=True)
    elif which == "box":
        m = configs.box3d(5, 4, 4, 2, seed=3)
        fs = (1.0, (0.6, 0.2, -0.1), 0.7)
        W = state.perturbed(m, *fs, eps=0.1, seed=4)
    else:
        m = configs.sphere_shell(6, 3, 3)
        fs = configs.FREESTREAM[4]
        W = state.bow_shock(m, *fs)
    Winf = state.winf(*fs)
    H = orc.build_hierarchy(m, 3, 0.5)
    Wa, ha = orc.vcycle(H, W, Winf, orc.Options(), 2)
    try:
        orc.use_timing_build(4)
        Wb, hb = orc.vcycle(H, W, Winf, orc.Options(), 2)
    finally:
        orc.use_parity_build()
    assert np.array_equal(Wa, Wb) and np.array_equal(ha, hb)
