"""C-ABI library: loads, exports every symbol include/gmg.h declares, and its
host-side setup (coloring, renumbering, agglomeration, coarse geometry) is
bit-exact against the oracle.  CPU only: no compute call touches a GPU."""
import os
import re

import numpy as np
import pytest

from synth import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def G():
    from paper_2509_06347_b200 import _build
    _build.build()
    from paper_2509_06347_b200 import gmg
    gmg.lib()
    return gmg


def test_exports_every_header_symbol(G):
    hdr = open(os.path.join(ROOT, "include", "gmg.h")).read()
    declared = set(re.findall(r"\b(gmg_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(G.ABI_SYMBOLS)
    L = G.lib()
    for name in declared:
        assert hasattr(L, name), name


def test_default_options(G):
    o = G.gmg_default_options()
    assert (o.dim, o.gamma, o.cfl_imp, o.cfl_exp, o.n_sweeps, o.n_levels, o.pre_smooth, o.post_smooth) == \
        (3, 1.4, 10.0, 0.5, 6, 3, 1, 0)
    assert (o.skew_limit, o.r_factor, o.fine_smoother, o.df_mode, o.nranks) == (0.5, 1.0, 0, 0, 1)


def test_invalid_options_rejected(G):
    for kw in [dict(dim=4), dict(n_sweeps=0), dict(pre_smooth=2), dict(post_smooth=1), dict(df_mode=4),
               dict(df_mode=3, beta=1.5), dict(r_factor=0.5), dict(n_levels=4), dict(nranks=2)]:
        with pytest.raises(G.GmgError) as e:
            G.gmg_create(G.gmg_default_options(**kw))
        assert e.value.status == G.GMG_EINVAL


MESHES = {
    "quad4": lambda: configs.quad_grid(4, 4),
    "trisq": lambda: configs.tri_square(8, 8, seed=3),
    "config1": lambda: configs.config(1),
    "box": lambda: configs.box3d(4, 3, 3, 1, seed=5),
    "naca_small": lambda: configs.naca_ogrid(ni=64, n_quad=8, n_tri=4),
    "sphere_small": lambda: configs.sphere_shell(6, 3, 3),
    "cyl_small": lambda: configs.cylinder_ogrid(ni=32, nr=12),
}


@pytest.mark.parametrize("name", list(MESHES))
def test_maps_bit_exact_vs_oracle(G, orc, name):
    m = MESHES[name]()
    s = G.Solver(m, n_levels=3, build_only=True)
    H = orc.build_hierarchy(m, 3, 0.5)
    assert s.n_levels == len(H)
    for l, e in enumerate(H):
        color, perm, parent = s.maps(l)
        assert np.array_equal(color, e["color"]), f"color level {l}"
        assert s.n_colors(l) == e["ncolor"]
        assert np.array_equal(perm, orc.perm_from_color(e["color"])), f"perm level {l}"
        if e["parent"] is not None:
            assert np.array_equal(parent, e["parent"]), f"parent level {l}"
        else:
            assert np.all(parent == -1)
        g = s.geometry(l)
        lv = e["level"]
        for k in ("vol", "ctr", "left", "right", "avec", "fctr", "ngauss"):
            assert np.array_equal(g[k], getattr(lv, k)), f"{k} level {l}"
    s.close()


def test_user_coloring_validated(G):
    m = configs.quad_grid(3, 3)
    ctx = G.gmg_create(G.gmg_default_options(dim=2))
    G.gmg_load_mesh(ctx, m)
    with pytest.raises(G.GmgError) as e:
        G.gmg_set_coloring(ctx, 0, np.ones(9, np.int32))
    assert e.value.status == G.GMG_ECOLOR
    j, i = np.divmod(np.arange(9), 3)
    good = ((i + j) % 2 + 1).astype(np.int32)[::-1].copy()   # the other checkerboard
    G.gmg_set_coloring(ctx, 0, good)
    nb, st = G.gmg_build_hierarchy(ctx, 1)
    col, perm, _ = G.gmg_get_maps(ctx, 0)
    assert np.array_equal(col, good)
    G.gmg_destroy(ctx)


def test_topology_errors(G):
    m = configs.quad_grid(2, 2)
    ctx = G.gmg_create(G.gmg_default_options(dim=2))
    bad = configs.quad_grid(2, 2)
    bad.right = bad.right.copy()
    bad.right[bad.right >= 0][0:1] = 99
    idx = np.nonzero(bad.right >= 0)[0][0]
    bad.right[idx] = 99                                 # out of range
    with pytest.raises(G.GmgError) as e:
        G.gmg_load_mesh(ctx, bad)
    assert e.value.status == G.GMG_ETOPO
    open_ = configs.quad_grid(2, 2)
    open_.avec = open_.avec.copy()
    open_.avec[0, 0] *= 2.0                             # breaks closure of its cells
    with pytest.raises(G.GmgError) as e:
        G.gmg_load_mesh(ctx, open_)
    assert e.value.status == G.GMG_ETOPO
    G.gmg_load_mesh(ctx, m)
    G.gmg_destroy(ctx)


def test_stall_truncates_hierarchy(G):
    s = G.Solver(configs.single_cell(2), n_levels=3, build_only=True)
    assert s.n_levels == 1 and s.build_status == G.GMG_ESTALL


def test_state_calls_require_workspace(G):
    ctx = G.gmg_create(G.gmg_default_options(dim=2))
    G.gmg_load_mesh(ctx, configs.quad_grid(2, 2))
    G.gmg_build_hierarchy(ctx, 2)
    with pytest.raises(G.GmgError) as e:
        G.gmg_vcycle(ctx, 1)
    assert e.value.status == G.GMG_ESTATE
    assert G.gmg_workspace_bytes(ctx) > 0
    G.gmg_destroy(ctx)
