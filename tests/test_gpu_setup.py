"""Device-side setup: Algorithm 1 coloring and
Algorithm 3 agglomeration run on the GPU (gmg_options.setup_device = 1) must
give the host setup's hierarchy bit for bit -- colors, renumbering, parent
maps and the coarse geometry built from them -- on every mesh family, with
and without the partition constraint, and on a disconnected mesh (the
Algorithm-1 restart at the least uncolored id)."""
import dataclasses

import numpy as np
import pytest

from synth import configs
from synth.mesh import Mesh

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


def _concat(a: Mesh, b: Mesh) -> Mesh:
    """two meshes side by side, no shared face (a disconnected mesh)"""
    na = a.vol.size
    shift = lambda r: np.where(r >= 0, r + na, r)
    return dataclasses.replace(
        a, vol=np.concatenate([a.vol, b.vol]), ctr=np.concatenate([a.ctr, b.ctr + 10.0], axis=1),
        left=np.concatenate([a.left, b.left + na]), right=np.concatenate([a.right, shift(b.right)]),
        avec=np.concatenate([a.avec, b.avec], axis=1), fctr=np.concatenate([a.fctr, b.fctr + 10.0], axis=1),
        ngauss=np.concatenate([a.ngauss, b.ngauss]), name="disconnected")


MESHES = {
    "config1": lambda: configs.config(1),
    "config2": lambda: configs.config(2),
    "cylinder": lambda: configs.cylinder_ogrid(64, 24),
    "box": lambda: configs.box3d(9, 7, 6, 2, seed=5),
    "sphere": lambda: configs.sphere_shell(10, 4, 4),
    "disconnected": lambda: _concat(configs.box3d(5, 4, 3, 1, seed=1), configs.box3d(4, 4, 4, 2, seed=2)),
}


def _hier(G, m, dev, part=None, P=1):
    kw = dict(setup_device=dev)
    if part is not None:
        kw.update(part=part, local_domains=P)
    s = G.Solver(m, n_levels=3, build_only=True, **kw)
    out = []
    for l in range(s.n_levels):
        col, perm, par = s.maps(l)
        geo = s.geometry(l)
        out.append((col, perm, par, geo))
    s.close()
    return out


@pytest.mark.parametrize("name", list(MESHES))
def test_device_setup_equals_host(G, name):
    m = MESHES[name]()
    h = _hier(G, m, 0)
    d = _hier(G, m, 1)
    assert len(h) == len(d)
    for (c0, p0, q0, g0), (c1, p1, q1, g1) in zip(h, d):
        assert np.array_equal(c0, c1)
        assert np.array_equal(p0, p1)
        assert np.array_equal(q0, q1)
        for k in g0:
            assert np.array_equal(g0[k], g1[k]), k


@pytest.mark.parametrize("P", [2, 5])
def test_device_setup_partitioned(G, P):
    m = configs.sphere_shell(10, 4, 4)
    part = G.gmg_partition_rcb(m.ctr, P)
    h = _hier(G, m, 0, part, P)
    d = _hier(G, m, 1, part, P)
    for (c0, p0, q0, _), (c1, p1, q1, _) in zip(h, d):
        assert np.array_equal(c0, c1) and np.array_equal(p0, p1) and np.array_equal(q0, q1)


def _oracle_maps(orc, m, part=None):
    """the oracle's hierarchy (O1-O3): per level (color, perm, parent, geometry)"""
    H = orc.build_hierarchy(m, 3, 0.5, part=part)
    out = []
    for k, e in enumerate(H):
        lv = e["level"]
        par = e["parent"] if e["parent"] is not None else np.full(lv.n, -1, np.int64)
        geo = dict(vol=lv.vol, ctr=lv.ctr, left=lv.left, right=lv.right, avec=lv.avec, fctr=lv.fctr,
                   ngauss=lv.ngauss)
        out.append((e["color"], orc.perm_from_color(e["color"]), par, geo))
    return out


@pytest.mark.slow
def test_device_setup_full_size_vs_oracle(G, orc):
    """config 4 (998,400 cells, the benchmark's mesh): the DEVICE-built
    hierarchy (Algorithms 1 and 3 on the GPU) against the ORACLE's, bit for
    bit -- colors, renumbering, parent maps and the coarse geometry."""
    m = configs.config(4)
    d = _hier(G, m, 1)
    o = _oracle_maps(orc, m)
    assert len(d) == len(o)
    for l, ((c1, p1, q1, g1), (c0, p0, q0, g0)) in enumerate(zip(d, o)):
        assert np.array_equal(c1, c0), l
        assert np.array_equal(p1, p0), l
        assert np.array_equal(q1, q0), l
        for k in g0:
            assert np.array_equal(np.asarray(g1[k]).ravel(), np.asarray(g0[k]).ravel()), (l, k)


@pytest.mark.parametrize("name", ["sphere", "disconnected"])
def test_device_setup_vs_oracle(G, orc, name):
    m = MESHES[name]()
    d = _hier(G, m, 1)
    o = _oracle_maps(orc, m)
    for (c1, p1, q1, g1), (c0, p0, q0, g0) in zip(d, o):
        assert np.array_equal(c1, c0) and np.array_equal(p1, p0) and np.array_equal(q1, q0)
        for k in g0:
            assert np.array_equal(np.asarray(g1[k]).ravel(), np.asarray(g0[k]).ravel()), k


def test_device_built_hierarchy_runs_identically(G):
    """V-cycles on the device-built hierarchy give the same bits as on the
    host-built one (same colors, order and parents -> same arithmetic)."""
    from synth import state
    m = configs.sphere_shell(10, 4, 4)
    fs = configs.FREESTREAM[4]
    W, Winf = state.bow_shock(m, *fs), state.winf(*fs)
    out = []
    for dev in (0, 1):
        s = G.Solver(m, n_levels=3, setup_device=dev)
        s.set_state(W, Winf)
        h = s.vcycle(3)
        out.append((h, s.get_state(0)))
        s.close()
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
