"""Partitioned path, host side: partitioner,
partition-constrained hierarchy (bit-exact vs the oracle), halo plans --
checked in one process over all local domains, and across two processes
with torch.distributed gloo (world_size 2).  CPU only."""
import os
import socket

import numpy as np
import pytest

from synth import configs


@pytest.fixture(scope="module")
def G():
    from paper_2509_06347_b200 import _build, gmg
    _build.build()
    gmg.lib()
    return gmg


MESHES = {
    "config1": lambda: configs.config(1),
    "box": lambda: configs.box3d(6, 5, 4, 2, seed=3),
    "sphere_small": lambda: configs.sphere_shell(6, 3, 3),
}


def test_rcb_partition(G):
    m = configs.box3d(6, 6, 4, 1, seed=2)
    for P in (1, 2, 3, 4, 8):
        part = G.gmg_partition_rcb(m.ctr, P)
        assert part.min() == 0 and part.max() == P - 1
        cnt = np.bincount(part, minlength=P)
        assert cnt.max() - cnt.min() <= 1                    # balanced to one cell
        assert np.array_equal(part, G.gmg_partition_rcb(m.ctr, P))   # deterministic
        from synth.partition import rcb
        assert np.array_equal(part, rcb(m.ctr, P))                   # the reference arm's restatement


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("P", [2, 4])
def test_partitioned_hierarchy_matches_oracle(G, orc, name, P):
    """Agglomeration never crosses a partition face; maps stay
    bit-exact vs the oracle run with the same partition."""
    m = MESHES[name]()
    part = G.gmg_partition_rcb(m.ctr, P)
    s = G.Solver(m, n_levels=3, build_only=True, part=part, local_domains=P)
    H = orc.build_hierarchy(m, 3, 0.5, part=part)
    assert s.n_levels == len(H)
    for l, e in enumerate(H):
        color, perm, parent = s.maps(l)
        assert np.array_equal(color, e["color"])
        if e["parent"] is not None:
            assert np.array_equal(parent, e["parent"])
            # coarse cells never straddle partitions
            pc = np.full(parent.max() + 1, -1)
            lp = e["part"] if e["part"] is not None else part
            for i, c in enumerate(parent):
                assert pc[c] in (-1, lp[i])
                pc[c] = lp[i]
    s.close()


def _plans(s, P, level):
    return [s.halo(level, d) for d in range(P)]


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("P", [2, 3, 4])
def test_halo_plans_consistent(G, orc, name, P):
    m = MESHES[name]()
    part = G.gmg_partition_rcb(m.ctr, P)
    s = G.Solver(m, n_levels=3, build_only=True, part=part, local_domains=P)
    H = orc.build_hierarchy(m, 3, 0.5, part=part)
    for l in range(s.n_levels):
        lv = H[l]["level"]
        lpart = part if l == 0 else H[l]["part"]
        col = H[l]["color"]
        plans = _plans(s, P, l)
        owned_all = np.concatenate([p["owned"] for p in plans])
        assert np.array_equal(np.sort(owned_all), np.arange(lv.n))          # owned sets partition the cells
        inn = lv.right >= 0
        L, R = lv.left[inn], lv.right[inn]
        for r, p in enumerate(plans):
            assert np.all(lpart[p["owned"]] == r)
            # owned in (color, boundary first) blocks (boundary = has a face
            # neighbour on another partition: exchange overlap); inside a
            # block the cells follow the Morton key of their centroid
            mine = lpart == r
            bnd = np.zeros(lv.n, bool)
            bnd[L[mine[L] & ~mine[R]]] = True
            bnd[R[mine[R] & ~mine[L]]] = True
            o = p["owned"]
            key = col[o].astype(np.int64) * 2 + (~bnd[o])
            assert np.all(np.diff(key) >= 0)
            assert len(np.unique(o)) == len(o)
            # ghosts = exactly the non-owned face neighbours of owned cells
            gh = np.unique(np.concatenate([R[mine[L] & ~mine[R]], L[mine[R] & ~mine[L]]]))
            assert np.array_equal(np.sort(p["ghost"]), gh)
            assert set(p["peers"].tolist()) == set(lpart[gh].tolist())
        nc = s.n_colors(l)
        for r, p in enumerate(plans):
            npr = len(p["peers"])
            for k, q in enumerate(p["peers"]):
                pq = plans[q]
                kk = list(pq["peers"]).index(r)
                nq = len(pq["peers"])
                for c in range(nc):
                    snd = p["send"][p["send_off"][c * npr + k]:p["send_off"][c * npr + k + 1]]
                    rcv = pq["recv"][pq["recv_off"][c * nq + kk]:pq["recv_off"][c * nq + kk + 1]]
                    assert np.array_equal(snd, rcv), (l, r, q, c)        # element-wise identical groups
                    assert np.all(col[snd] == c + 1) and np.all(np.diff(snd) > 0)
    s.close()


def _check_targets(owned, off, k, g, peers, ghost_of_peer, n_own_of_peer):
    """every fused-halo target must be the peer's ghost copy of the same natural cell"""
    for i in range(len(owned)):
        for m in range(off[i], off[i + 1]):
            q = peers[k[m]]
            gl = g[m] - n_own_of_peer[q]
            if not (0 <= gl < len(ghost_of_peer[q]) and ghost_of_peer[q][gl] == owned[i]):
                return False
    return True


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("P", [2, 3])
def test_p2p_targets_local_domains(G, name, P, monkeypatch):
    """Fused P2P halo addressing (host side): each owned boundary cell's
    targets are exactly the peers' ghost copies of that cell, and every ghost
    of every domain is targeted by its owner exactly once."""
    m = MESHES[name]()
    part = G.gmg_partition_rcb(m.ctr, P)
    s = G.Solver(m, n_levels=3, build_only=True, part=part, local_domains=P, p2p=1)
    for l in range(s.n_levels):
        plans = _plans(s, P, l)
        ghost_of = {r: p["ghost"] for r, p in enumerate(plans)}
        n_own = {r: len(p["owned"]) for r, p in enumerate(plans)}
        hit = {r: np.zeros(len(p["ghost"]), int) for r, p in enumerate(plans)}
        for r, p in enumerate(plans):
            off, k, g = G.gmg_get_p2p_targets(s.ctx, l, r)
            assert _check_targets(p["owned"], off, k, g, p["peers"], ghost_of, n_own)
            for m_ in range(len(k)):
                hit[p["peers"][k[m_]]][g[m_] - n_own[p["peers"][k[m_]]]] += 1
        for r in hit:
            assert np.all(hit[r] == 1)
    s.close()


def _worker(rank, world, port, name, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_06347_b200 import gmg
        m = MESHES[name]()
        part = gmg.gmg_partition_rcb(m.ctr, world)
        s = gmg.Solver(m, n_levels=3, build_only=True, part=part, nranks=world, rank=rank, nccl_id=bytes(128), p2p=1)
        ok = True
        for l in range(s.n_levels):
            mine = s.halo(l, 0)
            allp = [None] * world
            dist.all_gather_object(allp, {k: (v.tolist() if hasattr(v, "tolist") else v) for k, v in mine.items()})
            nc = s.n_colors(l)
            for k, peer in enumerate(mine["peers"]):
                other = allp[peer]
                kk = other["peers"].index(rank)
                npr, nq = len(mine["peers"]), len(other["peers"])
                for c in range(nc):
                    snd = mine["send"][mine["send_off"][c * npr + k]:mine["send_off"][c * npr + k + 1]].tolist()
                    rcv = other["recv"][other["recv_off"][c * nq + kk]:other["recv_off"][c * nq + kk + 1]]
                    ok &= snd == rcv
            owned = [None] * world
            dist.all_gather_object(owned, mine["owned"].tolist())
            n = s.n_cells(l)
            ok &= sorted(sum(owned, [])) == list(range(n))
            # fused P2P halo targets built from each rank's own view of its peers
            off, k, g = gmg.gmg_get_p2p_targets(s.ctx, l, 0)
            ghost_of = {r: allp[r]["ghost"] for r in range(world)}
            n_own = {r: len(allp[r]["owned"]) for r in range(world)}
            ok &= _check_targets(mine["owned"], off, k, g, mine["peers"], ghost_of, n_own)
        s.close()
        # NEXT-1 host setup on this rank's domain (owned + ghost geometry, slots, p2 operators): the
        # workspace sizing runs it; it must succeed on every rank and add to the first-order workspace
        s0 = gmg.Solver(m, n_levels=3, build_only=True, part=part, nranks=world, rank=rank, nccl_id=bytes(128))
        s1 = gmg.Solver(m, n_levels=3, build_only=True, part=part, nranks=world, rank=rank, nccl_id=bytes(128),
                        fine_operator=1)
        b0, b1 = gmg.gmg_workspace_bytes(s0.ctx), gmg.gmg_workspace_bytes(s1.ctx)
        ok &= b0 > 0 and b1 > b0
        s0.close()
        s1.close()
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["config1", "box"])
def test_two_process_gloo_halo_symmetry(G, name):
    """world_size-2 gloo run: each process builds only its own rank's domain
    (nranks = 2, as under torchrun) and the plans agree across processes."""
    import multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
