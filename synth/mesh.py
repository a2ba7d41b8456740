"""Unstructured mesh container + a vectorised face/geometry builder.

The mesh format is the one the C ABI (`include/gmg.h`, gmg_load_mesh) and the
oracle both ingest:

* cells: ``vol[n]``, ``ctr[d][n]`` (SoA)
* faces: ``left[nf]`` (owner cell), ``right[nf]`` (other cell, or
  ``-(patch+1)`` for a boundary face), ``avec[d][nf]`` the area vector
  ``S_f n_f`` pointing left -> right (outward from ``left``), ``fctr[d][nf]``
  the face centre, ``ngauss[nf]`` the number of Gauss points M_f of that face
  (2 per 2D segment, 3 per triangle, 4 per quad; PAPER.md:164-176 / SPEC S:75).
* ``patch_kind[n_patches]``: FARFIELD / SLIP / NOSLIP / EXTRAP.

Geometry is computed ONCE here, in numpy float64; nothing downstream
recomputes it.  This file contains no arithmetic of the paper's method.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

FARFIELD, SLIP, NOSLIP, EXTRAP = 0, 1, 2, 3

# cell types
TRI2, QUAD2, TET, PRISM = 0, 1, 2, 3

# local face templates (cyclic node order inside each face)
_FACES = {
    TRI2: [(0, 1), (1, 2), (2, 0)],
    QUAD2: [(0, 1), (1, 2), (2, 3), (3, 0)],
    TET: [(0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)],
    PRISM: [(0, 1, 2), (3, 4, 5), (0, 1, 4, 3), (1, 2, 5, 4), (2, 0, 3, 5)],
}
_NNODES = {TRI2: 3, QUAD2: 4, TET: 4, PRISM: 6}


@dataclass
class Mesh:
    dim: int
    vol: np.ndarray          # [n] float64
    ctr: np.ndarray          # [d][n] float64
    left: np.ndarray         # [nf] int64
    right: np.ndarray        # [nf] int64 (<0: -(patch+1))
    avec: np.ndarray         # [d][nf] float64
    fctr: np.ndarray         # [d][nf] float64
    ngauss: np.ndarray       # [nf] int8
    patch_kind: np.ndarray   # [n_patches] int32
    name: str = ""
    meta: dict = field(default_factory=dict)
    # high-order geometry (NEXT-1, third-order CGKS fine operator):
    m2: np.ndarray = None    # [d(d+1)/2][n] central second moments (1/|Omega|) int (x-x_c)_a (x-x_c)_b dV,
                             #   components xx, xy, (xz,) yy, (yz, zz)  -- upper triangle, row major
    gp: np.ndarray = None    # [d][G][nf] face Gauss points (G = 2 in 2D, 4 in 3D; triangles pad slot 3)
    gw: np.ndarray = None    # [G][nf] Gauss weights, sum_k gw[k][f] = 1 (padding weight 0)

    @property
    def n_cells(self) -> int:
        return int(self.vol.shape[0])

    @property
    def n_faces(self) -> int:
        return int(self.left.shape[0])

    @property
    def n_interior(self) -> int:
        return int(np.count_nonzero(self.right >= 0))

    def contiguous(self) -> "Mesh":
        for k in ("vol", "ctr", "avec", "fctr", "m2", "gp", "gw"):
            if getattr(self, k) is not None:
                setattr(self, k, np.ascontiguousarray(getattr(self, k), dtype=np.float64))
        self.left = np.ascontiguousarray(self.left, dtype=np.int64)
        self.right = np.ascontiguousarray(self.right, dtype=np.int64)
        self.ngauss = np.ascontiguousarray(self.ngauss, dtype=np.int8)
        self.patch_kind = np.ascontiguousarray(self.patch_kind, dtype=np.int32)
        return self


def _cross(a, b):
    return np.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                     a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                     a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], axis=-1)


def _tet_vol_ctr(a, b, c, d):
    v = np.abs(np.einsum("ij,ij->i", b - a, _cross(c - a, d - a))) / 6.0
    return v, (a + b + c + d) / 4.0


def _simplex_m2(P, scale):
    """sum over a simplex of int x_a x_b for vertices P (list of [k][d], already
    shifted to the cell centroid): scale * (sum_i p_ia p_ib + (sum_i p_ia)(sum_i p_ib)),
    scale = |T|/12 (triangle) or |T|/20 (tetrahedron).  Returns [k][d][d]."""
    S = sum(P)
    out = np.einsum("ka,kb->kab", S, S)
    for p in P:
        out += np.einsum("ka,kb->kab", p, p)
    return out * scale[:, None, None]


def _cell_m2(dim, nodes, cell_type, conn, ctr, vol):
    """central second moments (1/|Omega|) int (x-x_c)(x-x_c)^T dV, exact for the
    straight-sided cells (fan triangulation / tetrahedral split of the cell)."""
    n = cell_type.shape[0]
    M = np.zeros((n, dim, dim))
    for t in np.unique(cell_type):
        idx = np.nonzero(cell_type == t)[0]
        c = conn[idx]
        X = [nodes[c[:, i]] - ctr[idx] for i in range(_NNODES[int(t)])]
        if t in (TRI2, QUAD2):
            tris = [(0, 1, 2)] if t == TRI2 else [(0, 1, 2), (0, 2, 3)]
            for (a, b, cc) in tris:
                e1, e2 = X[b] - X[a], X[cc] - X[a]
                ar = 0.5 * np.abs(e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0])
                M[idx] += _simplex_m2([X[a], X[b], X[cc]], ar / 12.0)
        else:
            tets = [(0, 1, 2, 3)] if t == TET else [(0, 1, 2, 5), (0, 1, 5, 4), (0, 4, 5, 3)]
            for (a, b, cc, d) in tets:
                v = np.abs(np.einsum("ij,ij->i", X[b] - X[a], _cross(X[cc] - X[a], X[d] - X[a]))) / 6.0
                M[idx] += _simplex_m2([X[a], X[b], X[cc], X[d]], v / 20.0)
    M /= vol[:, None, None]
    iu = np.triu_indices(dim)
    return np.ascontiguousarray(M[:, iu[0], iu[1]].T)


def _face_gauss(dim, nodes, fnodes):
    """Gauss points of every face (3 per triangle, 4 per quad;
    2 per 2D segment) and weights normalised to sum 1 over the face."""
    nf = fnodes.shape[0]
    if dim == 2:
        a, b = nodes[fnodes[:, 0]], nodes[fnodes[:, 1]]
        h = (b - a) / (2.0 * np.sqrt(3.0))
        m = 0.5 * (a + b)
        gp = np.stack([m - h, m + h], axis=0)                      # [G][nf][d]
        gw = np.full((2, nf), 0.5)
    else:
        gp = np.zeros((4, nf, 3))
        gw = np.zeros((4, nf))
        tri = fnodes[:, 3] < 0
        a, b, c = (nodes[fnodes[tri, i]] for i in range(3))
        for k, (l0, l1, l2) in enumerate([(2 / 3, 1 / 6, 1 / 6), (1 / 6, 2 / 3, 1 / 6), (1 / 6, 1 / 6, 2 / 3)]):
            gp[k, tri] = l0 * a + l1 * b + l2 * c
            gw[k, tri] = 1.0 / 3.0
        gp[3, tri] = (a + b + c) / 3.0
        q = ~tri
        a, b, c, d = (nodes[fnodes[q, i]] for i in range(4))
        g = 1.0 / np.sqrt(3.0)
        for k, (xi, eta) in enumerate([(-g, -g), (g, -g), (g, g), (-g, g)]):
            N = [(1 - xi) * (1 - eta) / 4, (1 + xi) * (1 - eta) / 4, (1 + xi) * (1 + eta) / 4, (1 - xi) * (1 + eta) / 4]
            gp[k, q] = N[0] * a + N[1] * b + N[2] * c + N[3] * d
            dxi = (-(1 - eta) * a + (1 - eta) * b + (1 + eta) * c - (1 + eta) * d) / 4
            deta = (-(1 - xi) * a - (1 + xi) * b + (1 + xi) * c + (1 - xi) * d) / 4
            J = _cross(dxi, deta)
            gw[k, q] = np.sqrt((J * J).sum(1))
        gw[:, q] /= gw[:, q].sum(0)[None, :]
    return np.ascontiguousarray(np.transpose(gp, (2, 0, 1))), gw


def build_mesh(dim, nodes, cell_type, conn, patch_of, patch_kind, name="", meta=None) -> Mesh:
    """Build faces + geometry.

    nodes: [nn][dim]; cell_type: [n] int; conn: [n][6] node ids (padded -1),
    natural cell id = row.  patch_of(face_ctr [k][dim], avec [k][dim]) -> [k]
    patch index for boundary faces.
    """
    nodes = np.asarray(nodes, dtype=np.float64)
    cell_type = np.asarray(cell_type)
    conn = np.asarray(conn, dtype=np.int64)
    n = cell_type.shape[0]

    # ---- cell geometry -------------------------------------------------
    vol = np.zeros(n)
    ctr = np.zeros((n, dim))
    for t in np.unique(cell_type):
        idx = np.nonzero(cell_type == t)[0]
        c = conn[idx]
        if t in (TRI2, QUAD2):
            k = _NNODES[t]
            x = nodes[c[:, :k], 0]
            y = nodes[c[:, :k], 1]
            x1 = np.roll(x, -1, axis=1)
            y1 = np.roll(y, -1, axis=1)
            cr = x * y1 - x1 * y
            a2 = cr.sum(axis=1)  # 2*signed area
            cx = ((x + x1) * cr).sum(axis=1) / (3.0 * a2)
            cy = ((y + y1) * cr).sum(axis=1) / (3.0 * a2)
            vol[idx] = np.abs(a2) * 0.5
            ctr[idx] = np.stack([cx, cy], axis=1)
        elif t == TET:
            v, g = _tet_vol_ctr(*(nodes[c[:, i]] for i in range(4)))
            vol[idx], ctr[idx] = v, g
        elif t == PRISM:
            P = [nodes[c[:, i]] for i in range(6)]
            vs, gs = zip(*[_tet_vol_ctr(P[0], P[1], P[2], P[5]),
                           _tet_vol_ctr(P[0], P[1], P[5], P[4]),
                           _tet_vol_ctr(P[0], P[4], P[5], P[3])])
            V = vs[0] + vs[1] + vs[2]
            vol[idx] = V
            ctr[idx] = (vs[0][:, None] * gs[0] + vs[1][:, None] * gs[1] + vs[2][:, None] * gs[2]) / V[:, None]
        else:
            raise ValueError(t)

    # ---- face instances --------------------------------------------------
    inst_cell, inst_loc, inst_nodes = [], [], []
    for t in np.unique(cell_type):
        idx = np.nonzero(cell_type == t)[0]
        for lf, tpl in enumerate(_FACES[int(t)]):
            fn = np.full((idx.shape[0], 4), -1, dtype=np.int64)
            fn[:, :len(tpl)] = conn[idx][:, list(tpl)]
            inst_cell.append(idx)
            inst_loc.append(np.full(idx.shape[0], lf))
            inst_nodes.append(fn)
    inst_cell = np.concatenate(inst_cell)
    inst_loc = np.concatenate(inst_loc)
    inst_nodes = np.concatenate(inst_nodes)
    key = np.sort(np.where(inst_nodes < 0, np.iinfo(np.int64).max, inst_nodes), axis=1)
    # generator order: (cell, local face)
    order0 = np.lexsort((inst_loc, inst_cell))
    inst_cell, inst_loc, inst_nodes, key = inst_cell[order0], inst_loc[order0], inst_nodes[order0], key[order0]
    ordk = np.lexsort((np.arange(key.shape[0]), key[:, 3], key[:, 2], key[:, 1], key[:, 0]))
    ks = key[ordk]
    same_next = np.all(ks[1:] == ks[:-1], axis=1)
    if same_next.size and np.any(same_next[1:] & same_next[:-1]):
        raise ValueError("non-manifold face (shared by >2 cells)")
    first = np.ones(ks.shape[0], dtype=bool)
    first[1:] = ~same_next
    # partner instance for interior faces
    partner = np.full(ks.shape[0], -1, dtype=np.int64)
    pi = np.nonzero(same_next)[0]
    partner[ordk[pi]] = ordk[pi + 1]
    partner[ordk[pi + 1]] = ordk[pi]
    # each physical face is owned by its first instance in generator order
    owner_inst = np.nonzero((partner < 0) | (partner > np.arange(ks.shape[0])))[0]
    interior = partner[owner_inst] >= 0
    fi = np.concatenate([owner_inst[interior], owner_inst[~interior]])
    nf = fi.shape[0]
    left = inst_cell[fi]
    right = np.where(partner[fi] >= 0, inst_cell[np.maximum(partner[fi], 0)], -1)
    fnodes = inst_nodes[fi]

    # ---- face geometry ----------------------------------------------------
    if dim == 2:
        a = nodes[fnodes[:, 0]]
        b = nodes[fnodes[:, 1]]
        avec = np.stack([b[:, 1] - a[:, 1], -(b[:, 0] - a[:, 0])], axis=1)
        fctr = 0.5 * (a + b)
        ngauss = np.full(nf, 2, dtype=np.int8)
    else:
        avec = np.zeros((nf, 3))
        fctr = np.zeros((nf, 3))
        ngauss = np.zeros(nf, dtype=np.int8)
        tri = fnodes[:, 3] < 0
        a, b, c = (nodes[fnodes[tri, i]] for i in range(3))
        avec[tri] = 0.5 * _cross(b - a, c - a)
        fctr[tri] = (a + b + c) / 3.0
        ngauss[tri] = 3
        q = ~tri
        a, b, c, d = (nodes[fnodes[q, i]] for i in range(4))
        avec[q] = 0.5 * _cross(c - a, d - b)
        t1 = 0.5 * _cross(b - a, c - a)
        t2 = 0.5 * _cross(c - a, d - a)
        w1 = np.sqrt((t1 * t1).sum(1))[:, None]
        w2 = np.sqrt((t2 * t2).sum(1))[:, None]
        fctr[q] = (w1 * (a + b + c) / 3.0 + w2 * (a + c + d) / 3.0) / (w1 + w2)
        ngauss[q] = 4
    # orient outward from the left cell (convex cells)
    cmean = np.zeros((n, dim))
    cnt = np.zeros(n)
    for t in np.unique(cell_type):
        idx = np.nonzero(cell_type == t)[0]
        k = _NNODES[int(t)]
        cmean[idx] = nodes[conn[idx, :k]].mean(axis=1)
        cnt[idx] = k
    s = np.einsum("ij,ij->i", fctr - cmean[left], avec)
    avec[s < 0] *= -1.0

    bnd = right < 0
    if np.any(bnd):
        pidx = np.asarray(patch_of(fctr[bnd], avec[bnd]), dtype=np.int64)
        right = right.copy()
        right[bnd] = -(pidx + 1)

    gp, gw = _face_gauss(dim, nodes, fnodes)
    m = Mesh(dim=dim, vol=vol, ctr=np.ascontiguousarray(ctr.T), left=left, right=right,
             avec=np.ascontiguousarray(avec.T), fctr=np.ascontiguousarray(fctr.T), ngauss=ngauss,
             patch_kind=np.asarray(patch_kind, dtype=np.int32), name=name, meta=dict(meta or {}),
             m2=_cell_m2(dim, nodes, cell_type, conn, ctr, vol), gp=gp, gw=gw)
    m.meta.setdefault("n_nodes", int(nodes.shape[0]))
    m.meta.setdefault("cell_type_counts", {int(t): int(np.count_nonzero(cell_type == t)) for t in np.unique(cell_type)})
    return m.contiguous()


def closure_error(m: Mesh) -> float:
    """max_i |sum_f sigma_if A_f| / sum_f |A_f|  (PAPER.md:454 closure)."""
    d = m.dim
    acc = np.zeros((m.n_cells, d))
    sarea = np.zeros(m.n_cells)
    S = np.sqrt((m.avec ** 2).sum(0))
    for k in range(d):
        np.add.at(acc[:, k], m.left, m.avec[k])
        inn = m.right >= 0
        np.add.at(acc[:, k], m.right[inn], -m.avec[k][inn])
    np.add.at(sarea, m.left, S)
    np.add.at(sarea, m.right[m.right >= 0], S[m.right >= 0])
    return float(np.max(np.sqrt((acc ** 2).sum(1)) / sarea))
