"""Seeded synthetic meshes shaped like BASELINE.json's configs.

config 1  2D 32x32 unit square, each square split by a seeded random diagonal
config 2  2D NACA0012 O-grid, 256 around x (48 quad + 16 triangulated) layers
config 3  2D cylinder O-grid, 512 x 196 quads
config 4  3D sphere shell: cubed sphere 6 x 40^2 columns, 16 prism + 12 tet layers
config 5  config 4 with n = round(40 sqrt(P)) columns per cube-face edge

plus tiny meshes for brute-force pins.  Geometry only; no method arithmetic.
"""
from __future__ import annotations

import math

import numpy as np

from .mesh import (EXTRAP, FARFIELD, NOSLIP, PRISM, QUAD2, SLIP, TET, TRI2,
                   build_mesh)


# ---------------------------------------------------------------------------
# 2D
# ---------------------------------------------------------------------------
def _grid_nodes(nx, ny, x0=0.0, x1=1.0, y0=0.0, y1=1.0):
    xs = np.linspace(x0, x1, nx + 1)
    ys = np.linspace(y0, y1, ny + 1)
    X, Y = np.meshgrid(xs, ys, indexing="xy")  # [ny+1][nx+1]
    return np.stack([X.ravel(), Y.ravel()], axis=1)


def quad_grid(nx=4, ny=4, patch_kinds=(FARFIELD,)):
    """Structured nx x ny unit-square quad grid (cells row-major)."""
    nodes = _grid_nodes(nx, ny)
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    i, j = i.ravel(), j.ravel()
    n0 = j * (nx + 1) + i
    conn = np.full((nx * ny, 6), -1, dtype=np.int64)
    conn[:, :4] = np.stack([n0, n0 + 1, n0 + nx + 2, n0 + nx + 1], axis=1)
    ctype = np.full(nx * ny, QUAD2)
    pk = list(patch_kinds)

    def patch_of(fc, av):
        if len(pk) == 1:
            return np.zeros(fc.shape[0], dtype=np.int64)
        # 4 sides: x=0, x=1, y=0, y=1 -> patch 0..3 (mod len)
        side = np.where(np.abs(av[:, 0]) > np.abs(av[:, 1]), np.where(fc[:, 0] < 0.5, 0, 1),
                        np.where(fc[:, 1] < 0.5, 2, 3))
        return side % len(pk)

    return build_mesh(2, nodes, ctype, conn, patch_of, pk, name=f"quad{nx}x{ny}")


def tri_square(nx=32, ny=32, seed=1, uniform=False, patch_kinds=(FARFIELD,)):
    """Config 1: unit square, nx*ny squares each split by a diagonal.

    uniform=True uses the same diagonal everywhere (honeycomb dual -> 2
    colors, the P:429-432 structured pin); otherwise the diagonal of each
    square is drawn from a seeded RNG.
    """
    rng = np.random.default_rng(seed)
    nodes = _grid_nodes(nx, ny)
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    i, j = i.ravel(), j.ravel()
    a = j * (nx + 1) + i
    b, c, d = a + 1, a + nx + 2, a + nx + 1
    flip = np.zeros(nx * ny, dtype=bool) if uniform else rng.integers(0, 2, nx * ny).astype(bool)
    t1 = np.where(flip[:, None], np.stack([a, b, d], 1), np.stack([a, b, c], 1))
    t2 = np.where(flip[:, None], np.stack([b, c, d], 1), np.stack([a, c, d], 1))
    tris = np.stack([t1, t2], axis=1).reshape(-1, 3)
    conn = np.full((tris.shape[0], 6), -1, dtype=np.int64)
    conn[:, :3] = tris
    ctype = np.full(tris.shape[0], TRI2)
    pk = list(patch_kinds)

    def patch_of(fc, av):
        if len(pk) == 1:
            return np.zeros(fc.shape[0], dtype=np.int64)
        side = np.where(np.abs(av[:, 0]) > np.abs(av[:, 1]), np.where(fc[:, 0] < 0.5, 0, 1),
                        np.where(fc[:, 1] < 0.5, 2, 3))
        return side % len(pk)

    return build_mesh(2, nodes, ctype, conn, patch_of, pk,
                      name=f"trisq{nx}x{ny}{'u' if uniform else ''}s{seed}")


def _ogrid(surface, outer, n_layers, first_frac, n_tri_layers, seed):
    """O-grid between a closed surface polyline and an outer polyline (same
    count, same orientation); geometric radial spacing; the outermost
    n_tri_layers quad layers are split by seeded random diagonals."""
    ni = surface.shape[0]
    L = n_layers + n_tri_layers
    # geometric growth so that sum of L spacings = 1 with the first = first_frac
    lo, hi = 1.0 + 1e-12, 3.0
    for _ in range(200):
        q = 0.5 * (lo + hi)
        tot = first_frac * (q ** L - 1.0) / (q - 1.0)
        lo, hi = (q, hi) if tot < 1.0 else (lo, q)
    q = 0.5 * (lo + hi)
    s = np.concatenate([[0.0], np.cumsum(first_frac * q ** np.arange(L))])
    s /= s[-1]
    P = surface[None, :, :] + (outer - surface)[None, :, :] * s[:, None, None]  # [L+1][ni][2]
    nodes = P.reshape(-1, 2)
    rng = np.random.default_rng(seed)
    conn, ctype = [], []
    for k in range(L):
        for i in range(ni):
            i1 = (i + 1) % ni
            a, b = k * ni + i, k * ni + i1
            c, d = (k + 1) * ni + i1, (k + 1) * ni + i
            if k < n_layers:
                conn.append([a, b, c, d, -1, -1])
                ctype.append(QUAD2)
            else:
                if rng.integers(0, 2):
                    conn += [[a, b, c, -1, -1, -1], [a, c, d, -1, -1, -1]]
                else:
                    conn += [[a, b, d, -1, -1, -1], [b, c, d, -1, -1, -1]]
                ctype += [TRI2, TRI2]
    return nodes, np.array(ctype), np.array(conn, dtype=np.int64)


def naca_ogrid(ni=256, n_quad=48, n_tri=16, r_out=20.0, first=1e-4, seed=0):
    """Config 2: NACA0012 (closed TE) O-grid, wall NOSLIP, farfield R=20c."""
    th = 2.0 * np.pi * np.arange(ni) / ni
    x = 0.5 * (1.0 + np.cos(th))
    yt = 0.6 * (0.2969 * np.sqrt(x) - 0.1260 * x - 0.3516 * x ** 2 + 0.2843 * x ** 3 - 0.1036 * x ** 4)
    y = np.where(th <= np.pi, yt, -yt)
    surf = np.stack([x, y], 1)
    outer = np.stack([0.5 + r_out * np.cos(th), r_out * np.sin(th)], 1)
    dist = float(np.mean(np.linalg.norm(outer - surf, axis=1)))
    nodes, ctype, conn = _ogrid(surf, outer, n_quad, first / dist, n_tri, seed)
    pk = [NOSLIP, FARFIELD]

    def patch_of(fc, av):
        return np.where(np.linalg.norm(fc - np.array([0.5, 0.0]), axis=1) < 2.0, 0, 1)

    return build_mesh(2, nodes, ctype, conn, patch_of, pk, name=f"naca{ni}x{n_quad}+{n_tri}")


def cylinder_ogrid(ni=512, nr=196, r_in=0.5, r_out=6.0, first=2e-3, n_tri=0, seed=0):
    """Config 3: full-cylinder O-grid. wall SLIP, upstream (x<0) FARFIELD,
    downstream EXTRAP."""
    th = 2.0 * np.pi * np.arange(ni) / ni
    surf = r_in * np.stack([np.cos(th), np.sin(th)], 1)
    outer = r_out * np.stack([np.cos(th), np.sin(th)], 1)
    nodes, ctype, conn = _ogrid(surf, outer, nr - n_tri, first / (r_out - r_in), n_tri, seed)
    pk = [SLIP, FARFIELD, EXTRAP]

    def patch_of(fc, av):
        r = np.linalg.norm(fc, axis=1)
        return np.where(r < 0.5 * (r_in + r_out), 0, np.where(fc[:, 0] < 0.0, 1, 2))

    return build_mesh(2, nodes, ctype, conn, patch_of, pk, name=f"cyl{ni}x{nr}")


# ---------------------------------------------------------------------------
# 3D
# ---------------------------------------------------------------------------
def _prism_to_tets(pc, gid):
    """Split prisms [k][6] (bottom a,b,c; top d,e,f above them) into 3 tets
    each with the min-global-id rule (Dompierre et al.), conforming for any
    global numbering gid."""
    k = pc.shape[0]
    g = gid[pc]
    m = np.argmin(g, axis=1)
    r = m % 3
    top = m >= 3
    perm = np.zeros((k, 6), dtype=np.int64)
    for rr in range(3):
        bot = [rr, (rr + 1) % 3, (rr + 2) % 3]
        sel = (r == rr) & ~top
        perm[sel] = bot + [x + 3 for x in bot]
        sel = (r == rr) & top
        perm[sel] = [x + 3 for x in bot] + bot
    V = np.take_along_axis(pc, perm, axis=1)
    G = gid[V]
    case1 = np.minimum(G[:, 1], G[:, 5]) < np.minimum(G[:, 2], G[:, 4])
    t1 = np.where(case1[:, None], V[:, [0, 1, 2, 5]], V[:, [0, 1, 2, 4]])
    t2 = np.where(case1[:, None], V[:, [0, 1, 5, 4]], V[:, [0, 4, 2, 5]])
    t3 = V[:, [0, 4, 5, 3]]
    return np.stack([t1, t2, t3], axis=1).reshape(-1, 4)


def _hex_columns_to_cells(qcols, parity, nsurf, n_prism, n_tet, gid):
    """qcols [nc][4] surface-node quads (cyclic), parity [nc]; radial layer k
    node = k*nsurf + surface node.  Returns ctype, conn in natural order
    (column-major: column, layer, sub-cell)."""
    nc = qcols.shape[0]
    q0, q1, q2, q3 = (qcols[:, i] for i in range(4))
    tA = np.where(parity[:, None] == 0, np.stack([q0, q1, q2], 1), np.stack([q0, q1, q3], 1))
    tB = np.where(parity[:, None] == 0, np.stack([q0, q2, q3], 1), np.stack([q1, q2, q3], 1))
    L = n_prism + n_tet
    per_col = 2 * n_prism + 6 * n_tet
    conn = np.full((nc, per_col, 6), -1, dtype=np.int64)
    ctype = np.zeros((nc, per_col), dtype=np.int64)
    pos = 0
    for k in range(L):
        for tri in (tA, tB):
            prism = np.concatenate([tri + k * nsurf, tri + (k + 1) * nsurf], axis=1)
            if k < n_prism:
                conn[:, pos, :] = prism
                ctype[:, pos] = PRISM
                pos += 1
            else:
                tets = _prism_to_tets(prism, gid).reshape(nc, 3, 4)
                conn[:, pos:pos + 3, :4] = tets
                ctype[:, pos:pos + 3] = TET
                pos += 3
    return ctype.reshape(-1), conn.reshape(-1, 6)


def sphere_shell(n=40, n_prism=16, n_tet=12, r_in=0.5, r_out=5.0, beta=3.0, seed=0):
    """Config 4 (n=40, ~998k cells) / config 5 (n = round(40 sqrt(P))).

    Cubed-sphere surface (equiangular, 6 n^2 columns), radial layers
    geometrically clustered at the wall; hex -> 2 prisms (diagonal by column
    parity), outer layers prism -> 3 tets by the min-global-node rule over a
    seeded random node numbering (conforming, irregular).  Patches: wall SLIP,
    upstream (x<0) FARFIELD, downstream EXTRAP."""
    t = np.linspace(-np.pi / 4, np.pi / 4, n + 1)
    A, B = np.meshgrid(np.tan(t), np.tan(t), indexing="ij")  # [i][j]
    one = np.ones_like(A)
    faces = [(one, A, B), (-one, B, A), (A, one, B), (B, -one, A), (A, B, one), (B, A, -one)]
    pts, quads, par = [], [], []
    off = 0
    for (X, Y, Z) in faces:
        P = np.stack([X, Y, Z], -1).reshape(-1, 3)
        P /= np.linalg.norm(P, axis=1, keepdims=True)
        pts.append(P)
        ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        ii, jj = ii.ravel(), jj.ravel()
        base = off + ii * (n + 1) + jj
        quads.append(np.stack([base, base + (n + 1), base + (n + 1) + 1, base + 1], 1))
        par.append((ii + jj) % 2)
        off += (n + 1) ** 2
    pts = np.concatenate(pts)
    quads = np.concatenate(quads)
    par = np.concatenate(par)
    # deduplicate shared cube edges / corners
    key = np.round(pts * 1e9).astype(np.int64)
    _, uid, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
    inv = inv.ravel()
    surf = pts[uid]
    quads = inv[quads]
    nsurf = surf.shape[0]
    L = n_prism + n_tet
    s = (np.exp(beta * np.arange(L + 1) / L) - 1.0) / (np.exp(beta) - 1.0)
    r = r_in + (r_out - r_in) * s
    nodes = (r[:, None, None] * surf[None, :, :]).reshape(-1, 3)
    rng = np.random.default_rng(seed)
    gid = rng.permutation(nodes.shape[0])
    ctype, conn = _hex_columns_to_cells(quads, par, nsurf, n_prism, n_tet, gid)
    pk = [SLIP, FARFIELD, EXTRAP]

    def patch_of(fc, av):
        rr = np.linalg.norm(fc, axis=1)
        return np.where(rr < 0.5 * (r_in + r_out), 0, np.where(fc[:, 0] < 0.0, 1, 2))

    return build_mesh(3, nodes, ctype, conn, patch_of, pk, name=f"sphere{n}_{n_prism}p{n_tet}t",
                      meta={"r_in": r_in, "r_out": r_out})


def box3d(nx=3, ny=3, nz=3, n_prism_layers=0, seed=0, patch_kinds=(FARFIELD, SLIP, NOSLIP, EXTRAP)):
    """Small 3D unit box: each hex -> 2 prisms (column parity); layers z <
    n_prism_layers stay prisms, the rest -> 3 tets each (random numbering).
    Patches: x=0 / x=1 / y sides / z sides -> patch_kinds cycled."""
    xs, ys, zs = (np.linspace(0, 1, k + 1) for k in (nx, ny, nz))
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    nodes = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
    nsl = (nx + 1) * (ny + 1)
    jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    ii, jj = ii.ravel(), jj.ravel()
    base = jj * (nx + 1) + ii
    quads = np.stack([base, base + 1, base + nx + 2, base + nx + 1], 1)
    par = (ii + jj) % 2
    rng = np.random.default_rng(seed)
    gid = rng.permutation(nodes.shape[0])
    ctype, conn = _hex_columns_to_cells(quads, par, nsl, n_prism_layers, nz - n_prism_layers, gid)
    pk = list(patch_kinds)

    def patch_of(fc, av):
        ax = np.argmax(np.abs(av), axis=1)
        side = np.where(ax == 0, np.where(fc[:, 0] < 0.5, 0, 1), np.where(ax == 1, 2, 3))
        return side % len(pk)

    return build_mesh(3, nodes, ctype, conn, patch_of, pk, name=f"box{nx}x{ny}x{nz}p{n_prism_layers}s{seed}")


def single_cell(dim=2):
    if dim == 2:
        return quad_grid(1, 1)
    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=np.float64)
    conn = np.array([[0, 1, 2, 3, -1, -1]])
    return build_mesh(3, nodes, np.array([TET]), conn, lambda fc, av: np.zeros(fc.shape[0], dtype=np.int64),
                      [FARFIELD], name="tet1")


def two_cells():
    """Two unit squares sharing a face."""
    return quad_grid(2, 1)


def config(k: int, P: int = 1):
    """The BASELINE.json configs by 1-based index."""
    if k == 1:
        return tri_square(32, 32, seed=1)
    if k == 2:
        return naca_ogrid()
    if k == 3:
        return cylinder_ogrid()
    if k == 4:
        return sphere_shell(40)
    if k == 5:
        return sphere_shell(int(round(40 * math.sqrt(P))))
    raise ValueError(k)


# free-stream / farfield states per config: (rho, velocity, p) with a_inf = 1
FREESTREAM = {
    1: (1.0, (0.5, 0.0), 1.0 / 1.4),
    2: (1.0, (0.5, 0.0), 1.0 / 1.4),
    3: (1.0, (8.0, 0.0), 1.0 / 1.4),
    4: (1.0, (8.0, 0.0, 0.0), 1.0 / 1.4),
    5: (1.0, (8.0, 0.0, 0.0), 1.0 / 1.4),
}
