"""Seeded initial states W[nv][n] (conservative, SoA, natural order).

Primitive -> conservative is the definition of the state variables
(W = (rho, rho u, rho E), E = p/((gamma-1) rho) + |u|^2/2);
no residual / sweep arithmetic lives here.
"""
from __future__ import annotations

import numpy as np

GAMMA = 1.4


def prim_to_cons(rho, u, p, gamma=GAMMA):
    rho = np.asarray(rho, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)  # [d][n]
    p = np.asarray(p, dtype=np.float64)
    d = u.shape[0]
    W = np.empty((d + 2,) + rho.shape)
    W[0] = rho
    W[1:d + 1] = rho * u
    W[d + 1] = p / (gamma - 1.0) + 0.5 * rho * (u * u).sum(0)
    return np.ascontiguousarray(W)


def winf(rho, vel, p, gamma=GAMMA):
    return prim_to_cons(np.array(rho), np.asarray(vel, dtype=np.float64), np.array(p), gamma).reshape(-1)


def uniform(mesh, rho, vel, p, gamma=GAMMA):
    n = mesh.n_cells
    vel = np.asarray(vel, dtype=np.float64)
    return prim_to_cons(np.full(n, rho), np.repeat(vel[:, None], n, 1), np.full(n, p), gamma)


def perturbed(mesh, rho, vel, p, eps=0.05, seed=0, gamma=GAMMA):
    """Free stream with seeded multiplicative noise on rho, u, p."""
    rng = np.random.default_rng(seed)
    n, d = mesh.n_cells, mesh.dim
    vel = np.asarray(vel, dtype=np.float64)
    r = rho * (1.0 + eps * rng.uniform(-1, 1, n))
    u = vel[:, None] + eps * (np.abs(vel).max() + 0.1) * rng.uniform(-1, 1, (d, n))
    pp = p * (1.0 + eps * rng.uniform(-1, 1, n))
    return prim_to_cons(r, u, pp, gamma)


def gaussian_bump(mesh, rho, vel, p, x0=(0.5, 0.5), amp=0.1, width2=0.01, jump=False, gamma=GAMMA):
    """Config 1 state: rho = 1 + 0.1 exp(-|x-x0|^2/0.01); with jump=True also a
    tanh pressure jump x10 at x = 0.5 so that DF spans (0, 1]."""
    n, d = mesh.n_cells, mesh.dim
    x = mesh.ctr
    r2 = ((x - np.asarray(x0, dtype=np.float64)[:, None]) ** 2).sum(0)
    r = rho * (1.0 + amp * np.exp(-r2 / width2))
    pp = np.full(n, p)
    if jump:
        pp = p * (1.0 + 4.5 * (1.0 - np.tanh((x[0] - 0.5) / 0.02)))
    vel = np.asarray(vel, dtype=np.float64)
    return prim_to_cons(r, np.repeat(vel[:, None], n, 1), pp, gamma)


def bow_shock(mesh, rho, vel, p, r_wall=0.5, standoff=0.25, width=0.05, gamma=GAMMA):
    """Synthetic bow-shock state for kernel benches (config 3/4): behind
    r_s(theta) = r_wall + standoff (1 + theta^2) the gas is slowed and
    compressed (normal-shock-like jump ratios), blended by tanh."""
    x = mesh.ctr
    d = mesh.dim
    r = np.sqrt((x ** 2).sum(0))
    cos_t = np.clip(-x[0] / np.maximum(r, 1e-300), -1.0, 1.0)
    theta = np.arccos(cos_t)
    rs = r_wall + standoff * (1.0 + theta ** 2)
    s = 0.5 * (1.0 - np.tanh((r - rs) / width))  # 1 inside the shock layer
    vel = np.asarray(vel, dtype=np.float64)
    rho2, p2, uf = 5.5 * rho, 60.0 * p, 0.18
    rr = rho + (rho2 - rho) * s
    pp = p + (p2 - p) * s
    u = vel[:, None] * (1.0 - (1.0 - uf) * s)[None, :]
    return prim_to_cons(rr, u, pp, gamma)
