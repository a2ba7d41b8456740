"""Pure-Python brute-force checkers for tiny meshes (<= ~64 cells).

Independent of both the C oracle and the CUDA path: written from the paper's
algorithms directly, used only to pin the oracle (SURVEY.md §8(c) pins).
"""
from __future__ import annotations

import math


def adjacency(n, left, right):
    nb = [[] for _ in range(n)]
    for l, r in zip(left.tolist(), right.tolist()):
        if r >= 0:
            nb[l].append(r)
            nb[r].append(l)
    return [sorted(x) for x in nb]


def color_alg1(n, left, right):
    """Algorithm 1: BFS waves from cell 0 in ascending id; each
    newly reached cell takes the least positive color unused by its colored
    neighbours; restart from the least uncolored id if disconnected."""
    nb = adjacency(n, left, right)
    col = [0] * n
    for start in range(n):
        if col[start]:
            continue
        col[start] = 1
        q = [start]
        while q:
            v = q.pop(0)
            for w in nb[v]:
                if col[w] == 0:
                    used = {col[j] for j in nb[w]}
                    k = 1
                    while k in used:
                        k += 1
                    col[w] = k
                    q.append(w)
    return col


def greedy_sequential_gs(cells_in_order, update):
    """Sequential Gauss-Seidel: update(i) for each i in the given order."""
    for i in cells_in_order:
        update(i)


def euler_T(dim, gamma, W, n):
    rho = W[0]
    U = sum(W[1 + k] / rho * n[k] for k in range(dim))
    m2 = sum(W[1 + k] * W[1 + k] for k in range(dim))
    p = (gamma - 1.0) * (W[dim + 1] - 0.5 * m2 / rho)
    return [rho * U] + [W[1 + k] * U + p * n[k] for k in range(dim)] + [(W[dim + 1] + p) * U]


def norm(v):
    return math.sqrt(sum(x * x for x in v))
