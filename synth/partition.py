"""Seeded-input helper: recursive coordinate bisection of cell centroids.

Numpy restatement of the rule libgmg's gmg_partition_rcb uses (split the
longest extent; the first np_left/np cells in (coordinate, natural id) order go
left), so the oracle-side reference arm can build the same partitioned
workload without calling the product library.  Not method arithmetic: the
partition is an input (part[] of gmg_load_mesh).
"""
from __future__ import annotations

import numpy as np


def rcb(ctr, nparts):
    ctr = np.asarray(ctr, dtype=np.float64)
    dim, n = ctr.shape
    part = np.zeros(n, dtype=np.int32)
    stack = [(np.arange(n), 0, nparts)]
    while stack:
        ids, p0, np_ = stack.pop()
        if np_ <= 1 or ids.size <= 1:
            part[ids] = p0
            continue
        ext = [ctr[k, ids].max() - ctr[k, ids].min() for k in range(dim)]
        axis = int(np.argmax(ext))          # first axis of maximal extent
        nl = np_ // 2
        m = ids.size * nl // np_
        order = np.lexsort((ids, ctr[axis, ids]))
        s = ids[order]
        stack.append((s[m:], p0 + nl, np_ - nl))
        stack.append((s[:m], p0, nl))
    return part
