"""Bench-pattern inputs of tools/order_sim.cpp: bench.py's coords in their factor order and the m
nearest PRECEDING neighbours of every point (own kd-tree search; distance ties are not
resolved as the reference does, which the traffic model does not need)."""
import os

import numpy as np
from scipy.spatial import cKDTree

n, m, seed = 1_000_000, 20, 2310
os.makedirs("/tmp/sim", exist_ok=True)
coords = np.random.default_rng(seed).uniform(size=(n, 2))
xy = np.ascontiguousarray(coords[np.random.default_rng(seed + 3).permutation(n)])
nbr = np.full((n, m), -1, dtype=np.int32)
tree = cKDTree(xy)
todo = np.arange(1, n)
k = 2 * m + 16
while todo.size:
    k = min(k, n)
    _, ii = tree.query(xy[todo], k=k, workers=-1)
    left = []
    for r, i in enumerate(todo):
        c = ii[r][ii[r] < i]
        if c.size >= min(m, i) or k >= n:
            nbr[i, : min(m, c.size)] = c[:m]
        else:
            left.append(i)
    todo = np.array(left, dtype=np.int64)
    k *= 4
xy.tofile("/tmp/sim/xy.bin")
nbr.tofile("/tmp/sim/nbr.bin")
