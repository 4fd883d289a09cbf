"""Parent-row reuse of the level-scheduled multi-column solves (CPU only).

For the bench pattern (n uniform points, random order, m nearest previous
neighbours) prints, for the non-head levels, the number of DISTINCT parent
rows a sweep over K consecutive levels gathers, relative to its total number
of gathers: the best DRAM-traffic ratio any schedule that keeps K levels of
gathers L2-resident could reach, and the level distance of the parents.
Used by DESIGN.md (t = 50 solve traffic)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import vl_oracle as O  # noqa: E402  (kNN only: analysis tool, not the product path)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--m", type=int, default=20)
    ap.add_argument("--head-levels", type=int, default=160)
    a = ap.parse_args()
    xy = np.random.default_rng(0).uniform(size=(a.n, 2))
    perm = np.random.default_rng(1).permutation(a.n)
    nbr = np.asarray(O.knn_previous(np.ascontiguousarray(xy[perm]), a.m, workers=-1))
    lev = np.zeros(a.n, dtype=np.int64)
    for i in range(a.n):
        row = nbr[i]
        row = row[row >= 0]
        if row.size:
            lev[i] = lev[row].max() + 1
    cnt = np.bincount(lev)
    print("levels", len(cnt), "rows per level (every 20th):", cnt[::20].tolist())
    order = np.argsort(lev, kind="stable")
    ptr = np.concatenate([[0], np.cumsum(cnt)])
    for K in (1, 2, 4, 8, 16):
        tot = uniq = 0
        for L in range(a.head_levels, len(cnt), K):
            rows = order[ptr[L]:ptr[min(L + K, len(cnt))]]
            nb = nbr[rows].ravel()
            nb = nb[nb >= 0]
            tot += nb.size
            uniq += np.unique(nb).size
        print(f"K={K:2d} levels per sweep: distinct parents / gathers = {uniq / tot:.3f}")
    ld = (lev[:, None] - lev[np.maximum(nbr, 0)])[nbr >= 0]
    print("parent level distance percentiles 10/25/50/75/90:", np.percentile(ld, [10, 25, 50, 75, 90]).tolist())


if __name__ == "__main__":
    main()
