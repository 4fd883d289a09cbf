"""BASELINE config 5 kernel sweep: random unit-lower-triangular B (row i takes
min(i, m) distinct parents uniform on [0, i)), off-diagonals N(0,1)/m (SURVEY
D10: keeps the solves bounded), D ~ U(0.5, 1.5); fp64 B X, B^T X, B^-1 X,
B^-T X for t in {1, 16, 64}.  GB/s against the SURVEY 8(d) algorithmic byte
count 12*nnz + 4*(n+1) + 16*n*t, fraction of the measured HBM copy peak.

Also runs the same four ops on the kNN factor of the headline workload
(--knn) for comparison.  Prints one JSON line per (pattern, n, m, t).

Each cell is checked once against scipy on a 4-column slice (products and
solves, max relative error) so a fast-but-wrong kernel cannot enter the table.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2310_12000_b200 as vg  # noqa: E402
from paper_2310_12000_b200 import _lib  # noqa: E402
from paper_2310_12000_b200.vecchia import Pattern, build_factor, neighbor_array  # noqa: E402


def random_parents(n, m, rng):
    """Row i: min(i, m) distinct parents uniform on [0, i) (BASELINE config 5)."""
    nbr = np.full((n, m), -1, dtype=np.int64)
    i = np.arange(n)
    for k in range(m):
        nbr[:, k] = np.floor(rng.random(n) * i).astype(np.int64)
    nbr[i[:, None] <= np.arange(m)[None, :]] = -1
    # resample duplicates within a row until all parents are distinct
    for _ in range(64):
        s = np.sort(nbr, axis=1)
        dup_rows = np.nonzero(((s[:, 1:] == s[:, :-1]) & (s[:, 1:] >= 0)).any(axis=1))[0]
        if dup_rows.size == 0:
            break
        for r in dup_rows:
            k = min(r, m)
            nbr[r, :k] = rng.choice(r, size=k, replace=False)
    return nbr.astype(np.int32)


def csr_of(nbr, vals, n):
    """B in factor order: unit diagonal plus the ELL off-diagonal entries."""
    mask = nbr >= 0
    rows = np.repeat(np.arange(n), mask.sum(axis=1))
    cols = nbr[mask].astype(np.int64)
    data = vals[mask]
    L = sp.csr_matrix((data, (rows, cols)), shape=(n, n))
    return (L + sp.identity(n, format="csr")).tocsr()


def time_op(fn, reps):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(reps):
        fn()
    ev1.record()
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="1000000,3000000,10000000")
    ap.add_argument("--ms", default="10,20,30")
    ap.add_argument("--ts", default="1,16,64")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--knn", action="store_true", help="also the kNN factor of the headline workload")
    ap.add_argument("--check", type=int, default=1, help="scipy check on a 4-column slice (n <= 3e6)")
    ap.add_argument("--kinds", default=None, help="comma list of patterns (random, knn); default random[,knn]")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    peak = 6552.0
    try:
        peak = float(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    out = open(a.out, "w") if a.out else None
    cells = []
    for n in [int(float(x)) for x in a.ns.split(",")]:
        for m in [int(x) for x in a.ms.split(",")]:
            kinds = a.kinds.split(",") if a.kinds else ["random"] + (["knn"] if a.knn else [])
            for kind in kinds:
                rng = np.random.default_rng(5 + n + m)
                xy = rng.uniform(size=(n, 2))
                t0 = time.time()
                if kind == "random":
                    nbr = random_parents(n, m, rng)
                    order_kind = 0
                else:
                    perm = np.random.default_rng(1).permutation(n)
                    nbr = neighbor_array(xy, perm, m)
                    xy = np.ascontiguousarray(xy[perm])
                    order_kind = 1
                tg = time.time() - t0
                t0 = time.time()
                pat = Pattern(xy, nbr, order_kind)
                tp = time.time() - t0
                f = build_factor(xy, vg.CovarianceSpec(1.0, 0.02, 1.5), pat, want_grad=False)
                if kind == "random":
                    vals = rng.standard_normal((n, m)) / m
                    vals[nbr < 0] = 0.0
                    D = rng.uniform(0.5, 1.5, size=n)
                    _lib.call("vl_factor_set", f.ctx.h, f.h, 3, _lib.ptr(np.ascontiguousarray(vals[pat.sperm])))
                    _lib.call("vl_factor_set", f.ctx.h, f.h, 0, _lib.ptr(np.ascontiguousarray(D[pat.sperm])))
                nnz = pat.nnz_off + n
                meta = {"pattern": kind, "n": n, "m": m, "nnz": nnz, "levels_fwd": pat.n_levels,
                        "levels_bwd": pat.n_levels_T, "max_children": pat.max_children,
                        "gen_s": round(tg, 2), "pattern_s": round(tp, 2)}
                print(json.dumps({"setup": meta}), flush=True)
                Bcsr = None
                if a.check and n <= 3_000_000:
                    vv = np.zeros((n, m))
                    _lib.call("vl_factor_get", f.ctx.h, f.h, 3, _lib.ptr(vv))
                    vv = vv[pat.siperm]
                    Bcsr = csr_of(nbr, vv, n)
                for t in [int(x) for x in a.ts.split(",")]:
                    X = torch.randn(n, t, dtype=torch.float64, device="cuda")
                    Y = torch.empty_like(X)
                    res = {}
                    for name, fn, arg in [("B", "vl_spmm", 0), ("Bt", "vl_spmm", 1),
                                          ("Binv", "vl_sptrsv", 0), ("Btinv", "vl_sptrsv", 1)]:
                        def run():
                            _lib.call(fn, f.ctx.h, f.h, arg, t, _lib.ptr(X), _lib.ptr(Y))
                        ms = time_op(run, a.reps)
                        by = 12 * nnz + 4 * (n + 1) + 16 * n * t
                        cell = {"ms": round(ms, 4), "GBps": round(by / ms / 1e6, 1),
                                "frac": round(by / ms / 1e6 / peak, 3)}
                        if Bcsr is not None:
                            run()
                            torch.cuda.synchronize()
                            k = min(t, 4)
                            xs = X[:, :k].cpu().numpy()[pat.siperm]
                            ys = Y[:, :k].cpu().numpy()[pat.siperm]
                            if name == "B":
                                ref = Bcsr @ xs
                            elif name == "Bt":
                                ref = Bcsr.T @ xs
                            elif name == "Binv":
                                ref = spla.spsolve_triangular(Bcsr, xs, lower=True, unit_diagonal=True)
                            else:
                                ref = spla.spsolve_triangular(Bcsr.T.tocsr(), xs, lower=False, unit_diagonal=True)
                            cell["relerr"] = float(np.abs(ys - ref).max() / max(np.abs(ref).max(), 1e-300))
                        res[name] = cell
                    line = {**meta, "t": t, "bytes_formula": "12*nnz + 4*(n+1) + 16*n*t (nnz incl. diagonal)", "peak_GBps": peak,
                            **res}
                    cells.append(line)
                    print(json.dumps(line), flush=True)
                    if out:
                        out.write(json.dumps(line) + "\n")
                        out.flush()
                    del X, Y
                del f, pat
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
