"""Kernel microbench: B / B^T products and triangular solves at n x t, GB/s
against the SURVEY 8(d) algorithmic byte count 12*nnz + 4*(n+1) + 16*n*t."""
import argparse
import json
import time

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2310_12000_b200 as vg
from paper_2310_12000_b200 import _lib
from paper_2310_12000_b200.vecchia import Pattern, build_factor, neighbor_array


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--m", type=int, default=20)
    ap.add_argument("--ts", default="1,16,50,64")
    ap.add_argument("--orders", default="1")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    xy = rng.uniform(size=(a.n, 2))
    perm = np.random.default_rng(1).permutation(a.n)
    t0 = time.time()
    nbr = neighbor_array(xy, perm, a.m)
    print(f"knn {time.time() - t0:.2f}s", flush=True)
    xyp = np.ascontiguousarray(xy[perm])
    peak = 6552.0
    for ok in [int(o) for o in a.orders.split(",")]:
        t0 = time.time()
        pat = Pattern(xyp, nbr, ok)
        print(f"pattern order={ok} {time.time() - t0:.2f}s levels fwd={pat.n_levels} bwd={pat.n_levels_T} "
              f"maxchildren={pat.max_children}", flush=True)
        spec = vg.CovarianceSpec(1.0, 0.02, 1.5)
        f = build_factor(xyp, spec, pat, want_grad=True)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(2):
            f2 = build_factor(xyp, spec, pat, want_grad=True)
        ev0.record()
        for _ in range(3):
            f2 = build_factor(xyp, spec, pat, want_grad=True)
        ev1.record(); torch.cuda.synchronize()
        print(f"factor_build+grad {ev0.elapsed_time(ev1)/3:.3f} ms", flush=True)
        nnz = pat.nnz_off + a.n
        for t in [int(x) for x in a.ts.split(",")]:
            X = torch.randn(a.n, t, dtype=torch.float64, device="cuda") / 20
            Y = torch.empty_like(X)
            res = {}
            for name, fn, args in [("B", "vl_spmm", (0,)), ("Bt", "vl_spmm", (1,)),
                                   ("Binv", "vl_sptrsv", (0,)), ("Btinv", "vl_sptrsv", (1,))]:
                def run():
                    _lib.call(fn, f.ctx.h, f.h, *args, t, _lib.ptr(X), _lib.ptr(Y))
                for _ in range(3):
                    run()
                torch.cuda.synchronize()
                ev0.record()
                for _ in range(a.reps):
                    run()
                ev1.record(); torch.cuda.synchronize()
                ms = ev0.elapsed_time(ev1) / a.reps
                by = 12 * nnz + 4 * (a.n + 1) + 16 * a.n * t
                res[name] = {"ms": round(ms, 4), "GBps": round(by / ms / 1e6, 1), "frac": round(by / ms / 1e6 / peak, 3)}
            print(json.dumps({"order": ok, "t": t, **res}), flush=True)


if __name__ == "__main__":
    main()
