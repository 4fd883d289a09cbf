"""BASELINE config 2: n = 1e5, rho = 0.05, m = 20, t = 50, Bernoulli-logit,
VADU vs LRAC (pivoted-Cholesky rank k = 1000, eq7 split): full Newton mode
finding + NLL + gradient on one GPU (s/eval, CG counts).

--oracle also runs the CPU restatement of the reference (oracle/, the
tests' checker) on the same inputs -- same ordering, neighbours, probes --
and reports its wall time and the GPU-vs-oracle relative differences of the
NLL and the gradient at full config-2 size.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (synthetic data generator shared with the headline bench)
import paper_2310_12000_b200 as vg  # noqa: E402
from paper_2310_12000_b200.estimate import FitConfig, _Objective  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--rho", type=float, default=0.05)
    ap.add_argument("--t", type=int, default=50)
    ap.add_argument("--rank", type=int, default=1000)
    ap.add_argument("--seed", type=int, default=2310)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--precs", default="vadu,lrac")
    ap.add_argument("--oracle", default="", help="comma list of preconditioners to also run on the CPU oracle")
    ap.add_argument("--newton-grad-tol", type=float, default=1e-6,
                    help="BackendConfig.newton_grad_tol (DESIGN 6: the fp64 noise floor of |d1 - Q b|)")
    ap.add_argument("--prof", action="store_true", help="per-tag kernel times of the timed evaluations")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    ns = argparse.Namespace(n=a.n, seed=a.seed)
    coords, _ = bench.synth(ns)
    b_true = bench.latent_field(coords, a.rho, a.seed)
    y = (np.random.default_rng(a.seed + 4).uniform(size=a.n) < 1.0 / (1.0 + np.exp(-b_true))).astype(float)
    X = np.zeros((a.n, 0))
    theta = np.array([1.0, a.rho])
    lines = []
    for prec in a.precs.split(","):
        backend = vg.BackendConfig(preconditioner=prec, t=a.t, cg_tol=1e-3, probe_seed=a.seed + 5,
                                   rank=a.rank if prec == "lrac" else None, newton_grad_tol=a.newton_grad_tol)
        cfg = FitConfig(m=20, ordering_seed=a.seed + 3, nu=1.5, backend=backend)
        obj = _Objective(y, X, coords, vg.get_likelihood("bernoulli-logit"), cfg)
        val, grad = obj.evaluate(theta, np.zeros(0), np.zeros(0), want_grad=True)  # warm-up
        torch.cuda.synchronize()
        from paper_2310_12000_b200 import _lib
        L = _lib.lib()
        if a.prof:
            L.vl_prof_enable.argtypes = [_lib.c_void_p, _lib.c_int]
            L.vl_prof_reset.argtypes = [_lib.c_void_p]
            L.vl_prof_report.argtypes = [_lib.c_void_p, _lib.C.c_char_p, _lib.c_int, _lib.P_int64]
            _lib.check(L.vl_prof_reset(obj.pattern.ctx.h))
            _lib.check(L.vl_prof_enable(obj.pattern.ctx.h, 1))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            val, grad = obj.evaluate(theta, np.zeros(0), np.zeros(0), want_grad=True)
        e1.record()
        torch.cuda.synchronize()
        s_eval = e0.elapsed_time(e1) / 1e3 / a.steps
        tags = None
        if a.prof:
            buf = _lib.C.create_string_buffer(1 << 16)
            nl = _lib.C.c_int64(0)
            _lib.check(L.vl_prof_report(obj.pattern.ctx.h, buf, 1 << 16, _lib.C.byref(nl)))
            _lib.check(L.vl_prof_enable(obj.pattern.ctx.h, 0))
            tags = {}
            for ln in buf.value.decode().splitlines():
                tg, cnt, tms, _ = ln.split("\t")
                tags[tg] = {"launches": int(cnt) // a.steps, "ms_per_eval": round(float(tms) / a.steps, 3)}
        fct, st, pr = obj.last
        line = {"config": "C2", "newton_grad_tol": a.newton_grad_tol, "n": a.n, "m": 20, "t": a.t, "rho": a.rho, "preconditioner": prec,
                "rank": a.rank if prec == "lrac" else None, "s_per_eval": s_eval, "evals_per_s": 1.0 / s_eval,
                "nll": float(val), "grad_log_theta": [float(g) for g in grad],
                "newton_steps": int(st.newton_iters), "newton_cg": [int(c) for c in st.cg_iters],
                "probe_cg_mean": float(np.mean(pr.iters)) if pr.iters is not None else None}
        if tags is not None:
            line["kernels"] = tags
        if prec in a.oracle.split(","):
            from oracle import vl_oracle as O
            ocfg = O.Cfg(preconditioner=prec, t=a.t, cg_tol=1e-3, probe_seed=a.seed + 5,
                         rank=a.rank if prec == "lrac" else None, newton_grad_tol=a.newton_grad_tol)
            t0 = time.perf_counter()
            oval, og, oinfo = O.evaluate(obj.xy, obj.nbr.astype(np.int64), obj.y, np.zeros(a.n), obj.X, 1.0, a.rho, 1.5,
                                     O.Lik("bernoulli-logit"), ocfg)
            cpu_s = time.perf_counter() - t0
            ograd = np.asarray(og["dtheta"]) * theta
            line["oracle"] = {"s_per_eval": cpu_s, "cores": os.cpu_count(), "nll": float(oval),
                              "grad_log_theta": [float(g) for g in ograd],
                              "nll_rel": abs(val - oval) / abs(oval),
                              "grad_rel": float(np.max(np.abs(grad - ograd) / np.abs(ograd))),
                              "newton_cg": [int(c) for c in oinfo["state"].cg_iters],
                              "speedup": cpu_s / s_eval}
        lines.append(line)
        print(json.dumps(line), flush=True)
        del obj
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as fh:
            for ln in lines:
                fh.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()
