"""Measured spread between the device path and the reference fixtures, per
case: b*, NLL, dtheta/dbeta/dxi relative errors (prints one JSON line per
case).  Used to set the bars in tests/test_gpu_laplace.py."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from _golden import LAPLACE_CASES, load, scal  # noqa: E402

import paper_2310_12000_b200 as vg  # noqa: E402
from paper_2310_12000_b200.vecchia import build_factor  # noqa: E402


def rel(a, b):
    a, b = np.atleast_1d(np.asarray(a, float)), np.atleast_1d(np.asarray(b, float))
    if a.size == 0:
        return 0.0
    return float(np.abs(a - b).max() / max(1e-300, np.abs(b).max()))


def relv(a, b):
    a, b = np.atleast_1d(np.asarray(a, float)), np.atleast_1d(np.asarray(b, float))
    return [float(abs(x - y) / max(1e-300, abs(y))) for x, y in zip(a, b)]


for name in LAPLACE_CASES:
    g = load(name)
    spec = vg.CovarianceSpec(scal(g, "sigma2"), scal(g, "rho"), scal(g, "nu"))
    f = build_factor(g["coords"], spec, g["nbr"], g["perm"])
    fam = str(g["family"])
    lik = vg.get_likelihood(fam, **({"shape": float(g["shape"])} if fam == "gamma" else {}))
    rank = int(g["rank"])
    cfg = vg.BackendConfig(preconditioner=str(g["precond"]), t=int(g["t"]), probe_seed=int(g["probe_seed"]),
                           rank=None if rank < 0 else rank)
    perm = g["perm"]
    st = vg.find_mode(f, lik, g["y"][perm], g["F"][perm], cfg)
    pr, P = vg.make_probes(f, st, cfg)
    val = vg.neg_marginal_loglik(st, f, cfg, probes=pr, P=P)
    gr = vg.gradient(st, f, lik, g["X"][perm], cfg, probes=pr, P=P)
    print(json.dumps({"case": name, "newton": [st.newton_iters, int(g["newton_iters"])],
                      "b": rel(st.b, g["b"]), "Z": rel(pr.Z, g["Z"]), "nll": rel(val, g["nll"]),
                      "dtheta": relv(gr["dtheta"], g["dtheta"]), "dbeta": relv(gr["dbeta"], g["dbeta"]),
                      "dxi": relv(gr["dxi"], g["dxi"]),
                      "cg_len_maxdiff": int(np.abs(np.array([t.order for t in pr.tridiags]) - g["tri_len"]).max())}),
          flush=True)
