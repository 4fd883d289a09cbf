"""Config-2 LRAC (n=1e5, rank 1000) device evaluations at several
newton_grad_tol values against the reference fixture (c2_lrac_n1e5.npz):
Newton steps, convergence and NLL / dtheta relative differences."""
import json
import os
import sys

import numpy as np

ROOT = os.environ.get("C2_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import paper_2310_12000_b200 as vg  # noqa: E402
from paper_2310_12000_b200.vecchia import build_factor, neighbor_array  # noqa: E402
from _golden import GOLDEN  # noqa: E402

z = np.load(os.path.join(GOLDEN, "c2_lrac_n1e5.npz"))
meta = json.loads(str(z["meta"]))
n = meta["n"]
coords = np.random.default_rng(meta["seed"]).uniform(size=(n, 2))
y = np.unpackbits(z["y_bits"])[:n].astype(float)
perm = vg.order_random(n, meta["ordering_seed"])
f = build_factor(coords, vg.CovarianceSpec(1.0, meta["rho"], 1.5), neighbor_array(coords, perm, 20), perm)
lik = vg.get_likelihood("bernoulli-logit")
for tol in [float(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1e-5,2e-5,4e-5").split(",")]:
    cfg = vg.BackendConfig(preconditioner="lrac", rank=1000, t=50, cg_tol=1e-3, probe_seed=meta["probe_seed"],
                           newton_grad_tol=tol)
    try:
        st = vg.find_mode(f, lik, y[perm], np.zeros(n), cfg)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"lib": vg._lib.LIB_PATH if hasattr(vg._lib, "LIB_PATH") else "", "tol": tol,
                          "error": str(e)[:200]}), flush=True)
        continue
    pr, P = vg.make_probes(f, st, cfg)
    nll = vg.neg_marginal_loglik(st, f, cfg, probes=pr, P=P)
    g = vg.gradient(st, f, lik, np.zeros((n, 0)), cfg, probes=pr, P=P)
    print(json.dumps({"root": ROOT, "tol": tol, "newton": st.newton_iters, "ref_newton": meta["newton_iters"],
                      "b_rel": float(np.abs(st.b[::97] - z["b_stride"]).max() / np.abs(z["b_stride"]).max()),
                      "nll_rel": abs(nll - meta["nll"]) / abs(meta["nll"]),
                      "dtheta_rel": [abs(a - r) / abs(r) for a, r in zip(g["dtheta"], meta["dtheta"])]}), flush=True)
