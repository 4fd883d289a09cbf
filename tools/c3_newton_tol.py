"""Config-3 (bench workload) device evaluations at several newton_grad_tol
values against the reference's own result (tests/golden/c3_reference.json):
shows where the Newton stopping step lands and how NLL / dtheta move with it."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
import paper_2310_12000_b200 as vg  # noqa: E402
from paper_2310_12000_b200.vecchia import build_factor, neighbor_array  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tols", default="1e-5,8e-6,6e-6,5e-6,4e-6,3e-6")
ap.add_argument("--maxits", default="")
a = ap.parse_args()
ref = json.load(open(os.path.join(ROOT, "tests", "golden", "c3_reference.json")))
n, rho, seed = ref["n"], ref["rho"], ref["seed"]
coords, _ = bench.synth(argparse.Namespace(n=n, seed=seed))
b = bench.latent_field(coords, rho, seed)
y = (np.random.default_rng(seed + 4).uniform(size=n) < 1.0 / (1.0 + np.exp(-b))).astype(float)
perm = vg.order_random(n, ref["ordering_seed"])
nbr = neighbor_array(coords, perm, 20)
f = build_factor(coords, vg.CovarianceSpec(1.0, rho, 1.5), nbr, perm)
lik = vg.get_likelihood("bernoulli-logit")
for tol in [float(x) for x in a.tols.split(",")]:
    cfg = vg.BackendConfig(t=50, cg_tol=1e-3, probe_seed=ref["probe_seed"], newton_grad_tol=tol)
    try:
        st = vg.find_mode(f, lik, y[perm], np.zeros(n), cfg)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"tol": tol, "error": f"{type(e).__name__}: {e}"}), flush=True)
        continue
    pr, P = vg.make_probes(f, st, cfg)
    nll = vg.neg_marginal_loglik(st, f, cfg, probes=pr, P=P)
    g = vg.gradient(st, f, lik, np.zeros((n, 0)), cfg, probes=pr, P=P)
    print(json.dumps({"tol": tol, "newton_iters": st.newton_iters, "newton_cg": list(map(int, st.cg_iters)),
                      "ref_newton_cg": ref["newton_cg"], "nll": nll, "nll_rel": abs(nll - ref["nll"]) / abs(ref["nll"]),
                      "dtheta": list(map(float, g["dtheta"])),
                      "dtheta_rel": [abs(x - r) / abs(r) for x, r in zip(g["dtheta"], ref["dtheta"])],
                      "y_sha_match": bench._sha(y.astype(np.uint8)) == ref["y_sha256"]}), flush=True)
