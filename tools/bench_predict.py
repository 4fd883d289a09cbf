"""Prediction benchmark (config 4 shaped): n training + n_p prediction points,
Poisson-log responses, VADU mode, prediction blocks, latent mean and the
simulation variance estimator with s samples (one JSON line).  Synthetic
inputs: uniform coords, a Vecchia-sampled latent field (m_sim=30)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_12000_b200 as vg  # noqa: E402
from paper_2310_12000_b200.vecchia import build_factor, neighbor_array  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=500_000)
    ap.add_argument("--np", type=int, default=500_000)
    ap.add_argument("--m", type=int, default=20)
    ap.add_argument("--s", type=int, default=1000)
    ap.add_argument("--chunk", type=int, default=64)
    ap.add_argument("--rho", type=float, default=0.02)
    ap.add_argument("--rng", default="device")
    a = ap.parse_args()
    T = vg.device.torch() if hasattr(vg, "device") else None
    import torch
    rng = np.random.default_rng(4)
    N = a.n + a.np
    xy = rng.uniform(size=(N, 2))
    spec = vg.CovarianceSpec(1.0, a.rho, 1.5)
    # latent field by Vecchia sampling over all N points
    permS = vg.order_random(N, 99)
    fS = build_factor(xy, spec, neighbor_array(xy, permS, 30), permS)
    g = rng.standard_normal(N)
    bS = fS.solve_B(np.sqrt(fS.D) * g)
    latent = np.empty(N)
    latent[permS] = bS
    lik = vg.get_likelihood("poisson")
    y = lik.sample(latent[: a.n], rng)
    perm = vg.order_random(a.n, 7)
    t0 = time.perf_counter()
    f = build_factor(xy[: a.n], spec, neighbor_array(xy[: a.n], perm, a.m), perm)
    cfg = vg.BackendConfig(preconditioner="vadu", t=50, cg_tol=1e-3)
    st = vg.find_mode(f, lik, y[perm], np.zeros(a.n), cfg)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    blocks = vg.prediction_blocks(f, xy[a.n:])
    omega = vg.latent_mean(st, blocks, np.zeros(a.np))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    var = vg.latent_var_sim(st, f, blocks, s=a.s, seed=5, cfg=cfg, chunk=a.chunk, rng=a.rng)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    truth = latent[a.n:]
    print(json.dumps({
        "metric": "prediction: latent mean + simulated variances", "config": {
            "workload": f"predict_n{a.n}_np{a.np}_s{a.s}", "m": a.m, "likelihood": "poisson", "rng": a.rng,
            "chunk": a.chunk, "cg_tol": cfg.cg_tol},
        "fit_mode_s": round(t1 - t0, 3), "blocks_mean_s": round(t2 - t1, 3), "var_sim_s": round(t3 - t2, 3),
        "samples_per_s": round(a.s / (t3 - t2), 2), "rmse": vg.rmse(omega, truth),
        "mean_var": float(var.mean()), "newton_iters": st.newton_iters}))


if __name__ == "__main__":
    main()
