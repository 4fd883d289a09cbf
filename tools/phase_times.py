"""Wall-clock split of one headline evaluation by phase (synchronised), and
the host-side hot spots (cProfile) -- finds time outside the tagged kernels."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2310_12000_b200 as vg  # noqa: E402
from paper_2310_12000_b200.estimate import FitConfig, _Objective  # noqa: E402
from paper_2310_12000_b200.laplace import find_mode, gradient, make_probes, neg_marginal_loglik  # noqa: E402
from paper_2310_12000_b200.vecchia import build_factor  # noqa: E402

n, rho, seed = 1_000_000, 0.02, 2310
import argparse  # noqa: E402
ns = argparse.Namespace(n=n, seed=seed)
coords, _ = bench.synth(ns)
b_true = bench.latent_field(coords, rho, seed)
y = (np.random.default_rng(seed + 4).uniform(size=n) < 1.0 / (1.0 + np.exp(-b_true))).astype(float)
cfg = FitConfig(m=20, ordering_seed=seed + 3, nu=1.5,
                backend=vg.BackendConfig(t=50, cg_tol=1e-3, probe_seed=seed + 5, newton_grad_tol=1e-5))
obj = _Objective(y, np.zeros((n, 0)), coords, vg.get_likelihood("bernoulli-logit"), cfg)
theta = np.array([1.0, rho])
obj.evaluate(theta, np.zeros(0), np.zeros(0), want_grad=True)
obj.evaluate(theta, np.zeros(0), np.zeros(0), want_grad=True)


def phases():
    out = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = build_factor(obj.xy, vg.CovarianceSpec(1.0, rho, 1.5), obj.pattern, want_grad=True)
    torch.cuda.synchronize(); t1 = time.perf_counter(); out["factor"] = t1 - t0
    st = find_mode(f, obj.lik0, obj.y, np.zeros(n), cfg.backend)
    torch.cuda.synchronize(); t2 = time.perf_counter(); out["find_mode"] = t2 - t1
    pr, P = make_probes(f, st, cfg.backend)
    torch.cuda.synchronize(); t3 = time.perf_counter(); out["make_probes"] = t3 - t2
    nll = neg_marginal_loglik(st, f, cfg.backend, probes=pr, P=P)
    torch.cuda.synchronize(); t4 = time.perf_counter(); out["nll"] = t4 - t3
    g = gradient(st, f, obj.lik0, obj.X, cfg.backend, probes=pr, P=P)
    torch.cuda.synchronize(); t5 = time.perf_counter(); out["gradient"] = t5 - t4
    out["total"] = t5 - t0
    return out


for _ in range(2):
    print({k: round(v * 1e3, 1) for k, v in phases().items()}, flush=True)
pr_ = cProfile.Profile()
pr_.enable()
phases()
pr_.disable()
pstats.Stats(pr_).sort_stats("tottime").print_stats(25)
st = pstats.Stats(pr_)
st.sort_stats("tottime").print_callers("reduce|take|perf_counter|_lib.py")
