"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``vlgp`` from /root/reference/pkg/src, runs the reference's own
public API (make_factor / factor_gradient / find_mode / make_probes /
neg_marginal_loglik / gradient / VecchiaFactor.solve_B) on small seeded
datasets and writes ``tests/golden/*.npz``.  The GPU box never reads
/root/reference: the tests only read these committed fixtures.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import vlgp  # noqa: F401
    return vlgp


def simulate(n, seed, rho, nu=1.5, family="bernoulli-logit", shape=2.0, F=None):
    """Dense-Cholesky GP draw + responses (same recipe as pkg/tests/util.py:11-42)."""
    from vlgp.covariance import CovarianceSpec, cov_matrix
    from vlgp.likelihoods import get_likelihood

    rng = np.random.default_rng(seed)
    coords = rng.uniform(size=(n, 2))
    spec = CovarianceSpec(1.0, rho, nu)
    b = np.linalg.cholesky(cov_matrix(spec, coords)) @ rng.standard_normal(n)
    lik = get_likelihood(family, **({"shape": shape} if family == "gamma" else {}))
    F = np.zeros(n) if F is None else F
    y = lik.sample(F + b, rng)
    return coords, y, lik


def _csr(prefix, M):
    M = M.tocsr()
    return {f"{prefix}_data": M.data, f"{prefix}_indices": M.indices.astype(np.int64),
            f"{prefix}_indptr": M.indptr.astype(np.int64)}


def laplace_case(name, n, seed, rho, m, t, precond="vadu", family="bernoulli-logit",
                 shape=2.0, rank=None, p=0, ordering_seed=7, probe_seed=3, theta=None,
                 nu=1.5, kernel_rhs=0):
    from vlgp.covariance import CovarianceSpec
    from vlgp.laplace import BackendConfig, find_mode, gradient, make_probes, neg_marginal_loglik
    from vlgp.vecchia import build_factor, factor_gradient, find_neighbors, order_random

    rng_x = np.random.default_rng(seed + 99)
    X = None
    F = np.zeros(n)
    if p:
        X = np.column_stack([np.ones(n)] + [rng_x.standard_normal(n) for _ in range(p - 1)])
        beta = np.linspace(0.2, -0.3, p)
        F = X @ beta
    else:
        beta = np.zeros(0)
    coords, y, lik = simulate(n, seed, rho, nu=nu, family=family, shape=shape, F=F)
    theta = (1.0, rho) if theta is None else theta
    spec = CovarianceSpec(theta[0], theta[1], nu)
    perm = order_random(n, ordering_seed)
    nb = find_neighbors(coords, perm, m)
    f = build_factor(coords, spec, nb, perm)
    g_sig = factor_gradient(f, 0)
    g_rho = factor_gradient(f, 1)
    cfg = BackendConfig(preconditioner=precond, t=t, probe_seed=probe_seed, rank=rank)
    y_f = y[perm]
    F_f = F[perm]
    X_f = X[perm] if X is not None else np.zeros((n, 0))
    st = find_mode(f, lik, y_f, F_f, cfg)
    probes, P = make_probes(f, st, cfg)
    val = neg_marginal_loglik(st, f, cfg, probes=probes, P=P)
    grad = gradient(st, f, lik, X_f, cfg, probes=probes, P=P)
    nbr = np.full((n, m), -1, dtype=np.int64)
    for i, s in enumerate(nb):
        nbr[i, : len(s)] = s
    out = dict(
        n=n, m=m, t=t, seed=seed, rho=rho, nu=nu, sigma2=theta[0], theta=np.array(theta),
        family=family, shape=shape, precond=precond, rank=-1 if rank is None else rank,
        ordering_seed=ordering_seed, probe_seed=probe_seed, coords=coords, y=y, F=F,
        X=np.zeros((n, 0)) if X is None else X, beta=beta, perm=perm, nbr=nbr,
        D=f.D, dD_sig=g_sig.dD, dD_rho=g_rho.dD, b=st.b, W=st.W, logp=st.logp, quad=st.quad,
        newton_iters=st.newton_iters, Z=probes.Z, solves=probes.solves, psolves=probes.psolves,
        tri_diag=np.concatenate([tr.diag for tr in probes.tridiags]),
        tri_len=np.array([tr.order for tr in probes.tridiags]),
        tri_off=np.concatenate([tr.off for tr in probes.tridiags]),
        logdet_P=P.logdet(), nll=val, dtheta=grad["dtheta"], dbeta=grad["dbeta"],
        dxi=grad["dxi"],
    )
    out.update(_csr("B", f.B))
    out.update(_csr("dB_rho", g_rho.dB))
    if kernel_rhs:
        Xr = np.random.default_rng(seed + 5).standard_normal((n, kernel_rhs))
        out.update(kx=Xr, kBx=f.B @ Xr, kBtx=f.B.T @ Xr, kBinvx=f.solve_B(Xr),
                   kBtinvx=f.solve_B(Xr, transpose=True), kQx=f.apply_precision(Xr),
                   kSx=f.apply_sigma_tilde(Xr))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: n={n} nll={val:.12g} dtheta={grad['dtheta']} newton={st.newton_iters}")


def register_poisson():
    """Test-only Poisson (log link) family registered into the REFERENCE so the
    rest of its pipeline runs unmodified (config 4 has no
    reference family)."""
    import vlgp.likelihoods as L
    from scipy.special import gammaln

    if "poisson" in L._FAMILIES:
        return

    class Poisson(L.Likelihood):
        name = "poisson"

        def validate(self, y):
            return np.asarray(y, dtype=float)

        def log_density(self, y, mu):
            return y * mu - np.exp(mu) - gammaln(y + 1.0)

        def derivs(self, y, mu):
            e = np.exp(mu)
            return float(self.log_density(y, mu).sum()), y - e, -e, -e

        def sample(self, mu, rng):
            return rng.poisson(np.exp(mu)).astype(float)

    L._FAMILIES["poisson"] = Poisson


def predict_case(name, n, n_p, seed, rho, m, family="poisson", s=24, sim_seed=11, nu=1.5, ordering_seed=7):
    """Prediction path (config-4 shaped, scaled down): prediction_blocks,
    latent_mean, latent_var_sim (diag + full) and latent_var_exact."""
    from vlgp.covariance import CovarianceSpec, cov_matrix
    from vlgp.laplace import BackendConfig, find_mode
    from vlgp.likelihoods import get_likelihood
    from vlgp.predict import latent_mean, latent_var_exact, latent_var_sim
    from vlgp.vecchia import build_factor, find_neighbors, order_random, prediction_blocks

    register_poisson()
    rng = np.random.default_rng(seed)
    allc = rng.uniform(size=(n + n_p, 2))
    spec = CovarianceSpec(1.0, rho, nu)
    ball = np.linalg.cholesky(cov_matrix(spec, allc)) @ rng.standard_normal(n + n_p)
    coords, pcoords = allc[:n], allc[n:]
    lik = get_likelihood(family)
    y = lik.sample(ball[:n], rng)
    perm = order_random(n, ordering_seed)
    nb = find_neighbors(coords, perm, m)
    f = build_factor(coords, spec, nb, perm)
    cfg = BackendConfig(preconditioner="vadu", t=8, probe_seed=3)
    st = find_mode(f, lik, y[perm], np.zeros(n), cfg)
    blocks = prediction_blocks(f, pcoords)
    Fp = np.zeros(n_p)
    omega = latent_mean(st, blocks, Fp)
    var_sim, cov_sim = latent_var_sim(st, f, blocks, s=s, seed=sim_seed, cfg=cfg, full=True)
    var_exact = latent_var_exact(st, f, blocks)
    from vlgp.predict import latent_var_lanczos
    lz = {}
    for variant in ("none", "l1", "l2"):
        v, order = latent_var_lanczos(st, f, blocks, 20, variant=variant, cfg=cfg)
        lz[f"var_lz_{variant}"] = v
        lz[f"order_lz_{variant}"] = order
    nbr = np.full((n, m), -1, dtype=np.int64)
    for i, q in enumerate(nb):
        nbr[i, : len(q)] = q
    out = dict(n=n, n_p=n_p, m=m, seed=seed, rho=rho, nu=nu, sigma2=1.0, family=family, shape=1.0,
               precond="vadu", t=8, probe_seed=3, cg_tol=cfg.cg_tol, coords=coords, pcoords=pcoords, y=y,
               F=np.zeros(n), perm=perm, nbr=nbr, b=st.b, W=st.W, newton_iters=st.newton_iters,
               pred_nbr=np.stack(blocks.neighbors).astype(np.int64), Bpo_vals=blocks.Bpo.data.reshape(n_p, -1),
               Dp=blocks.Dp, omega=omega, s=s, sim_seed=sim_seed, var_sim=var_sim, cov_sim=cov_sim,
               var_exact=var_exact, truth=ball[n:], **lz)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: n={n} n_p={n_p} newton={st.newton_iters} var_sim[:3]={var_sim[:3]}")


def fit_case(name, n, seed, rho, m, t, family="bernoulli-logit", p=2, max_iters=6, shape=2.0):
    """The reference's fit() driver (Nesterov + backtracking) on a small problem."""
    from vlgp.estimate import FitConfig, fit
    from vlgp.laplace import BackendConfig

    rng_x = np.random.default_rng(seed + 99)
    X = np.column_stack([np.ones(n)] + [rng_x.standard_normal(n) for _ in range(p - 1)])
    F = X @ np.linspace(0.2, -0.3, p)
    coords, y, lik = simulate(n, seed, rho, family=family, shape=shape, F=F)
    cfg = FitConfig(m=m, ordering_seed=4, max_iters=max_iters,
                    backend=BackendConfig(preconditioner="vadu", t=t, probe_seed=9, cg_tol=1e-6))
    res = fit(y, X, coords, lik, cfg)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), n=n, m=m, t=t, family=family, shape=shape, coords=coords,
                        y=y, X=X, max_iters=max_iters, theta=res.theta, beta=res.beta, xi=res.xi,
                        objective=res.objective, trace_obj=np.array([r["objective"] for r in res.trace]),
                        trace_lr=np.array([r["lr"] for r in res.trace]), n_evaluations=res.n_evaluations,
                        iterations=res.iterations, converged=res.converged)
    print(f"{name}: theta={res.theta} beta={res.beta} obj={res.objective:.10g} evals={res.n_evaluations}")


def cli_case(name):
    """The reference's own file formats end to end: cmd_simulate -> cmd_fit
    (model JSON) -> cmd_predict (predictions CSV), committed as fixtures."""
    import json

    from vlgp.cli import cmd_fit, cmd_predict, cmd_simulate

    d = os.path.join(HERE, name)
    os.makedirs(d, exist_ok=True)
    from vlgp.cli import _read_csv, _write_csv

    sim = {"n": 300, "d": 2, "likelihood": {"family": "bernoulli-logit"},
           "covariance": {"sigma2": 1.0, "rho": 0.1, "nu": 1.5},
           "fixed_effects": {"beta": [0.3], "design": "intercept"}, "seeds": {"simulation": 31}}
    full = os.path.join(d, "all.csv")
    cmd_simulate(sim, full)
    h, a = _read_csv(full)
    _, tr = _read_csv(os.path.join(d, "all.truth.csv"))
    data = os.path.join(d, "train.csv")
    pred_in = os.path.join(d, "pred.csv")
    _write_csv(data, h, a[:260].tolist())
    _write_csv(pred_in, h + ["b"], np.column_stack([a[260:], tr[260:, 0]]).tolist())
    os.remove(full)
    os.remove(os.path.join(d, "all.truth.csv"))
    fitcfg = {"likelihood": {"family": "bernoulli-logit"}, "m": 10, "nu": 1.5,
              "backend": {"preconditioner": "vadu", "t": 8, "cg_tol": 1e-6},
              "optimizer": {"max_iters": 4}, "seeds": {"ordering": 5, "probes": 6}}
    with open(os.path.join(d, "fit.json"), "w") as fh:
        json.dump(fitcfg, fh)
    cmd_fit(data, fitcfg, os.path.join(d, "model.json"))
    predcfg = {"prediction": {"method": "exact"}, "scores": ["rmse", "log-score"]}
    with open(os.path.join(d, "predict.json"), "w") as fh:
        json.dump(predcfg, fh)
    cmd_predict(os.path.join(d, "model.json"), data, pred_in, predcfg, os.path.join(d, "predictions.csv"))
    print(f"{name}: written to {d}")


def knn_case(name, n, m, seed, ordering_seed):
    from vlgp.vecchia import find_neighbors, order_random

    coords = np.random.default_rng(seed).uniform(size=(n, 2))
    perm = order_random(n, ordering_seed)
    nb = find_neighbors(coords, perm, m)
    nbr = np.full((n, m), -1, dtype=np.int32)
    for i, s in enumerate(nb):
        nbr[i, : len(s)] = s
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), coords=coords, perm=perm,
                        nbr=nbr, m=m)
    print(f"{name}: n={n} m={m}")


def main():
    _import_ref()
    # configs[0]-shaped (scaled down): bernoulli-logit, nu=1.5, VADU
    laplace_case("logit_vadu_n400", 400, seed=11, rho=0.1, m=10, t=8, kernel_rhs=3)
    laplace_case("logit_vadu_n1500", 1500, seed=12, rho=0.05, m=20, t=16, kernel_rhs=2)
    laplace_case("logit_vadu_cov_n300", 300, seed=13, rho=0.1, m=8, t=6, p=2)
    laplace_case("probit_vadu_n300", 300, seed=14, rho=0.1, m=8, t=6,
                 family="bernoulli-probit", nu=2.5)
    laplace_case("gamma_vadu_n300", 300, seed=15, rho=0.1, m=8, t=6, family="gamma",
                 shape=2.0, nu=0.5)
    laplace_case("logit_lrac_n300", 300, seed=16, rho=0.1, m=8, t=6, precond="lrac", rank=30)
    laplace_case("gamma_lrac_cov_n300", 300, seed=17, rho=0.1, m=8, t=6, precond="lrac", rank=25,
                 family="gamma", shape=1.5, nu=2.5, p=2)
    knn_case("knn_n6000_m12", 6000, 12, seed=21, ordering_seed=22)
    register_poisson()
    laplace_case("poisson_vadu_n300", 300, seed=18, rho=0.1, m=8, t=6, family="poisson")
    for pc, sd in (("lva", 25), ("diag", 26), ("identity", 27)):
        laplace_case(f"logit_{pc}_n300", 300, seed=sd, rho=0.1, m=8, t=6, precond=pc)
    laplace_case("logit_pcholprec_n300", 300, seed=28, rho=0.1, m=8, t=6, precond="pchol-precision", rank=40)
    laplace_case("logit_rowsel_n300", 300, seed=29, rho=0.1, m=8, t=6, precond="rowsel", rank=40)
    laplace_case("gamma_l2_n300", 300, seed=30, rho=0.1, m=8, t=6, precond="l2", family="gamma", shape=2.0)
    predict_case("poisson_pred_n500", 500, 60, seed=19, rho=0.1, m=10)
    fit_case("fit_logit_n400", 400, seed=23, rho=0.1, m=10, t=8)
    fit_case("fit_gamma_n300", 300, seed=24, rho=0.1, m=8, t=6, family="gamma", max_iters=4)
    cli_case("cli_logit")


if __name__ == "__main__":
    main()
