"""GPU parity of the prediction path (config-4 shaped, Poisson) against the
reference-generated fixture: prediction blocks, latent mean, the simulation
variance estimator (same draws) and the exact variances."""

import numpy as np
import pytest

from _golden import load, scal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def case():
    import paper_2310_12000_b200 as vg
    from paper_2310_12000_b200.vecchia import build_factor
    g = load("poisson_pred_n500")
    spec = vg.CovarianceSpec(scal(g, "sigma2"), scal(g, "rho"), scal(g, "nu"))
    f = build_factor(g["coords"], spec, g["nbr"], g["perm"])
    lik = vg.get_likelihood("poisson")
    cfg = vg.BackendConfig(preconditioner="vadu", t=int(g["t"]), probe_seed=int(g["probe_seed"]))
    perm = g["perm"]
    st = vg.find_mode(f, lik, g["y"][perm], g["F"][perm], cfg)
    blocks = vg.prediction_blocks(f, g["pcoords"])
    return vg, g, f, st, cfg, blocks


def test_mode_and_blocks(case):
    vg, g, f, st, cfg, blocks = case
    assert st.newton_iters == int(g["newton_iters"])
    assert np.abs(st.b - g["b"]).max() <= 1e-8 * max(1.0, np.abs(g["b"]).max())
    np.testing.assert_array_equal(np.stack(blocks.neighbors), g["pred_nbr"])
    np.testing.assert_allclose(blocks.values, g["Bpo_vals"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(blocks.Dp, g["Dp"], rtol=1e-10)


def test_latent_mean(case):
    vg, g, f, st, cfg, blocks = case
    omega = vg.latent_mean(st, blocks, np.zeros(blocks.n_p))
    np.testing.assert_allclose(omega, g["omega"], rtol=1e-7, atol=1e-9)


def test_latent_var_sim_same_draws(case):
    vg, g, f, st, cfg, blocks = case
    var, cov = vg.latent_var_sim(st, f, blocks, s=int(g["s"]), seed=int(g["sim_seed"]), cfg=cfg, full=True, chunk=7)
    np.testing.assert_allclose(var, g["var_sim"], rtol=1e-7)
    np.testing.assert_allclose(cov, g["cov_sim"], rtol=1e-6, atol=1e-9)
    var2 = vg.latent_var_sim(st, f, blocks, s=int(g["s"]), seed=int(g["sim_seed"]), cfg=cfg)  # chunking invariant
    np.testing.assert_allclose(var2, var, rtol=1e-12)


def test_latent_var_exact(case):
    vg, g, f, st, cfg, blocks = case
    var = vg.latent_var_exact(st, f, blocks)
    np.testing.assert_allclose(var, g["var_exact"], rtol=1e-7)


def test_predict_latent_and_scores(case):
    vg, g, f, st, cfg, blocks = case
    pred = vg.predict_latent(st, f, blocks, np.zeros(blocks.n_p), method="simulation", cfg=cfg, s=16, seed=2)
    assert pred.var.shape == (blocks.n_p,) and np.all(pred.var > 0)
    vg.response_moments(pred, vg.get_likelihood("poisson"), n_s=50, seed=1)
    assert np.isfinite(vg.scores(pred, g["truth"], "rmse"))
    assert np.isfinite(vg.scores(pred, g["truth"], "log-score"))
    assert np.isfinite(vg.scores(pred, np.exp(g["truth"]), "crps"))


def test_duplicate_prediction_point_rejected(case):
    vg, g, f, st, cfg, blocks = case
    with pytest.raises(vg.DataError):
        vg.prediction_blocks(f, g["coords"][:3])


@pytest.mark.parametrize("variant", ["none", "l1", "l2"])
def test_latent_var_lanczos(case, variant):
    vg, g, f, st, cfg, blocks = case
    var, order = vg.latent_var_lanczos(st, f, blocks, 20, variant=variant, cfg=cfg)
    assert order == int(g[f"order_lz_{variant}"])
    np.testing.assert_allclose(var, g[f"var_lz_{variant}"], rtol=1e-7)


def _host_lanczos_none(Bm, D, W, Bpo, k):
    """predict.py:104-150 ("none") on the host with RT = Bpo^T kept sparse."""
    n = Bm.shape[0]
    RT = Bpo.T.tocsr()

    def op(v):
        return W * v + Bm.T @ ((Bm @ v) / D)

    start = np.asarray(RT.mean(axis=1)).ravel()
    Q = np.zeros((n, k))
    al, be = np.zeros(k), np.zeros(k - 1)
    Q[:, 0] = start / np.linalg.norm(start)
    for j in range(k):
        w = op(Q[:, j])
        al[j] = Q[:, j] @ w
        w -= al[j] * Q[:, j]
        if j:
            w -= be[j - 1] * Q[:, j - 1]
        for _ in range(2):
            w -= Q[:, :j + 1] @ (Q[:, :j + 1].T @ w)
        if j == k - 1:
            break
        be[j] = np.linalg.norm(w)
        Q[:, j + 1] = w / be[j]
    T = np.diag(al) + np.diag(be, 1) + np.diag(be, -1)
    S = (RT.T @ Q).T
    return np.einsum("kj,kj->j", S, np.linalg.solve(T, S))


def test_latent_var_lanczos_sparse_scale():
    """n = n_p = 3e4 (9e8 dense RT entries: beyond the dense formulation) against
    the same algorithm on the host with a sparse RT; odd rank (padded panel)."""
    import paper_2310_12000_b200 as vg
    from paper_2310_12000_b200.vecchia import build_factor, neighbor_array
    rng = np.random.default_rng(11)
    n = n_p = 30_000
    xy = rng.uniform(size=(n + n_p, 2))
    perm = vg.order_random(n, 5)
    spec = vg.CovarianceSpec(1.0, 0.05, 1.5)
    f = build_factor(xy[:n], spec, neighbor_array(xy[:n], perm, 10), perm, want_grad=False)
    lik = vg.get_likelihood("poisson")
    y = lik.sample(0.3 * rng.standard_normal(n), rng)
    cfg = vg.BackendConfig(preconditioner="vadu", t=4)
    st = vg.find_mode(f, lik, y[perm], np.zeros(n), cfg)
    blocks = vg.prediction_blocks(f, xy[n:])
    k = 31
    var, order = vg.latent_var_lanczos(st, f, blocks, k, variant="none", cfg=cfg)
    assert order == k
    corr = _host_lanczos_none(f.B, f.D, st.W, blocks.Bpo, k)
    np.testing.assert_allclose(var - blocks.Dp, corr, rtol=1e-7, atol=1e-12)
    for variant in ("l1", "l2"):
        v2, o2 = vg.latent_var_lanczos(st, f, blocks, k, variant=variant, cfg=cfg)
        assert o2 == k and np.all(np.isfinite(v2))
        if variant == "l1":   # symmetric form: the rank-k correction is a nonnegative quadratic form
            assert np.all(v2 >= blocks.Dp - 1e-12)


@pytest.mark.parametrize("variant", ["none", "l1", "l2"])
def test_latent_var_lanczos_full_rank_is_exact(case, variant):
    """At full Krylov rank every variant reproduces the exact variances."""
    vg, g, f, st, cfg, blocks = case
    var, order = vg.latent_var_lanczos(st, f, blocks, f.n, variant=variant, cfg=cfg)
    assert 1 <= order <= f.n
    np.testing.assert_allclose(var, vg.latent_var_exact(st, f, blocks), rtol=1e-6)
