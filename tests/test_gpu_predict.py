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
