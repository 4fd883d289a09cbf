"""The fit() driver on the device objective against the reference's own fit()
run (same seeds, same Nesterov/backtracking decisions), plus SAA bitwise
determinism (test_estimate.py:37-44 of the reference)."""

import numpy as np
import pytest

from _golden import load

pytestmark = pytest.mark.gpu


def _run(name):
    import paper_2310_12000_b200 as vg
    g = load(name)
    fam = str(g["family"])
    lik = vg.get_likelihood(fam, **({"shape": float(g["shape"])} if fam == "gamma" else {}))
    cfg = vg.FitConfig(m=int(g["m"]), ordering_seed=4, max_iters=int(g["max_iters"]),
                       backend=vg.BackendConfig(preconditioner="vadu", t=int(g["t"]), probe_seed=9, cg_tol=1e-6))
    return g, vg.fit(g["y"], g["X"], g["coords"], lik, cfg)


@pytest.mark.parametrize("name", ["fit_logit_n400", "fit_gamma_n300"])
def test_fit_follows_reference_trajectory(name):
    g, res = _run(name)
    assert res.n_evaluations == int(g["n_evaluations"])
    assert res.iterations == int(g["iterations"])
    np.testing.assert_allclose([r["objective"] for r in res.trace], g["trace_obj"], rtol=1e-8)
    np.testing.assert_allclose([r["lr"] for r in res.trace], g["trace_lr"], rtol=1e-12)
    np.testing.assert_allclose(res.theta, g["theta"], rtol=1e-6)
    np.testing.assert_allclose(res.beta, g["beta"], rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(res.xi, g["xi"], rtol=1e-6)


def test_fit_is_bitwise_reproducible():
    _, a = _run("fit_logit_n400")
    _, b = _run("fit_logit_n400")
    assert a.objective == b.objective
    assert np.array_equal(a.theta, b.theta) and np.array_equal(a.beta, b.beta)
