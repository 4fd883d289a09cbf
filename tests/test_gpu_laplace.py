"""GPU parity of the full Laplace evaluation (mode, probes, SLQ NLL, STE
gradient) against the reference-generated fixtures (tests/golden) and the
CPU oracle."""

import numpy as np
import pytest

from _golden import LAPLACE_CASES, load, scal, tridiags

pytestmark = pytest.mark.gpu

VADU_CASES = [c for c in LAPLACE_CASES if "lrac" not in c]
LRAC_CASES = [c for c in LAPLACE_CASES if "lrac" in c]


@pytest.fixture(scope="module")
def vg():
    import paper_2310_12000_b200 as vg
    return vg


def _setup(vg, g):
    from paper_2310_12000_b200.vecchia import build_factor
    spec = vg.CovarianceSpec(scal(g, "sigma2"), scal(g, "rho"), scal(g, "nu"))
    f = build_factor(g["coords"], spec, g["nbr"], g["perm"])
    fam = str(g["family"])
    lik = vg.get_likelihood(fam, **({"shape": float(g["shape"])} if fam == "gamma" else {}))
    rank = int(g["rank"])
    cfg = vg.BackendConfig(preconditioner=str(g["precond"]), t=int(g["t"]), probe_seed=int(g["probe_seed"]),
                           rank=None if rank < 0 else rank)
    perm = g["perm"]
    return f, lik, cfg, g["y"][perm], g["F"][perm], g["X"][perm]


def _rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(1e-300, np.abs(np.asarray(b)).max())


@pytest.mark.parametrize("name", VADU_CASES)
def test_mode_matches_reference(vg, name):
    g = load(name)
    f, lik, cfg, y, F, X = _setup(vg, g)
    st = vg.find_mode(f, lik, y, F, cfg)
    assert st.converged
    weak = str(g["precond"]) in ("diag", "identity", "pchol-precision", "rowsel", "l2")
    # the l2 diagonal uses diag(SigmaTilde) from device solves (SuperLU in the reference): the
    # gamma case's slow final Newton steps may stop one step apart at the same mode
    assert abs(st.newton_iters - int(g["newton_iters"])) <= (1 if weak else 0)
    # The last inexact-Newton step (CG to mode_cg_tol) fixes the mode only to ~1e-8 relative:
    # on the Poisson case a rounding-level change of the device products (fma vs. separate
    # product + add in one B^T pass) moves b* by 2e-8 while NLL and gradient stay at their bars.
    bar = 1e-6 if weak else (5e-8 if str(g["family"]) == "poisson" else 1e-8)
    assert _rel(st.b, g["b"]) <= bar
    assert _rel(st.W, g["W"]) <= bar
    # logp alone is not stationary at the mode (d logp / d b = d1 != 0), so it inherits the
    # mode's own bar scaled by |d1 . db| / |logp|: measured <= 1.1e-10 over these fixtures
    # (gamma_vadu_n300 moved from 6e-11 to 1.02e-10 when the solves' in-row summation order
    # changed with the late-dependency-last layout)
    assert st.logp == pytest.approx(float(g["logp"]), rel=1e-8 if weak else 5e-10)
    assert st.quad == pytest.approx(float(g["quad"]), rel=1e-8)


@pytest.mark.parametrize("name", VADU_CASES)
def test_nll_and_gradient_match_reference(vg, name):
    g = load(name)
    f, lik, cfg, y, F, X = _setup(vg, g)
    st = vg.find_mode(f, lik, y, F, cfg)
    probes, P = vg.make_probes(f, st, cfg)
    # diagonal preconditioners: ~190 CG steps per system amplify last-bit differences
    # (see test_oracle_golden); the others are held to the SURVEY 8(c) bars
    weak = str(g["precond"]) in ("diag", "identity", "pchol-precision", "rowsel", "l2")
    assert _rel(probes.Z, g["Z"]) <= (1e-7 if weak else 1e-8)
    val = vg.neg_marginal_loglik(st, f, cfg, probes=probes, P=P)
    ref_len = [len(d) for d, _ in tridiags(g)]
    got_len = [tr.order for tr in probes.tridiags]
    assert np.abs(np.array(got_len) - np.array(ref_len)).max() <= (5 if weak else 1)  # iteration-count flips
    assert val == pytest.approx(float(g["nll"]), rel=1e-8)
    grad = vg.gradient(st, f, lik, X, cfg, probes=probes, P=P)
    # SURVEY 8(c) bar: gradients within 1e-8 relative (measured spread <= 5.2e-9, Poisson dtheta[0];
    # tools/parity_report.py -> profiles/r2_parity_report.jsonl).  The weak preconditioners run
    # 60-190 CG steps per system and differ from the reference at the CG-tolerance level.
    rt, at = (5e-3, 1e-9) if weak else (1e-8, 1e-12)
    np.testing.assert_allclose(grad["dtheta"], g["dtheta"], rtol=rt, atol=at)
    np.testing.assert_allclose(grad["dbeta"], g["dbeta"], rtol=rt, atol=at)
    np.testing.assert_allclose(grad["dxi"], g["dxi"], rtol=rt, atol=at)


def test_probe_solves_match_oracle_replay(vg):
    # kernel-level replay: same B, D, W and Z -> CG solutions and tridiagonals
    from _golden import csr
    from oracle import vl_oracle as O
    g = load("logit_vadu_n1500")
    f, lik, cfg, y, F, X = _setup(vg, g)
    st = vg.find_mode(f, lik, y, F, cfg)
    probes, P = vg.make_probes(f, st, cfg)
    vg.neg_marginal_loglik(st, f, cfg, probes=probes, P=P)
    fo = O.Factor(f.coords, g["nbr"], 1.0, float(g["rho"]), 1.5, f.B, f.D)
    Wh = st.W
    op = O.system_matvec(fo, Wh, "eq6")
    Pv = O.Vadu(fo, Wh)
    U = probes.solves
    Z = probes.Z
    for i in range(0, probes.t, 3):
        res = O.pcg(op, Z[:, i], Pv.solve, cfg.mode_cg_tol, 1000, capture=True)
        if res.iters != probes.tridiags[i].order:
            continue  # stopping-rule flip under rounding: compared elsewhere
        assert _rel(U[:, i], res.u) <= 1e-10
        assert _rel(probes.tridiags[i].diag, res.diag) <= 1e-10


def test_sharded_gradient_path_matches_fused(vg):
    """The multi-GPU split of the gradient pass (row-stat allreduce rounds,
    probe-ordered gathers) run as a 1-rank NCCL group equals the fused pass."""
    import os
    import socket

    import torch
    import torch.distributed as dist
    from paper_2310_12000_b200.distributed import ProbeComm
    g = load("logit_vadu_n1500")
    f, lik, cfg, y, F, X = _setup(vg, g)
    st = vg.find_mode(f, lik, y, F, cfg)
    probes, P = vg.make_probes(f, st, cfg)
    vg.neg_marginal_loglik(st, f, cfg, probes=probes, P=P)
    ref = vg.gradient(st, f, lik, X, cfg, probes=probes, P=P)
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        comm = ProbeComm(force_split=True)
        got = vg.gradient(st, f, lik, X, cfg, probes=probes, P=P, comm=comm)
    finally:
        dist.destroy_process_group()
    np.testing.assert_allclose(got["dtheta"], ref["dtheta"], rtol=1e-10, atol=1e-12)


def test_lrac_pivoted_cholesky_matches_oracle(vg):
    from oracle import vl_oracle as O
    from paper_2310_12000_b200.laplace import LracFactorHandle
    g = load("logit_lrac_n300")
    f, lik, cfg, y, F, X = _setup(vg, g)
    lf = LracFactorHandle(f, int(g["rank"]))
    L_o, piv_o = O.pchol_sigma(f.coords, 1.0, float(g["rho"]), 1.5, int(g["rank"]))
    assert np.array_equal(lf.pivots, piv_o)
    assert _rel(lf.L(), L_o) <= 1e-10


@pytest.mark.parametrize("name", LRAC_CASES)
def test_lrac_nll_and_gradient_match_reference(vg, name):
    g = load(name)
    f, lik, cfg, y, F, X = _setup(vg, g)
    cfg = vg.BackendConfig(preconditioner="lrac", t=int(g["t"]), probe_seed=int(g["probe_seed"]),
                           rank=int(g["rank"]))
    st = vg.find_mode(f, lik, y, F, cfg)
    assert st.newton_iters == int(g["newton_iters"])
    assert _rel(st.b, g["b"]) <= 1e-8
    probes, P = vg.make_probes(f, st, cfg)
    assert _rel(probes.Z, g["Z"]) <= 1e-8
    assert P.logdet() == pytest.approx(float(g["logdet_P"]), rel=1e-8)   # W at a mode agreeing to ~1e-8
    val = vg.neg_marginal_loglik(st, f, cfg, probes=probes, P=P)
    assert val == pytest.approx(float(g["nll"]), rel=1e-8)
    grad = vg.gradient(st, f, lik, X, cfg, probes=probes, P=P)
    np.testing.assert_allclose(grad["dtheta"], g["dtheta"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(grad["dbeta"], g["dbeta"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(grad["dxi"], g["dxi"], rtol=1e-8, atol=1e-12)
