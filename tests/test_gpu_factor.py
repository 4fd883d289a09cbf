"""GPU parity: factor build, products and triangular solves vs the reference
fixtures and the CPU oracle (SURVEY 8(c) tolerances)."""

import numpy as np
import pytest

from _golden import csr, load, scal
from oracle import vl_oracle as O

pytestmark = pytest.mark.gpu

CASES = ["logit_vadu_n400", "logit_vadu_n1500", "probit_vadu_n300", "gamma_vadu_n300"]


@pytest.fixture(scope="module")
def vg():
    import paper_2310_12000_b200 as vg
    return vg


def _factor(vg, g, order_kind=1):
    from paper_2310_12000_b200.vecchia import build_factor
    spec = vg.CovarianceSpec(scal(g, "sigma2"), scal(g, "rho"), scal(g, "nu"))
    return build_factor(g["coords"], spec, g["nbr"], g["perm"], order_kind=order_kind)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("order_kind", [0, 1, 2])
def test_factor_values(vg, name, order_kind):
    g = load(name)
    f = _factor(vg, g, order_kind)
    s2 = scal(g, "sigma2")
    B = csr(g, "B")
    assert np.abs(f.D - g["D"]).max() / s2 <= 1e-12
    fB = f.B
    assert np.array_equal(fB.indptr, B.indptr) and np.array_equal(fB.indices, B.indices)
    assert np.abs(fB.data - B.data).max() <= 1e-10 * max(1.0, np.abs(B.data).max())
    g0 = vg.factor_gradient(f, 0)
    g1 = vg.factor_gradient(f, 1)
    assert np.abs(g0.dD - g["dD_sig"]).max() <= 1e-12
    dB = csr(g, "dB_rho")
    assert np.abs(g1.dB.data - dB.data).max() <= 1e-9 * max(1.0, np.abs(dB.data).max())
    assert np.abs(g1.dD - g["dD_rho"]).max() <= 1e-9 * max(1.0, np.abs(g["dD_rho"]).max())


@pytest.mark.parametrize("name", ["logit_vadu_n400", "logit_vadu_n1500"])
def test_kernel_ops_vs_reference(vg, name):
    g = load(name)
    f = _factor(vg, g)
    X = g["kx"]

    def rel(a, b):
        return np.abs(a - b).max() / max(1e-300, np.abs(b).max())

    # own factor: inherits the LU-vs-Cholesky factor differences
    assert rel(f.B_matvec(X), g["kBx"]) <= 1e-10
    assert rel(f.BT_matvec(X), g["kBtx"]) <= 1e-10
    assert rel(f.solve_B(X), g["kBinvx"]) <= 1e-9
    assert rel(f.solve_B(X, transpose=True), g["kBtinvx"]) <= 1e-9
    # replay: identical B and D -> kernel-level parity (rel <= 1e-12)
    f.set_values(csr(g, "B"), g["D"])
    assert rel(f.B_matvec(X), g["kBx"]) <= 1e-12
    assert rel(f.BT_matvec(X), g["kBtx"]) <= 1e-12
    assert rel(f.solve_B(X), g["kBinvx"]) <= 1e-12
    assert rel(f.solve_B(X, transpose=True), g["kBtinvx"]) <= 1e-12
    assert rel(f.apply_precision(X), g["kQx"]) <= 1e-12
    assert rel(f.apply_sigma_tilde(X), g["kSx"]) <= 1e-12


@pytest.mark.parametrize("t", [1, 3, 8, 13, 32, 50, 64, 100])
def test_ops_multi_rhs_vs_oracle(vg, t):
    rng = np.random.default_rng(t)
    n, m = 20000, 20
    xy = rng.uniform(size=(n, 2))
    nbr = vg.vecchia.neighbor_array(xy, np.arange(n), m)
    f = vg.vecchia.build_factor(xy, vg.CovarianceSpec(1.0, 0.05, 1.5), nbr)
    fo = O.Factor(xy, nbr, 1.0, 0.05, 1.5, f.B, f.D)
    X = rng.standard_normal((n, t))
    for got, want in [(f.B_matvec(X), fo.Bmul(X)), (f.BT_matvec(X), fo.BTmul(X)),
                      (f.solve_B(X), fo.solve_B(X)), (f.solve_B(X, True), fo.solve_B(X, True))]:
        assert np.abs(got - want).max() <= 1e-11 * np.abs(want).max()


def test_full_conditioning_exact(vg):
    # pkg/tests/test_vecchia.py:81-88: m = n-1 reproduces the dense inverse
    rng = np.random.default_rng(5)
    coords = rng.uniform(size=(50, 2))
    spec = vg.CovarianceSpec(1.0, 0.2, 1.5)
    f = vg.make_factor(coords, spec, 49, ordering_seed=1)
    from paper_2310_12000_b200.covariance import cov_matrix
    Sig = cov_matrix(spec, f.coords)
    Q = (f.B.T @ np.diag(1.0 / f.D) @ f.B)
    assert np.abs(Q - np.linalg.inv(Sig)).max() < 1e-8


def test_full_conditioning_n200(vg):
    # pkg/tests/test_vecchia.py:113-119 (m = 199, global-scratch build path)
    rng = np.random.default_rng(6)
    coords = rng.uniform(size=(200, 2))
    spec = vg.CovarianceSpec(1.0, 0.1, 1.5)
    f = vg.make_factor(coords, spec, 199, ordering_seed=2)
    from paper_2310_12000_b200.covariance import cov_matrix
    Sig = cov_matrix(spec, f.coords)
    assert np.abs(f.dense_sigma_tilde() - Sig).max() < 1e-8 * spec.sigma2


def test_three_point_hand_case(vg):
    coords = np.array([[0.0], [1.0], [3.0]])
    spec = vg.CovarianceSpec(1.5, 2.0, 0.5)
    nb = vg.find_neighbors(coords, np.arange(3), 1)
    f = vg.build_factor(coords, spec, nb)
    c01, c12 = 1.5 * np.exp(-0.5), 1.5 * np.exp(-1.0)
    B = f.B.toarray()
    assert B[1, 0] == pytest.approx(-c01 / 1.5, rel=1e-14)
    assert B[2, 1] == pytest.approx(-c12 / 1.5, rel=1e-14)
    np.testing.assert_allclose(f.D, [1.5, 1.5 - c01 * c01 / 1.5, 1.5 - c12 * c12 / 1.5], rtol=1e-14)


def test_m_zero_identity(vg):
    coords = np.random.default_rng(0).uniform(size=(15, 2))
    f = vg.build_factor(coords, vg.CovarianceSpec(2.3, 0.1, 1.5), [np.empty(0, int)] * 15)
    assert (f.B != np.eye(15)).sum() == 0
    np.testing.assert_allclose(f.D, 2.3)


def test_near_duplicates_raise(vg):
    coords = np.array([[0.0, 0.0], [0.5, 0.5], [0.5 + 1e-9, 0.5]])
    nb = vg.find_neighbors(coords, np.arange(3), 2)
    with pytest.raises(vg.FactorizationError):
        vg.build_factor(coords, vg.CovarianceSpec(1.0, 0.3, 1.5), nb)


def _random_parents(n, m, rng):
    """Row i: min(i, m) distinct parents uniform on [0, i) (BASELINE config 5)."""
    nbr = np.full((n, m), -1, dtype=np.int64)
    for i in range(1, n):
        k = min(i, m)
        nbr[i, :k] = rng.choice(i, size=k, replace=False)
    return nbr.astype(np.int32)


@pytest.mark.parametrize("t", [1, 16, 64])
@pytest.mark.parametrize("order_kind", [0, 1])
def test_ops_random_parents_vs_oracle(vg, t, order_kind):
    # config-5 style pattern: the first rows have hundreds of children, so the
    # B^T products run on work-balanced runs; order_kind 1 also takes the
    # SM-local product sweep (n >= 64 rows per SM)
    rng = np.random.default_rng(100 + t)
    n, m = 30000, 20
    xy = rng.uniform(size=(n, 2))
    nbr = _random_parents(n, m, rng)
    f = vg.vecchia.build_factor(xy, vg.CovarianceSpec(1.0, 0.05, 1.5), nbr, order_kind=order_kind)
    fo = O.Factor(xy, nbr.astype(np.int64), 1.0, 0.05, 1.5, f.B, f.D)
    X = rng.standard_normal((n, t))
    for got, want in [(f.B_matvec(X), fo.Bmul(X)), (f.BT_matvec(X), fo.BTmul(X)),
                      (f.solve_B(X), fo.solve_B(X)), (f.solve_B(X, True), fo.solve_B(X, True))]:
        assert np.abs(got - want).max() <= 1e-11 * np.abs(want).max()
