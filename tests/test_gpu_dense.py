"""The hand-written fp64 dense kernels of the low-rank paths (csrc/dense.cu)
against torch fp64 matmul / triangular inverse on the device: every
transpose combination, leading dimensions larger than the rows, alpha/beta,
the k-dimension weights of L^T W L, the lower-triangle (SYRK) mode and the
split-K path of long contractions."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2310_12000_b200 as vg  # noqa: F401
    from paper_2310_12000_b200 import _lib
    from paper_2310_12000_b200 import device as dev
    return torch, _lib, dev.context()


def _colmajor(torch, rows, cols, ld, gen):
    """A column-major rows x cols matrix with leading dimension ld: storage is
    a (cols, ld) row-major tensor; returns (storage, logical view)."""
    st = torch.randn(cols, ld, dtype=torch.float64, device="cuda", generator=gen)
    return st, st[:, :rows].T


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (37, 70, 19), (64, 64, 64), (130, 3, 5000), (5, 129, 300000),
                                   (1000, 1, 100000), (1000, 7, 20000), (1, 20000, 1000), (6, 5000, 700)])
def test_dgemm_matches_torch(env, ta, tb, m, n, k):
    torch, _lib, ctx = env
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k + 10 * ta + tb)
    ar, ac = (k, m) if ta else (m, k)
    br, bc = (n, k) if tb else (k, n)
    Ast, A = _colmajor(torch, ar, ac, ar + 3, g)
    Bst, B = _colmajor(torch, br, bc, br + 1, g)
    Cst, Cv = _colmajor(torch, m, n, m + 2, g)
    C0 = Cv.clone()
    opA = A.T if ta else A
    opB = B.T if tb else B
    alpha, beta = 0.75, -0.5
    _lib.call("vl_dgemm", ctx.h, ta, tb, m, n, k, alpha, _lib.ptr(Ast), ar + 3, _lib.ptr(Bst), br + 1, beta,
              _lib.ptr(Cst), m + 2, None, 0)
    want = alpha * (opA @ opB) + beta * C0
    scale = (opA.abs() @ opB.abs()).max().item() + 1.0
    assert (Cv - want).abs().max().item() <= 1e-13 * scale


@pytest.mark.parametrize("k,n", [(70, 1000), (1000, 100000)])
def test_weighted_syrk_lower(env, k, n):
    """M = L^T diag(w) L, lower triangle only, L stored n x k row-major (the
    pivoted-Cholesky factor's layout): column-major (k x n, ld k)."""
    torch, _lib, ctx = env
    g = torch.Generator(device="cuda").manual_seed(k)
    L = torch.randn(n, k, dtype=torch.float64, device="cuda", generator=g)
    w = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.1
    M = torch.full((k, k), 7.0, dtype=torch.float64, device="cuda")  # column-major storage of M^T
    _lib.call("vl_dgemm", ctx.h, 0, 1, k, k, n, 1.0, _lib.ptr(L), k, _lib.ptr(L), k, 0.0, _lib.ptr(M), k,
              _lib.ptr(w), 1)
    want = L.T @ (w[:, None] * L)
    got = M.T                                  # logical column-major view
    low = torch.tril(torch.ones(k, k, dtype=torch.bool, device="cuda"))
    assert ((got - want).abs()[low]).max().item() <= 1e-12 * want.abs().max().item()
    assert bool((got[~low] == 7.0).all())     # upper triangle untouched


@pytest.mark.parametrize("k", [1, 63, 64, 65, 300, 1000])
def test_trtri_lower(env, k):
    torch, _lib, ctx = env
    g = torch.Generator(device="cuda").manual_seed(k)
    A = torch.randn(k, k, dtype=torch.float64, device="cuda", generator=g)
    S = A @ A.T + k * torch.eye(k, dtype=torch.float64, device="cuda")
    Lrow = torch.linalg.cholesky(S)            # logical lower factor
    Lst = Lrow.T.contiguous()                  # column-major storage
    Li = torch.full((k, k), 3.0, dtype=torch.float64, device="cuda")
    _lib.call("vl_dtrtri_lower", ctx.h, k, _lib.ptr(Lst), k, _lib.ptr(Li), k)
    Linv = Li.T
    assert bool((torch.triu(Linv, 1) == 0).all())
    eye = torch.eye(k, dtype=torch.float64, device="cuda")
    assert (Lrow @ Linv - eye).abs().max().item() <= 1e-12
    want = torch.linalg.solve_triangular(Lrow, eye, upper=False)
    assert (Linv - want).abs().max().item() <= 1e-12 * want.abs().max().item()
