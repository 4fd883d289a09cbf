"""CPU oracle for the Vecchia-Laplace hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy/scipy, the algorithm of the reference
package ``vlgp`` (arXiv 2310.12000, /root/reference/pkg/src/vlgp) for the
path that the CUDA library replaces: Vecchia factor (B, D) and its
theta-derivatives, VADU/LRAC-preconditioned CG with Lanczos-tridiagonal
capture, damped-Newton mode finding, SLQ log-determinant and the
control-variate STE gradient.  Each function cites the reference file:line it
follows.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``cpu_baseline`` / ``--impl reference``) may import it, and only as the
checker or the timed CPU arm -- never as the thing measured or shipped.  The
product package ``paper_2310_12000_b200`` never imports this file.

Parity pin: ``tests/golden/make_golden.py`` runs the reference itself (in the
build container, where /root/reference exists) and stores its outputs as
fixtures; ``tests/test_oracle_golden.py`` checks this restatement against
them.  The arithmetic of the reference lives in scipy/numpy (SuperLU,
sparsetools, LAPACK gesv/potrf/stemr, cKDTree -- versions unpinned upstream,
``pkg/pyproject.toml:10-13``); this oracle calls the same library routines so
it reproduces the reference to rounding.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
from scipy.linalg import cho_factor, cho_solve, eigh_tridiagonal, solve_triangular
from scipy.sparse.linalg import splu
from scipy.spatial import cKDTree
from scipy.special import expit, log_ndtr, gammaln, digamma

SQRT3 = np.sqrt(3.0)
SQRT5 = np.sqrt(5.0)


class OracleError(Exception):
    """Base for oracle-side failures (mirrors vlgp.errors classes by .kind)."""

    kind = "numerical"


class OracleFactorizationError(OracleError):
    kind = "factorization"


class OracleBreakdownError(OracleError):
    kind = "breakdown"


class OracleConvergenceError(OracleError):
    kind = "convergence"

    def __init__(self, msg, last_state=None):
        super().__init__(msg)
        self.last_state = last_state


# --------------------------------------------------------------------------
# Matern kernel (covariance.py:93-124)
# --------------------------------------------------------------------------

def matern(r, sigma2, rho, nu):
    """covariance.py:93-102"""
    r = np.asarray(r, dtype=float)
    if nu == 0.5:
        return sigma2 * np.exp(-r / rho)
    if nu == 1.5:
        u = (SQRT3 / rho) * r
        return sigma2 * (1.0 + u) * np.exp(-u)
    u = (SQRT5 / rho) * r
    return sigma2 * (1.0 + u + u * u / 3.0) * np.exp(-u)


def matern_drho(r, sigma2, rho, nu):
    """d/d rho of the kernel (covariance.py:105-124, k = K_RHO)."""
    r = np.asarray(r, dtype=float)
    if nu == 0.5:
        u = r / rho
        return sigma2 * np.exp(-u) * u / rho
    if nu == 1.5:
        u = (SQRT3 / rho) * r
        return sigma2 * u * u * np.exp(-u) / rho
    u = (SQRT5 / rho) * r
    return sigma2 * u * u * (1.0 + u) * np.exp(-u) / (3.0 * rho)


# --------------------------------------------------------------------------
# Ordering and neighbour sets (vecchia.py:39-98)
# --------------------------------------------------------------------------

def random_order(n, seed):
    """vecchia.py:39-43"""
    return np.random.default_rng(seed).permutation(n)


def _closest_earlier(dist, i, m):
    """m smallest of dist[:i], ties -> lower index (vecchia.py:46-56)."""
    k = min(i, m)
    if k == i:
        cand = np.arange(i)
    else:
        part = np.argpartition(dist, k - 1)[:k]
        cand = np.flatnonzero(dist <= dist[part].max())
    return cand[np.lexsort((cand, dist[cand]))][:k]


def knn_previous(xy, m, brute_max=4096, workers=1):
    """Nearest-preceding neighbour sets on already-permuted coords.

    Returns an (n, m) int64 array padded with -1 (row i holds min(i, m)
    entries, nearest first).  Brute force below ``brute_max`` rows, windowed
    kd-tree above (vecchia.py:59-98); ``workers`` threads for the tree query
    (cKDTree's own parallel query; the selection is identical).
    """
    xy = np.atleast_2d(np.asarray(xy, dtype=float))
    n = xy.shape[0]
    out = np.full((n, max(m, 0)), -1, dtype=np.int64)
    if m == 0 or n == 1:
        return out
    nb = min(n, brute_max)
    for i in range(1, nb):
        d = np.sqrt(((xy[:i] - xy[i]) ** 2).sum(axis=1))
        # cdist computes sqrt(sum diff^2) per pair as well
        sel = _closest_earlier(d, i, m)
        out[i, : sel.size] = sel
    if nb < n:
        tree = cKDTree(xy)
        todo = np.arange(nb, n)
        k = min(n, 2 * m + 16)
        while todo.size:
            dd, ii = tree.query(xy[todo], k=k, workers=workers)
            earlier = ii < todo[:, None]
            ok = (earlier.sum(axis=1) >= m) | (k >= n)
            rows = np.flatnonzero(ok)
            if rows.size:
                # vectorised form of the per-row lexsort((cand, dist)) over the
                # earlier candidates: stable sort by index, then stable by distance
                ci = np.where(earlier[rows], ii[rows], n)
                cd = np.where(earlier[rows], dd[rows], np.inf)
                o = np.argsort(ci, axis=1, kind="stable")
                ci, cd = np.take_along_axis(ci, o, 1), np.take_along_axis(cd, o, 1)
                o = np.argsort(cd, axis=1, kind="stable")
                ci = np.take_along_axis(ci, o, 1)[:, :m]
                take = np.minimum(todo[rows], m)
                ci[np.arange(m)[None, :] >= take[:, None]] = -1
                ci[ci >= n] = -1
                out[todo[rows]] = ci
            todo = todo[~ok]
            k = min(n, 2 * k)
    return out


def nbr_lists(nbr):
    """(n, m) padded array -> list of int arrays (reference representation)."""
    return [row[row >= 0].astype(int) for row in np.asarray(nbr)]


def nbr_array(lists, m=None):
    """list of int arrays -> (n, m) padded int64 array."""
    n = len(lists)
    if m is None:
        m = max((len(x) for x in lists), default=0)
    out = np.full((n, m), -1, dtype=np.int64)
    for i, x in enumerate(lists):
        out[i, : len(x)] = x
    return out


# --------------------------------------------------------------------------
# Factor (vecchia.py:101-127, 220-337)
# --------------------------------------------------------------------------

@dataclass
class Factor:
    xy: np.ndarray          # permuted coords (n, d)
    nbr: np.ndarray         # (n, m) padded with -1
    sigma2: float
    rho: float
    nu: float
    B: sp.csr_matrix        # unit lower triangular, diag last in each row
    D: np.ndarray
    _lu: object = None
    grads: list = field(default_factory=list)   # [(dB, dD) for sigma2, rho]
    cache: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.D.shape[0]

    @property
    def lu(self):
        if self._lu is None:
            # vecchia.py:159-170: SuperLU, natural ordering, no pivoting
            self._lu = splu(self.B.tocsc(), permc_spec="NATURAL", diag_pivot_thresh=0.0,
                            options={"SymmetricMode": False})
        return self._lu

    def solve_B(self, v, transpose=False):
        """vecchia.py:172-174"""
        return self.lu.solve(np.asarray(v, dtype=float), trans="T" if transpose else "N")

    def Bmul(self, v):
        return self.B @ np.asarray(v, dtype=float)

    def BTmul(self, v):
        return self.B.T @ np.asarray(v, dtype=float)

    def precision(self, v):
        """B^T D^-1 B v (vecchia.py:176-183)"""
        t = self.B @ np.asarray(v, dtype=float)
        t = t / (self.D if t.ndim == 1 else self.D[:, None])
        return self.B.T @ t

    def sigma_tilde(self, v):
        """B^-1 D B^-T v (vecchia.py:185-192)"""
        x = self.solve_B(v, transpose=True)
        x = x * (self.D if x.ndim == 1 else self.D[:, None])
        return self.solve_B(x)


def _blocks(xy, nb_idx, pts, sigma2, rho, nu):
    """Kernel blocks for a batch of rows (vecchia.py:101-112)."""
    P = xy[nb_idx]
    dif = P[:, :, None, :] - P[:, None, :, :]
    r_nn = np.sqrt(np.einsum("cjkd,cjkd->cjk", dif, dif))
    dx = P - pts[:, None, :]
    r_ni = np.sqrt(np.einsum("cjd,cjd->cj", dx, dx))
    return matern(r_nn, sigma2, rho, nu), matern(r_ni, sigma2, rho, nu), r_nn, r_ni


def vecchia_factor(xy, nbr, sigma2, rho, nu, chunk=2048, d_floor_rel=1e-10):
    """Build B and D (vecchia.py:220-283): A = K^-1 k by LU, Cholesky only as
    a positive-definiteness check, D = sigma2 - k.A, CSR row = [-A, 1]."""
    xy = np.atleast_2d(np.asarray(xy, dtype=float))
    nbr = np.asarray(nbr)
    n = xy.shape[0]
    cnt = (nbr >= 0).sum(axis=1) if nbr.size else np.zeros(n, int)
    D = np.full(n, float(sigma2))
    A_rows = [None] * n
    for j in np.unique(cnt):
        if j == 0:
            continue
        ids = np.flatnonzero(cnt == j)
        for a in range(0, ids.size, chunk):
            rows = ids[a:a + chunk]
            nb = nbr[rows, :j]
            K, k, _, _ = _blocks(xy, nb, xy[rows], sigma2, rho, nu)
            try:
                np.linalg.cholesky(K)
            except np.linalg.LinAlgError:
                for loc in range(rows.size):
                    try:
                        np.linalg.cholesky(K[loc])
                    except np.linalg.LinAlgError:
                        raise OracleFactorizationError(
                            f"neighbour covariance of row {rows[loc]} not PD") from None
                raise
            A = np.linalg.solve(K, k[..., None])[..., 0]
            D[rows] = sigma2 - np.einsum("cj,cj->c", k, A)
            for loc, i in enumerate(rows):
                A_rows[i] = A[loc]
    bad = np.flatnonzero(D < d_floor_rel * sigma2)
    if bad.size:
        raise OracleFactorizationError(f"D_{int(bad[0])} = {D[bad[0]]:.3e} below floor")
    indptr = np.concatenate([[0], np.cumsum(cnt + 1)])
    indices = np.empty(indptr[-1], dtype=np.int64)
    data = np.empty(indptr[-1])
    for i in range(n):
        lo, hi = indptr[i], indptr[i + 1]
        indices[lo:hi - 1] = nbr[i, :cnt[i]]
        data[lo:hi - 1] = -A_rows[i] if cnt[i] else []
        indices[hi - 1] = i
        data[hi - 1] = 1.0
    B = sp.csr_matrix((data, indices, indptr), shape=(n, n))
    return Factor(xy, nbr, float(sigma2), float(rho), float(nu), B, D)


def vecchia_grads(f, chunk=2048):
    """[(dB, dD)] for (sigma2, rho) -- vecchia.py:286-337.  dB keeps B's
    pattern; off-diagonals written positionally (diagonal last)."""
    if f.grads:
        return f.grads
    n = f.n
    nbr = f.nbr
    cnt = (nbr >= 0).sum(axis=1) if nbr.size else np.zeros(n, int)
    dB0 = f.B.copy()
    dB0.data = np.zeros_like(dB0.data)
    g_sig = (dB0, f.D / f.sigma2)
    dD = np.full(n, float(matern_drho(0.0, f.sigma2, f.rho, f.nu)))
    dA_rows = [None] * n
    for j in np.unique(cnt):
        if j == 0:
            continue
        ids = np.flatnonzero(cnt == j)
        for a in range(0, ids.size, chunk):
            rows = ids[a:a + chunk]
            nb = nbr[rows, :j]
            K, k, r_nn, r_ni = _blocks(f.xy, nb, f.xy[rows], f.sigma2, f.rho, f.nu)
            dK = matern_drho(r_nn, f.sigma2, f.rho, f.nu)
            dk = matern_drho(r_ni, f.sigma2, f.rho, f.nu)
            A = np.linalg.solve(K, k[..., None])[..., 0]
            rhs = dk - np.einsum("cjk,ck->cj", dK, A)
            dA = np.linalg.solve(K, rhs[..., None])[..., 0]
            dD[rows] += -np.einsum("cj,cj->c", dA, k) - np.einsum("cj,cj->c", A, dk)
            for loc, i in enumerate(rows):
                dA_rows[i] = dA[loc]
    data = np.zeros_like(f.B.data)
    for i in range(n):
        lo, hi = f.B.indptr[i], f.B.indptr[i + 1]
        if cnt[i]:
            data[lo:hi - 1] = -dA_rows[i]
    dB1 = sp.csr_matrix((data, f.B.indices.copy(), f.B.indptr.copy()), shape=(n, n))
    f.grads = [g_sig, (dB1, dD)]
    return f.grads


def dprec_apply(f, g, V):
    """(dQ) V, dQ = dB^T D^-1 B + B^T D^-1 dB - B^T D^-1 dD D^-1 B
    (vecchia.py:340-354)."""
    dB, dD = g
    V = np.asarray(V, dtype=float)
    c = (slice(None), None) if V.ndim == 2 else slice(None)
    BV = f.B @ V
    dBV = dB @ V
    out = dB.T @ (BV / f.D[c])
    out += f.B.T @ (dBV / f.D[c])
    out -= f.B.T @ ((dD / f.D ** 2)[c] * BV)
    return out


def dprec_quad(f, g, v):
    """v^T dQ v (vecchia.py:357-361)"""
    dB, dD = g
    Bv = f.B @ v
    dBv = dB @ v
    return float(2.0 * (dBv / f.D) @ Bv - (dD / f.D ** 2) @ Bv ** 2)


# --------------------------------------------------------------------------
# Likelihoods (likelihoods.py:62-174)
# --------------------------------------------------------------------------

_LOG_SQRT_2PI = 0.5 * np.log(2.0 * np.pi)


class Lik:
    def __init__(self, family, shape=1.0):
        if family not in ("bernoulli-logit", "bernoulli-probit", "gamma", "poisson"):
            raise ValueError(family)
        self.family = family
        self.shape = float(shape)

    @property
    def n_xi(self):
        return 1 if self.family == "gamma" else 0

    def logdens(self, y, mu):
        if self.family == "bernoulli-logit":          # likelihoods.py:72-74
            return y * mu - np.logaddexp(0.0, mu)
        if self.family == "bernoulli-probit":         # likelihoods.py:104-106
            return log_ndtr((2.0 * y - 1.0) * mu)
        if self.family == "poisson":                  # test-registered family (make_golden.register_poisson)
            return y * mu - np.exp(mu) - gammaln(y + 1.0)
        a = self.shape                                # likelihoods.py:150-158
        return a * np.log(a) - gammaln(a) + (a - 1.0) * np.log(y) - a * mu - a * y * np.exp(-mu)

    def derivs(self, y, mu):
        """(sum log p, d1, d2, d3)"""
        if self.family == "bernoulli-logit":          # likelihoods.py:76-82
            p = expit(mu)
            w = p * (1.0 - p)
            d1, d2, d3 = y - p, -w, -w * (1.0 - 2.0 * p)
        elif self.family == "bernoulli-probit":       # likelihoods.py:108-115
            z = 2.0 * y - 1.0
            u = z * mu
            g = np.exp(-0.5 * u * u - _LOG_SQRT_2PI - log_ndtr(u))
            d1 = z * g
            d2 = -g * (u + g)
            d3 = z * g * ((u + g) ** 2 + g * (u + g) - 1.0)
        elif self.family == "poisson":
            e = np.exp(mu)
            d1, d2, d3 = y - e, -e, -e
        else:                                         # likelihoods.py:160-166
            a = self.shape
            w = a * y * np.exp(-mu)
            d1, d2, d3 = -a + w, -w, w
        return float(self.logdens(y, mu).sum()), d1, d2, d3

    def xi_derivs(self, y, mu):
        """likelihoods.py:164-170 (gamma) / 51-57 (others)"""
        n = len(np.atleast_1d(mu))
        if self.family != "gamma":
            return np.empty(0), np.empty((0, n)), np.empty((0, n))
        a = self.shape
        e = y * np.exp(-mu)
        dl = np.array([np.sum(np.log(a) + 1.0 - digamma(a) + np.log(y) - mu - e)])
        return dl, (-1.0 + e)[None, :], (-e)[None, :]


# --------------------------------------------------------------------------
# PCG with tridiagonal capture (iterative.py:104-178)
# --------------------------------------------------------------------------

@dataclass
class CGOut:
    u: np.ndarray
    iters: int
    res: float
    converged: bool
    diag: np.ndarray | None = None
    off: np.ndarray | None = None
    alphas: list | None = None
    betas: list | None = None


def pcg(matvec, b, psolve, tol, max_iter=1000, capture=False):
    """Algorithm 2 of the paper; stopping rule ||r|| < tol ||b||."""
    b = np.asarray(b, dtype=float)
    n = b.shape[0]
    nb = float(np.linalg.norm(b))
    if nb == 0.0:
        return CGOut(np.zeros(n), 0, 0.0, True, np.empty(0), np.empty(0), [], [])
    if psolve is None:
        psolve = lambda r: r.copy()  # noqa: E731
    u = np.zeros(n)
    r = b.copy()
    z = psolve(r)
    h = z.copy()
    rz = float(r @ z)
    dg, of, al, be = [], [], [], []
    a_prev, b_prev = 1.0, 0.0
    its, conv, res = 0, False, nb
    for l in range(max_iter):
        v = matvec(h)
        hv = float(h @ v)
        if hv <= 0.0:
            raise OracleBreakdownError(f"h^T A h = {hv:.3e}")
        alpha = rz / hv
        u += alpha * h
        r -= alpha * v
        res = float(np.linalg.norm(r))
        al.append(alpha)
        if capture:
            dg.append(1.0 / alpha + b_prev / a_prev)
            if l > 0:
                of.append(np.sqrt(b_prev) / a_prev)
        its = l + 1
        if res < tol * nb:
            conv = True
            break
        z = psolve(r)
        rzn = float(r @ z)
        if rzn <= 0.0:
            raise OracleBreakdownError(f"r^T z = {rzn:.3e}")
        beta = rzn / rz
        be.append(beta)
        rz = rzn
        h = z + beta * h
        a_prev, b_prev = alpha, beta
    return CGOut(u, its, res, conv, np.array(dg) if capture else None,
                 np.array(of) if capture else None, al, be)


def tridiag_logquad(diag, off):
    """e1^T log(T) e1 (iterative.py:56-92)."""
    k = diag.shape[0]
    if k == 0:
        return 0.0
    if k == 1:
        lam, V = diag.copy(), np.ones((1, 1))
    else:
        if not (np.all(np.isfinite(diag)) and np.all(np.isfinite(off))):
            raise OracleBreakdownError("non-finite Lanczos coefficients")
        try:
            lam, V = eigh_tridiagonal(diag, off)
        except np.linalg.LinAlgError:
            from scipy.linalg import eigh
            T = np.diag(diag) + np.diag(off, 1) + np.diag(off, -1)
            lam, V = eigh(T)
    if np.any(lam <= 0):
        raise OracleBreakdownError("non-positive Ritz value")
    return float(np.sum(V[0, :] ** 2 * np.log(lam)))


# --------------------------------------------------------------------------
# Preconditioners (preconditioners.py:101-214, 249-320)
# --------------------------------------------------------------------------

class Vadu:
    """P = B^T diag(W + 1/D) B (preconditioners.py:101-132, 349-350)."""

    name = "vadu"

    def __init__(self, f, W):
        self.f = f
        self.d = W + 1.0 / f.D
        self.sd = np.sqrt(self.d)

    def _cs(self, v, s):
        return v * s if v.ndim == 1 else v * s[:, None]

    def solve(self, b):
        x = self.f.solve_B(b, transpose=True)
        return self.f.solve_B(self._cs(x, 1.0 / self.d))

    def logdet(self):
        return float(np.log(self.d).sum())

    def sample(self, G):
        return self.f.B.T @ self._cs(G, self.sd)


class Sandwich(Vadu):
    """P = B^T diag(d) B with d = 1/D (lva, preconditioners.py:351-352)."""

    def __init__(self, f, d, name):
        self.f = f
        self.d = d
        self.sd = np.sqrt(d)
        self.name = name


class Diagonal:
    """P = diag(d): diag (W + diag(B^T D^-1 B), preconditioners.py:134-158,
    353-354; _precision_diag 240-246) and identity (d = 1)."""

    def __init__(self, d, name):
        self.d = d
        self.sd = np.sqrt(d)
        self.name = name

    def solve(self, b):
        return b / self.d if b.ndim == 1 else b / self.d[:, None]

    def logdet(self):
        return float(np.log(self.d).sum())

    def sample(self, G):
        return G * self.sd[:, None]


def precision_diag(f):
    """diag(B^T D^-1 B) (PrecisionAccessor.diag, preconditioners.py:228-240)."""
    B = f.B.tocsr()
    rows = np.repeat(np.arange(f.n), np.diff(B.indptr))
    return np.bincount(B.indices, weights=B.data ** 2 / f.D[rows], minlength=f.n)


def pchol_sigma(xy, sigma2, rho, nu, k, tol=0.0):
    """Greedy pivoted Cholesky of the exact covariance (preconditioners.py:288-320)."""
    n = xy.shape[0]
    d = np.full(n, float(sigma2))
    L = np.zeros((n, k))
    piv = []
    for j in range(k):
        if d.min() < -1e-10:
            raise OracleFactorizationError("pivoted Cholesky lost PSD")
        np.clip(d, 0.0, None, out=d)
        if d.sum() <= tol:
            return L[:, :j], np.array(piv, dtype=int)
        p = int(np.argmax(d))
        if d[p] <= 0.0:
            return L[:, :j], np.array(piv, dtype=int)
        row = matern(np.sqrt(((xy - xy[p]) ** 2).sum(axis=1)), sigma2, rho, nu)
        col = row - L[:, :j] @ L[p, :j]
        col /= np.sqrt(d[p])
        col[p] = np.sqrt(d[p])
        L[:, j] = col
        d -= col ** 2
        d[p] = 0.0
        piv.append(p)
    return L, np.array(piv, dtype=int)


class Lrac:
    """P = L L^T + diag(1/W), Woodbury (preconditioners.py:167-214)."""

    name = "lrac"

    def __init__(self, L, piv, W):
        self.U = L
        self.piv = piv
        self.e = 1.0 / W
        M = np.eye(L.shape[1]) + L.T @ (L * W[:, None])
        self.M_cho = cho_factor(M, lower=True)
        self.logdet_M = 2.0 * float(np.log(np.diag(self.M_cho[0])).sum())

    def _cs(self, v, s):
        return v * s if v.ndim == 1 else v * s[:, None]

    def solve(self, b):
        x = self._cs(b, 1.0 / self.e)
        w = cho_solve(self.M_cho, self.U.T @ x)
        return x - self._cs(self.U @ w, 1.0 / self.e)

    def logdet(self):
        return float(np.log(self.e).sum()) + self.logdet_M

    def sample(self, G_n, G_k):
        return self._cs(G_n, np.sqrt(self.e)) + self.U @ G_k


class LowRank(Lrac):
    """P = U U^T + diag(e) for pchol-precision / rowsel (e = W) and l2 (k = 0,
    e = diag(SigmaTilde) + 1/W) (preconditioners.py:161-214, 353-379)."""

    def __init__(self, U, e, name, piv=None):
        if np.any(e <= 0) or not np.all(np.isfinite(e)):
            raise OracleFactorizationError(f"{name} diagonal part must be positive and finite")
        self.U = U
        self.piv = piv
        self.e = e
        self.name = name
        M = np.eye(U.shape[1]) + U.T @ (U / e[:, None])
        self.M_cho = cho_factor(M, lower=True) if U.shape[1] else (np.zeros((0, 0)), True)
        self.logdet_M = 2.0 * float(np.log(np.diag(self.M_cho[0])).sum()) if U.shape[1] else 0.0

    def solve(self, b):
        if self.U.shape[1] == 0:
            return self._cs(b, 1.0 / self.e)
        return super().solve(b)


def pchol_precision(f, k, tol=0.0):
    """Pivoted Cholesky of B^T D^-1 B (PrecisionAccessor, preconditioners.py:228-246, 288-320)."""
    B = f.B.tocsr()
    Bc = f.B.tocsc()
    d = precision_diag(f).copy()
    n = f.n
    L = np.zeros((n, k))
    piv = []
    for j in range(k):
        if d.min() < -1e-10:
            raise OracleFactorizationError("pivoted Cholesky lost PSD")
        np.clip(d, 0.0, None, out=d)
        if d.sum() <= tol:
            return L[:, :j], np.array(piv, dtype=int)
        p = int(np.argmax(d))
        if d[p] <= 0.0:
            return L[:, :j], np.array(piv, dtype=int)
        col = np.zeros(n)
        col[Bc.indices[Bc.indptr[p]:Bc.indptr[p + 1]]] = Bc.data[Bc.indptr[p]:Bc.indptr[p + 1]]
        row = B.T @ (col / f.D)
        c = (row - L[:, :j] @ L[p, :j]) / np.sqrt(d[p])
        c[p] = np.sqrt(d[p])
        L[:, j] = c
        d -= c ** 2
        d[p] = 0.0
        piv.append(p)
    return L, np.array(piv, dtype=int)


def rowsel_U(f, k):
    """U = B_S^T D_S^-1/2 over the k rows with the largest sum_j B_ij^2 / D_i (preconditioners.py:323-335, 372-379)."""
    B = f.B.tocsr()
    scores = np.add.reduceat(B.data ** 2, B.indptr[:-1]) / f.D
    order = np.lexsort((np.arange(f.n), -scores))
    S = np.sort(order[:k])
    return (B[S].T @ sp.diags(1.0 / np.sqrt(f.D[S]))).toarray(), S


def diag_sigma_tilde(f):
    """vecchia.py:198-212"""
    X = f.solve_B(np.eye(f.n), transpose=True)
    return np.einsum("j,jc->c", f.D, X ** 2)


# --------------------------------------------------------------------------
# Laplace objective (laplace.py:51-580)
# --------------------------------------------------------------------------

@dataclass
class Cfg:
    """Subset of BackendConfig (laplace.py:51-84)."""

    preconditioner: str = "vadu"
    t: int = 50
    cg_tol: float = 10.0 ** (-1.5)
    cg_max_iter: int = 1000
    probe_seed: int = 0
    rank: int | None = None
    newton_max_iter: int = 100
    newton_grad_tol: float = 1e-6
    newton_obj_tol: float = 1e-8
    workers: int = 1          # host processes for the independent probe solves (not a reference knob)

    @property
    def split(self):
        return "eq7" if self.preconditioner in ("lrac", "l2") else "eq6"

    @property
    def mode_tol(self):
        return min(self.cg_tol, 1e-4)

    def k(self, n):
        if self.rank is not None:
            return self.rank
        return int(np.clip(np.ceil(200 * min(1.0, n / 1e4)), 20, 200))


@dataclass
class Mode:
    b: np.ndarray
    W: np.ndarray
    y: np.ndarray
    F: np.ndarray
    logp: float
    d1: np.ndarray
    d3: np.ndarray
    quad: float
    objective: float
    newton_iters: int
    converged: bool
    cg_iters: list = field(default_factory=list)

    @property
    def mu(self):
        return self.F + self.b


def make_precond(f, W, cfg):
    """laplace.py:118-153 -> preconditioners.build (338-387)."""
    if cfg.preconditioner in ("vadu", "l1"):
        return Vadu(f, W)
    if cfg.preconditioner == "lva":
        return Sandwich(f, 1.0 / f.D, "lva")
    if cfg.preconditioner == "diag":
        return Diagonal(W + precision_diag(f), "diag")
    if cfg.preconditioner == "identity":
        return Diagonal(np.ones(f.n), "identity")
    if cfg.preconditioner in ("pchol-precision", "rowsel"):
        key = (cfg.preconditioner, cfg.k(f.n))
        if key not in f.cache:
            f.cache[key] = (pchol_precision(f, cfg.k(f.n)) if cfg.preconditioner == "pchol-precision"
                            else rowsel_U(f, cfg.k(f.n)))
        U, piv = f.cache[key]
        return LowRank(U, W.copy(), cfg.preconditioner, piv)
    if cfg.preconditioner == "l2":
        if "diag_st" not in f.cache:
            f.cache["diag_st"] = diag_sigma_tilde(f)
        return LowRank(np.zeros((f.n, 0)), f.cache["diag_st"] + 1.0 / W, "l2")
    if cfg.preconditioner == "lrac":
        if np.any(W <= 0):
            raise ValueError("lrac needs W > 0")
        key = ("pchol", cfg.k(f.n))
        if key not in f.cache:
            f.cache[key] = pchol_sigma(f.xy, f.sigma2, f.rho, f.nu, cfg.k(f.n))
        L, piv = f.cache[key]
        return Lrac(L, piv, W)
    raise ValueError(cfg.preconditioner)


def system_matvec(f, W, split):
    """laplace.py:156-165"""
    if split == "eq7":
        return lambda v: f.sigma_tilde(v) + v / W
    return lambda v: W * v + f.precision(v)


def solve_sys(f, W, P, rhs, cfg, tol, capture=False):
    """laplace.py:168-182"""
    op = system_matvec(f, W, cfg.split)
    if cfg.split == "eq7":
        res = pcg(op, f.sigma_tilde(rhs), P.solve, tol, cfg.cg_max_iter, capture)
        return res.u / W, res
    res = pcg(op, rhs, P.solve, tol, cfg.cg_max_iter, capture)
    return res.u, res


def newton_mode(f, lik, y, F, cfg):
    """Damped Newton (laplace.py:204-287)."""
    y = np.asarray(y, dtype=float)
    F = np.asarray(F, dtype=float)
    n = f.n
    b = np.zeros(n)
    logp, d1, d2, d3 = lik.derivs(y, F + b)
    quad = 0.0
    obj = -logp
    gnorm = float(np.abs(d1).max())
    conv = False
    it = 0
    safety = 1.0
    cg_its = []
    for it in range(1, cfg.newton_max_iter + 1):
        W = np.maximum(-d2, 0.0)
        rhs = W * b + d1
        rn = float(np.linalg.norm(rhs))
        tol = cfg.mode_tol
        if rn > 0.0:
            tol = min(tol, max(safety * 0.25 * gnorm / rn, 1e-14))
        P = make_precond(f, W, cfg)
        bn, res = solve_sys(f, W, P, rhs, cfg, tol)
        cg_its.append(res.iters)
        delta = bn - b
        step, ok = 1.0, False
        for _ in range(11):
            bt = b + step * delta
            lt = float(lik.logdens(y, F + bt).sum())
            qt = float(bt @ f.precision(bt))
            ot = -lt + 0.5 * qt
            if ot <= obj + 1e-12 * (1.0 + abs(obj)):
                ok = True
                break
            step *= 0.5
        if not ok:
            break
        dobj = obj - ot
        b, obj, quad = bt, ot, qt
        logp, d1, d2, d3 = lik.derivs(y, F + b)
        gprev = gnorm
        gnorm = float(np.abs(d1 - f.precision(b)).max())
        if gnorm > 0.5 * gprev:
            safety = max(0.2 * safety, 1e-10)
        if gnorm < cfg.newton_grad_tol and dobj < cfg.newton_obj_tol * (1.0 + abs(obj)):
            conv = True
            break
    else:
        it = cfg.newton_max_iter
    W = np.maximum(-d2, 0.0)
    st = Mode(b, W, y, F, logp, d1, d3, float(b @ f.precision(b)), obj, it, conv, cg_its)
    if not conv:
        g = float(np.abs(d1 - f.precision(b)).max())
        if g >= cfg.newton_grad_tol:
            raise OracleConvergenceError("Newton did not converge", last_state=st)
        st.converged = True
    return st


@dataclass
class Probes:
    Z: np.ndarray
    G: np.ndarray | None = None
    Gk: np.ndarray | None = None
    solves: np.ndarray | None = None
    psolves: np.ndarray | None = None
    tri: list = field(default_factory=list)      # [(diag, off)]
    iters: list = field(default_factory=list)
    alphas: list = field(default_factory=list)
    betas: list = field(default_factory=list)

    @property
    def t(self):
        return self.Z.shape[1]


def base_normals(n, t, seed):
    """The probe base draws of preconditioners.py:121-122 / iterative.py:251-252."""
    return np.random.default_rng(seed).standard_normal((n, t))


def make_probes(f, st, cfg, Z=None):
    """laplace.py:312-315 -> iterative.py:247-257 -> P.sample_block."""
    P = make_precond(f, st.W, cfg)
    if Z is not None:
        return Probes(np.asarray(Z, dtype=float)), P
    rng = np.random.default_rng(cfg.probe_seed)
    if cfg.preconditioner not in ("lrac", "pchol-precision", "rowsel", "l2"):
        G = rng.standard_normal((f.n, cfg.t))
        return Probes(P.sample(G), G=G), P
    Gn = rng.standard_normal((f.n, cfg.t))
    Gk = rng.standard_normal((P.U.shape[1], cfg.t))
    return Probes(P.sample(Gn, Gk), G=Gn, Gk=Gk), P


_PAR = None   # (op, Z, psolve, tol, max_iter) inherited by forked probe workers


def _probe_column(i):
    from threadpoolctl import threadpool_limits
    op, Z, psolve, tol, max_iter = _PAR
    with threadpool_limits(1):
        res = pcg(op, Z[:, i], psolve, tol, max_iter, capture=True)
    return i, res


def probe_solves(f, st, P, cfg, pr, workers=None):
    """laplace.py:290-309: one capped-tolerance PCG per probe column.  With
    ``workers`` > 1 the (independent) columns are distributed over forked
    processes -- the same per-column arithmetic, results placed by column."""
    global _PAR
    if pr.solves is not None:
        return
    workers = cfg.workers if workers is None else workers
    op = system_matvec(f, st.W, cfg.split)
    U = np.empty_like(pr.Z)
    out = [None] * pr.t
    if workers > 1 and pr.t > 1:
        import multiprocessing as mp
        _PAR = (op, pr.Z, P.solve, cfg.mode_tol, cfg.cg_max_iter)
        try:
            with mp.get_context("fork").Pool(min(workers, pr.t)) as pool:
                for i, res in pool.imap_unordered(_probe_column, range(pr.t)):
                    out[i] = res
        finally:
            _PAR = None
    else:
        for i in range(pr.t):
            out[i] = pcg(op, pr.Z[:, i], P.solve, cfg.mode_tol, cfg.cg_max_iter, capture=True)
    for i, res in enumerate(out):
        U[:, i] = res.u
        pr.tri.append((res.diag, res.off))
        pr.iters.append(res.iters)
        pr.alphas.append(res.alphas)
        pr.betas.append(res.betas)
    pr.solves = U


def slq(P, pr):
    """iterative.py:260-277"""
    if pr.psolves is None:
        pr.psolves = P.solve(pr.Z)
    w = np.einsum("it,it->t", pr.Z, pr.psolves)
    tot = 0.0
    for i, (dg, of) in enumerate(pr.tri):
        if dg.shape[0] == 0:
            continue
        tot += w[i] * tridiag_logquad(dg, of)
    return tot / pr.t


def logdet_sys(f, st, cfg, pr, P):
    """laplace.py:318-337 (iterative backend)"""
    probe_solves(f, st, P, cfg, pr)
    s = slq(P, pr)
    exact = float(np.log(st.W).sum()) if cfg.split == "eq7" else float(np.log(f.D).sum())
    return exact + P.logdet() + s


def nll(f, st, cfg, pr, P):
    """laplace.py:340-348"""
    return -st.logp + 0.5 * st.quad + 0.5 * logdet_sys(f, st, cfg, pr, P)


def dense_precision(f):
    return (f.B.T @ sp.diags(1.0 / f.D) @ f.B).toarray()


def nll_exact(f, st):
    """Cholesky backend log-det (laplace.py:320-324) -- small-n checker."""
    A = dense_precision(f)
    A[np.diag_indices_from(A)] += st.W
    c, _ = cho_factor(A, lower=True)
    ld = float(np.log(f.D).sum()) + 2.0 * float(np.log(np.diag(c)).sum())
    return -st.logp + 0.5 * st.quad + 0.5 * ld


def _cv_rows(H, R, t):
    """Per-row control-variate weights (laplace.py:401-411)."""
    if t < 2:
        return np.zeros(H.shape[0])
    hm = H.mean(axis=1, keepdims=True)
    rm = R.mean(axis=1, keepdims=True)
    vr = ((R - rm) ** 2).sum(axis=1) / (t - 1)
    cv = ((H - hm) * (R - rm)).sum(axis=1) / (t - 1)
    c = np.zeros(H.shape[0])
    ok = vr >= 1e-300
    c[ok] = cv[ok] / vr[ok]
    return c


def lrac_dL(f, P, k):
    """laplace.py:369-386"""
    L, piv = P.U, P.piv
    if k == 0:
        return L / (2.0 * f.sigma2)
    R = L[piv, :]
    r = np.sqrt(((f.xy[:, None, :] - f.xy[piv][None, :, :]) ** 2).sum(axis=2))
    dS = matern_drho(r, f.sigma2, f.rho, f.nu)
    dSpp = dS[piv, :]
    X = solve_triangular(R, dSpp, lower=True)
    X = solve_triangular(R, X.T, lower=True).T
    Phi = np.tril(X, -1) + 0.5 * np.diag(np.diag(X))
    dR = R @ Phi
    return solve_triangular(R, (dS - L @ dR.T).T, lower=True).T


def ste(pr, U, V, dA_op, dP_trace=0.0, dP_op=None, return_hr=False):
    """iterative.py:280-304"""
    t = pr.t
    h = np.einsum("it,it->t", U, dA_op(V))
    if dP_op is None:
        out = float(h.mean())
        return (out, h, None) if return_hr else out
    r = np.einsum("it,it->t", V, dP_op(V))
    vr = float(np.var(r, ddof=1)) if t > 1 else 0.0
    if vr < 1e-300:
        out = float(h.mean())
    else:
        c = float(np.cov(h, r, ddof=1)[0, 1]) / vr
        out = float(c * dP_trace + np.mean(h - c * r))
    return (out, h, r) if return_hr else out


def gradient(f, st, lik, X, cfg, pr, P, details=None):
    """Iterative-backend gradient (laplace.py:439-580) for vadu and lrac."""
    X = np.asarray(X, dtype=float)
    if X.ndim == 1:
        X = X[:, None]
    W, b, d1, md3 = st.W, st.b, st.d1, -st.d3
    grads = vecchia_grads(f)
    dl_xi, d2xi, d3xi = lik.xi_derivs(st.y, st.mu)
    probe_solves(f, st, P, cfg, pr)
    if pr.psolves is None:
        pr.psolves = P.solve(pr.Z)
    U, V = pr.solves, pr.psolves
    t = pr.t
    eq7 = cfg.split == "eq7"
    # d logdet / d mu (laplace.py:389-436)
    plain = cfg.preconditioner not in ("vadu", "l1", "lrac")
    if cfg.preconditioner in ("vadu", "l1"):
        H = U * V
        R = (f.B @ V) ** 2
        c = _cv_rows(H, R, t)
        dmu = md3 * (c / (W + 1.0 / f.D) + (H - c[:, None] * R).mean(axis=1))
    elif plain:                                       # laplace.py:433-436
        c = np.zeros(f.n)
        if eq7:
            dmu = md3 * (1.0 / W - (U * V / W[:, None] ** 2).mean(axis=1))
        else:
            dmu = md3 * (U * V).mean(axis=1)
    else:
        H = U * V / W[:, None] ** 2
        R = (V / W[:, None]) ** 2
        c = _cv_rows(H, R, t)
        G2 = np.einsum("ij,ji->i", P.U, cho_solve(P.M_cho, P.U.T))
        dmu = md3 * (1.0 / W + c * (G2 - 1.0 / W) - (H - c[:, None] * R).mean(axis=1))
    s = 0.5 * dmu
    tvec, tres = solve_sys(f, W, P, s, cfg, cfg.mode_tol)
    dtheta = np.empty(2)
    hr = []
    for k in (0, 1):
        g = grads[k]
        dB, dD = g
        if eq7:
            ex = 0.0

            def dA_op(Vv, g=g):
                SV = f.sigma_tilde(Vv)
                return -f.sigma_tilde(dprec_apply(f, g, SV))
        else:
            ex = float((dD / f.D).sum())

            def dA_op(Vv, g=g):
                return dprec_apply(f, g, Vv)
        if plain:
            dPt, dP_op = 0.0, None
        elif cfg.preconditioner in ("vadu", "l1"):
            dPt = -float((dD / (f.D * (f.D * W + 1.0))).sum())

            def dP_op(Vv, g=g):
                dB_, _ = g
                BV = f.B @ Vv
                dBV = dB_ @ Vv
                return dprec_apply(f, g, Vv) + dB_.T @ (BV * W[:, None]) + f.B.T @ (dBV * W[:, None])
        else:
            dL = lrac_dL(f, P, k)
            T1 = P.U.T @ (W[:, None] * dL)
            dPt = 2.0 * float(np.trace(cho_solve(P.M_cho, T1)))

            def dP_op(Vv, dL=dL):
                return dL @ (P.U.T @ Vv) + P.U @ (dL.T @ Vv)
        est, h, r = ste(pr, U, V, dA_op, dPt, dP_op, return_hr=True)
        hr.append((h, r, dPt, ex))
        dtheta[k] = 0.5 * dprec_quad(f, g, b) + 0.5 * (ex + est) - float(tvec @ dprec_apply(f, g, b))
    r_xi = dl_xi.shape[0]
    dxi = np.empty(r_xi)
    for l in range(r_xi):
        m3 = -d3xi[l]
        if eq7:
            ex = float((m3 / W).sum())

            def dA_op(Vv, m3=m3):
                return -(m3 / W ** 2)[:, None] * Vv
        else:
            ex = 0.0

            def dA_op(Vv, m3=m3):
                return m3[:, None] * Vv
        if plain:
            dPt, dP_op = 0.0, None
        elif cfg.preconditioner in ("vadu", "l1"):
            dPt = float((m3 / (W + 1.0 / f.D)).sum())

            def dP_op(Vv, m3=m3):
                return f.B.T @ (m3[:, None] * (f.B @ Vv))
        else:
            G2 = np.einsum("ij,ji->i", P.U, cho_solve(P.M_cho, P.U.T))
            dPt = float((G2 * m3).sum() - (m3 / W).sum())

            def dP_op(Vv, m3=m3):
                return -(m3 / W ** 2)[:, None] * Vv
        est = ste(pr, U, V, dA_op, dPt, dP_op)
        dxi[l] = -dl_xi[l] + 0.5 * (ex + est) + float(tvec @ d2xi[l])
    dF = -d1 + s - W * tvec
    if details is not None:
        details.update(s=s, tvec=tvec, cv=c, hr=hr, tvec_iters=tres.iters)
    return {"dtheta": dtheta, "dbeta": X.T @ dF, "dxi": dxi}


# --------------------------------------------------------------------------
# Whole evaluation (estimate.py:125-150)
# --------------------------------------------------------------------------

def evaluate(xy, nbr, y, F, X, sigma2, rho, nu, lik, cfg, want_grad=True, G=None):
    """One _Objective.evaluate in factor order: factor -> mode -> probes ->
    NLL -> gradient.  Returns (nll, grad dict, dict of intermediates)."""
    f = vecchia_factor(xy, nbr, sigma2, rho, nu)
    st = newton_mode(f, lik, y, F, cfg)
    if G is not None and cfg.preconditioner == "vadu":
        P = make_precond(f, st.W, cfg)
        pr = Probes(P.sample(G), G=G)
    else:
        pr, P = make_probes(f, st, cfg)
    val = nll(f, st, cfg, pr, P)
    info = {"factor": f, "state": st, "probes": pr, "P": P}
    if not want_grad:
        return val, None, info
    g = gradient(f, st, lik, X, cfg, pr, P, details=info)
    return val, g, info


# --------------------------------------------------------------------------
# Prediction (vecchia.py:364-441, predict.py:45-101)
# --------------------------------------------------------------------------

def prediction_blocks(train_xy_f, pred_xy, m, sigma2, rho, nu):
    """vecchia.py:393-441: each prediction point conditions on its min(m, n)
    nearest training points (factor order; ties to the smaller index);
    Bpo row = -K^-1 k (LU solve as the reference), Dp = sigma2 - k.A.
    Returns (nbr (n_p, take), Bpo values (n_p, take), Dp (n_p,))."""
    n = train_xy_f.shape[0]
    n_p = pred_xy.shape[0]
    take = min(m, n)
    nbr = np.empty((n_p, take), dtype=np.int64)
    vals = np.empty((n_p, take))
    Dp = np.empty(n_p)
    for q in range(n_p):
        d = np.sqrt(((train_xy_f - pred_xy[q]) ** 2).sum(axis=1))
        if d.min() <= 1e-12:
            raise ValueError(f"prediction point {q} duplicates a training point")
        idx = np.lexsort((np.arange(n), d))[:take]
        X = train_xy_f[idx]
        K = matern(np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(axis=2)), sigma2, rho, nu)
        k = matern(d[idx], sigma2, rho, nu)
        A = np.linalg.solve(K, k)
        nbr[q] = idx
        vals[q] = -A
        Dp[q] = sigma2 - k @ A
    return nbr, vals, Dp


def latent_mean(b, nbr, vals, Fp):
    """predict.py:45-50: omega = F_p - Bpo b*."""
    return Fp + (-(vals * b[nbr]).sum(axis=1))


def latent_var_sim(f, W, nbr, vals, Dp, s, seed, cg_tol, cg_max_iter=1000, full=False):
    """predict.py:70-101 with the VADU eq6 system: per sample z3 = W^1/2 z1 +
    B^T D^-1/2 z2 (z1, z2 drawn in that order from default_rng(seed)),
    u = (W + Q)^-1 z3 by PCG at cg_tol, z4 = Bpo u, acc += z4^2."""
    rng = np.random.default_rng(seed)
    n = f.n
    P = Vadu(f, W)
    op = system_matvec(f, W, "eq6")
    acc = np.zeros((len(Dp), len(Dp))) if full else np.zeros(len(Dp))
    for _ in range(s):
        z1 = rng.standard_normal(n)
        z2 = rng.standard_normal(n)
        z3 = np.sqrt(W) * z1 + f.B.T @ (z2 / np.sqrt(f.D))
        res = pcg(op, z3, P.solve, cg_tol, cg_max_iter)
        z4 = (vals * res.u[nbr]).sum(axis=1)
        acc = acc + (np.outer(z4, z4) if full else z4 ** 2)
    if full:
        return Dp + np.diag(acc) / s, np.diag(Dp) + acc / s
    return Dp + acc / s
