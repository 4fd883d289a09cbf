"""Host-side pieces of the iterative kernels: Lanczos tridiagonals from the CG
coefficients, Gauss quadrature for SLQ, the control-variate STE combiner, and
the ProbeSet cache protocol.

Mirrors vlgp/iterative.py: Tridiag (47-92), ProbeSet (222-244), slq_logdet
(260-277), ste_grad_logdet (280-304).  The per-probe CG runs (the heavy part)
happen on the device; only t short coefficient sequences and 2-6 scalars per
probe come back to the host.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import eigh_tridiagonal

from .errors import BreakdownError, ConfigError

CG_TOL_DEFAULT = 10.0 ** (-1.5)
CG_MAX_ITER_DEFAULT = 1000


@dataclass
class Tridiag:
    """Symmetric tridiagonal matrix (diagonal, off-diagonal)."""

    diag: np.ndarray
    off: np.ndarray

    @property
    def order(self):
        return self.diag.shape[0]

    def eigh(self):
        if self.order == 0:
            return np.empty(0), np.empty((0, 0))
        if self.order == 1:
            return self.diag.copy(), np.ones((1, 1))
        if not (np.all(np.isfinite(self.diag)) and np.all(np.isfinite(self.off))):
            raise BreakdownError("non-finite Lanczos coefficients")
        try:
            return eigh_tridiagonal(self.diag, self.off)
        except np.linalg.LinAlgError:
            from scipy.linalg import eigh as dense_eigh
            try:
                return dense_eigh(self.dense())
            except np.linalg.LinAlgError as exc:
                raise BreakdownError(f"tridiagonal eigendecomposition failed: {exc}") from None

    def dense(self):
        T = np.diag(self.diag)
        if self.off.size:
            T += np.diag(self.off, 1) + np.diag(self.off, -1)
        return T

    def quadrature_logdet(self):
        """e_1^T log(T) e_1."""
        lam, V = self.eigh()
        if np.any(lam <= 0):
            raise BreakdownError(f"non-positive tridiagonal eigenvalue {lam.min():.3e} in SLQ")
        return float(np.sum(V[0, :] ** 2 * np.log(lam)))


def tridiag_from_cg(alphas, betas, iters):
    """Lanczos tridiagonal from the CG coefficients of one column:
    T_ll = 1/a_l + b_{l-1}/a_{l-1},  T_{l-1,l} = sqrt(b_{l-1})/a_{l-1}
    (iterative.py:155-158)."""
    dg, of = [], []
    a_prev, b_prev = 1.0, 0.0
    for l in range(iters):
        a = float(alphas[l])
        dg.append(1.0 / a + b_prev / a_prev)
        if l > 0:
            of.append(np.sqrt(b_prev) / a_prev)
        if l + 1 < iters:
            a_prev, b_prev = a, float(betas[l])
    return Tridiag(np.array(dg), np.array(of))


@dataclass
class ProbeSet:
    """Probe vectors z_i ~ N(0, P), one per column, plus per-probe caches.

    On this backend Z, solves and psolves live on the device (n x t, storage
    order); ``Z`` / ``solves`` / ``psolves`` give numpy views in factor order.
    """

    Z_dev: object
    seed: int
    precond_tag: str
    pattern: object = None
    solves_dev: object = None
    tridiags: list = field(default_factory=list)
    psolves_dev: object = None
    weights: np.ndarray | None = None
    iters: np.ndarray | None = None
    shard: tuple = (0, None)   # (first global probe column, global t) for sharded runs

    @property
    def t(self):
        return int(self.Z_dev.shape[1])

    @property
    def n(self):
        return int(self.Z_dev.shape[0])

    def _host(self, x):
        return None if x is None else self.pattern.from_dev(x)

    @property
    def Z(self):
        return self._host(self.Z_dev)

    @property
    def solves(self):
        return self._host(self.solves_dev)

    @property
    def psolves(self):
        return self._host(self.psolves_dev)


def slq_from_parts(weights, tridiags, t):
    """(1/t) sum_i w_i e1^T log(T_i) e1 (iterative.py:260-277)."""
    if len(tridiags) != len(weights):
        raise ConfigError("one tridiagonal per probe is required")
    total = 0.0
    for w, tri in zip(weights, tridiags):
        if tri.order == 0:
            continue
        total += float(w) * tri.quadrature_logdet()
    return total / t


def ste_combine(h, r, dP_trace):
    """c dP_trace + mean(h - c r), c = Cov(h, r)/Var(r) (iterative.py:293-304)."""
    h = np.asarray(h, dtype=float)
    t = h.shape[0]
    if r is None:
        return float(h.mean())
    r = np.asarray(r, dtype=float)
    var_r = float(np.var(r, ddof=1)) if t > 1 else 0.0
    if var_r < 1e-300:
        return float(h.mean())
    c = float(np.cov(h, r, ddof=1)[0, 1]) / var_r
    return float(c * dP_trace + np.mean(h - c * r))
