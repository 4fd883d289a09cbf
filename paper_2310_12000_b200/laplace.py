"""Mode finding, marginal likelihood and its gradient -- device backend.

Drop-in for the iterative backend of vlgp/laplace.py: same names, arguments,
return types and errors (BackendConfig 51-84, LaplaceState 87-102, find_mode
204-287, make_probes 312-315, neg_marginal_loglik 340-348, gradient
439-580).  Everything n-sized stays in HBM (storage order); the host sees
only scalars, t per-probe tridiagonals and the gradient.

Objective:  L = -log p(y | mu*) + 0.5 b*^T SigmaTilde^-1 b* + 0.5 log det(SigmaTilde W + I)
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np
from scipy.special import digamma

from . import _lib
from . import device as dev
from .errors import CapabilityError, ConfigError, ConvergenceError, FactorizationError
from .iterative import (CG_MAX_ITER_DEFAULT, CG_TOL_DEFAULT, ProbeSet, slq_from_parts, ste_combine,
                        tridiag_from_cg)

MODE_CG_TOL_CAP = 1e-4
EQ5_VARIANTS = ("lrac", "l2")
SUPPORTED_PRECONDITIONERS = ("vadu", "l1", "lva", "diag", "identity", "lrac", "pchol-precision", "rowsel", "l2")
# low-rank-plus-diagonal variants (Woodbury on the device, csrc/lrac.cu)
LOWRANK_VARIANTS = ("lrac", "pchol-precision", "rowsel", "l2")
# eq6 variants on the device (csrc/laplace.cu precond_dinv): sandwich B^T diag(d) B or diagonal diag(d)
EQ6_VARIANT_ID = {"vadu": 0, "l1": 1, "lva": 2, "diag": 3, "identity": 4}
CV_VARIANTS = ("vadu", "l1", "lrac")  # variants with a control variate in the gradient (laplace.py:414-431)


def default_rank(n):
    """Default low-rank size: 200 scaled by n/1e4, clamped to [20, 200] (preconditioners.py:390-392)."""
    return int(np.clip(np.ceil(200 * min(1.0, n / 1e4)), 20, 200))


@dataclass(frozen=True)
class BackendConfig:
    """How linear algebra is performed during likelihood evaluations."""

    backend: str = "iterative"
    preconditioner: str = "vadu"
    t: int = 50
    cg_tol: float = CG_TOL_DEFAULT
    cg_max_iter: int = CG_MAX_ITER_DEFAULT
    probe_seed: int = 0
    logdet_split: str = "auto"
    rank: int | None = None
    newton_max_iter: int = 100
    newton_grad_tol: float = 1e-6
    newton_obj_tol: float = 1e-8

    def __post_init__(self):
        if self.backend not in ("cholesky", "iterative"):
            raise ConfigError(f"unknown backend {self.backend!r}")
        if self.t < 1:
            raise ConfigError("t must be >= 1")
        if self.logdet_split not in ("auto", "eq6", "eq7"):
            raise ConfigError(f"unknown logdet split {self.logdet_split!r}")

    def resolved_split(self):
        if self.logdet_split != "auto":
            return self.logdet_split
        return "eq7" if self.preconditioner in EQ5_VARIANTS else "eq6"

    @property
    def mode_cg_tol(self):
        return min(self.cg_tol, MODE_CG_TOL_CAP)


def _check_supported(cfg):
    if cfg.backend != "iterative":
        raise CapabilityError("the device backend implements the iterative path; the dense 'cholesky' "
                              "backend is the reference's CPU oracle")
    if cfg.preconditioner not in SUPPORTED_PRECONDITIONERS:
        raise CapabilityError(f"preconditioner {cfg.preconditioner!r} is not available on the device backend "
                              f"(supported: {', '.join(SUPPORTED_PRECONDITIONERS)})")
    want = "eq7" if cfg.preconditioner in EQ5_VARIANTS else "eq6"
    if cfg.resolved_split() != want:
        raise CapabilityError(f"the device {cfg.preconditioner} path uses the {want} log-determinant split")


class LracFactorHandle:
    """Rank-k pivoted Cholesky of the exact covariance, cached on the factor
    like the reference's factor.cache[("sigma_pchol", k)] (laplace.py:128-136)."""

    def __init__(self, factor, k, tol=0.0, kind=0):
        # kind 0: pivoted Cholesky of Sigma (lrac); 1: of the precision (pchol-precision); 2: rowsel
        self.factor = factor
        self.k = int(k)
        piv = np.zeros(self.k, dtype=np.int32)
        keff = C.c_int(0)
        h = C.c_void_p()
        if kind == 0:
            _lib.call("vl_lrac_create", factor.ctx.h, factor.h, self.k, float(tol), C.byref(h), _lib.ptr(piv),
                      C.byref(keff))
        else:
            _lib.call("vl_lowrank_create", factor.ctx.h, factor.h, int(kind), self.k, float(tol), C.byref(h),
                      _lib.ptr(piv), C.byref(keff))
        self.h = h
        self.keff = int(keff.value)
        self.pivots = piv[: self.keff].astype(int)

    def L(self):
        """L (n x k) in factor order (numpy)."""
        f = self.factor
        out = np.empty((f.n, self.k))
        _lib.call("vl_lrac_get_L", f.ctx.h, self.h, _lib.ptr(out))
        res = np.empty_like(out)
        res[f.pattern.sperm] = out
        return res[:, : self.keff]

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().vl_lrac_destroy(self.h)
        except Exception:
            pass


def lrac_factor(factor, cfg):
    """The theta-only low-rank factor of the variant, cached on the factor
    (laplace.py:128-136): lrac -> Sigma's pivoted Cholesky, pchol-precision ->
    the precision's, rowsel -> B_S^T D_S^-1/2."""
    k = cfg.rank if cfg.rank is not None else default_rank(factor.n)
    kind = {"lrac": 0, "pchol-precision": 1, "rowsel": 2}[cfg.preconditioner]
    key = (("sigma_pchol", "prec_pchol", "rowsel")[kind], int(k))
    lf = factor.cache.get(key)
    if lf is None:
        lf = LracFactorHandle(factor, k, kind=kind)
        factor.cache[key] = lf
    return lf


def diag_sigma_tilde_dev(factor):
    """diag(SigmaTilde) on the device (vecchia.py:198-212), cached on the factor."""
    d = factor.cache.get("diag_sigma_tilde")
    if d is None:
        d = dev.empty(factor.ctx, factor.n, 1)
        _lib.call("vl_diag_sigma_tilde", factor.ctx.h, factor.h, _lib.ptr(d))
        factor.cache["diag_sigma_tilde"] = d
    return d


class LaplaceState:
    """Converged mode and everything the likelihood/gradient needs at it.

    Vectors live on the device (storage order); attribute access returns
    numpy arrays in factor order like the reference's dataclass.
    """

    def __init__(self, pattern, dev_vecs, y, F, logp, quad, objective, newton_iters, converged, cg_iters=()):
        self._pattern = pattern
        self._dev = dev_vecs          # b, W, d1, d3, y, F (device, storage order)
        self._y = y
        self._F = F
        self.logp = float(logp)
        self.quad = float(quad)
        self.objective = float(objective)
        self.newton_iters = int(newton_iters)
        self.converged = bool(converged)
        self.cg_iters = list(cg_iters)
        self._cache = {}

    def _host(self, key):
        v = self._cache.get(key)
        if v is None:
            v = self._pattern.from_dev(self._dev[key])[:, 0]
            self._cache[key] = v
        return v

    @property
    def b(self):
        return self._host("b")

    @property
    def W(self):
        return self._host("W")

    @property
    def d1(self):
        return self._host("d1")

    @property
    def d3(self):
        return self._host("d3")

    @property
    def y(self):
        return self._y

    @property
    def F(self):
        return self._F

    @property
    def mu(self):
        return self._F + self.b

    def with_converged(self, flag):
        s = LaplaceState(self._pattern, self._dev, self._y, self._F, self.logp, self.quad, self.objective,
                         self.newton_iters, flag, self.cg_iters)
        return s


def _col(pattern, v):
    return pattern.to_dev(np.asarray(v, dtype=float)[:, None])


def find_mode(factor, lik, y, F, cfg, trace=None):
    """Damped Newton iteration for the penalised-likelihood mode b*."""
    _check_supported(cfg)
    y = lik.validate(y)
    F = np.asarray(F, dtype=float)
    pat = factor.pattern
    ctx = factor.ctx
    n = factor.n
    y_d, F_d = _col(pat, y), _col(pat, F)
    b, W, d1, d3 = (dev.empty(ctx, n, 1) for _ in range(4))
    lk = _lib.VlLik(lik.family_id, float(lik.shape_param))
    nc = _lib.VlNewtonCfg(float(cfg.mode_cg_tol), int(cfg.cg_max_iter), int(cfg.newton_max_iter),
                          float(cfg.newton_grad_tol), float(cfg.newton_obj_tol),
                          EQ6_VARIANT_ID.get(cfg.preconditioner, 0))
    out = (C.c_double * 8)()
    cg_its = np.zeros(max(cfg.newton_max_iter, 1), dtype=np.int32)
    if cfg.preconditioner == "lrac":
        lf = lrac_factor(factor, cfg)
        st = _lib.lib().vl_find_mode_lrac(ctx.h, factor.h, lf.h, C.byref(lk), C.byref(nc), _lib.ptr(y_d),
                                          _lib.ptr(F_d), _lib.ptr(b), _lib.ptr(W), _lib.ptr(d1), _lib.ptr(d3), out,
                                          _lib.ptr(cg_its), int(cg_its.size))
    elif cfg.preconditioner in ("pchol-precision", "rowsel", "l2"):
        l2 = cfg.preconditioner == "l2"
        lf = None if l2 else lrac_factor(factor, cfg)
        dst = diag_sigma_tilde_dev(factor) if l2 else None
        st = _lib.lib().vl_find_mode_lowrank(ctx.h, factor.h, None if l2 else lf.h, 2 if l2 else 1,
                                             _lib.ptr(dst) if l2 else None, C.byref(lk), C.byref(nc),
                                             _lib.ptr(y_d), _lib.ptr(F_d), _lib.ptr(b), _lib.ptr(W), _lib.ptr(d1),
                                             _lib.ptr(d3), out, _lib.ptr(cg_its), int(cg_its.size))
    else:
        st = _lib.lib().vl_find_mode(ctx.h, factor.h, C.byref(lk), C.byref(nc), _lib.ptr(y_d), _lib.ptr(F_d),
                                     _lib.ptr(b), _lib.ptr(W), _lib.ptr(d1), _lib.ptr(d3), out,
                                     _lib.ptr(cg_its), int(cg_its.size))
    state = LaplaceState(pat, {"b": b, "W": W, "d1": d1, "d3": d3, "y": y_d, "F": F_d}, y, F,
                         out[0], out[1], out[2], int(out[4]), bool(out[5]), cg_its[: int(out[6])].tolist())
    if trace is not None:
        trace.append(state.objective)
    if st == 42:
        msg = _lib.lib().vl_last_error().decode()
        raise ConvergenceError(msg, last_state=state.with_converged(False))
    _lib.check(st)
    return state


class Eq6Preconditioner:
    """The eq6 preconditioners on the device (preconditioners.py:101-158,
    338-387): vadu / l1 (B^T diag(W + 1/D) B), lva (B^T diag(1/D) B), diag
    (diag(W + diag(B^T D^-1 B))) and identity.  ``dinv`` (device) holds 1/d
    of the sandwich or diagonal; ``pkind`` 0 = sandwich, 1 = diagonal."""

    def __init__(self, factor, W_dev, name="vadu"):
        self.factor = factor
        self.W_dev = W_dev
        self.name = name
        self.variant = EQ6_VARIANT_ID[name]
        self.pkind = 0 if self.variant <= 2 else 1
        self.dinv = dev.empty(factor.ctx, factor.n, 1)
        _lib.call("vl_precond_dinv", factor.ctx.h, factor.h, self.variant, _lib.ptr(W_dev), _lib.ptr(self.dinv))
        self._sums = None
        self._logdet = None

    def sums(self):
        if self._sums is None:
            out = np.zeros(6)
            _lib.call("vl_factor_sums", self.factor.ctx.h, self.factor.h, _lib.ptr(self.W_dev), _lib.ptr(out))
            self._sums = out
        return self._sums

    def logdet(self):
        if self._logdet is None:
            out = np.zeros(1)
            _lib.call("vl_sum_log", self.factor.ctx.h, self.factor.n, _lib.ptr(self.dinv), _lib.ptr(out))
            self._logdet = -float(out[0])
        return self._logdet


VaduPreconditioner = Eq6Preconditioner


class LracPreconditioner:
    """P = L L^T + diag(e) on the device (LowRankPlusDiagonalPreconditioner,
    preconditioners.py:161-214): lrac (L from Sigma, e = 1/W, eq7 system),
    pchol-precision / rowsel (e = W, eq6) and l2 (k = 0, e = diag(SigmaTilde)
    + 1/W, eq7; the reference's diagonal 'l2')."""

    def __init__(self, factor, W_dev, lf, name="lrac"):
        self.factor = factor
        self.W_dev = W_dev
        self.lf = lf
        self.name = name
        out = np.zeros(2)
        h = C.c_void_p()
        if name == "lrac":
            _lib.call("vl_lrac_prepare", factor.ctx.h, lf.h, _lib.ptr(W_dev), C.byref(h), _lib.ptr(out))
        else:
            self.einv = dev.empty(factor.ctx, factor.n, 1)
            kind = 2 if name == "l2" else 1
            dst = diag_sigma_tilde_dev(factor) if name == "l2" else None
            if name != "l2":
                nonpos = np.zeros(1)
                _lib.call("vl_sum_log", factor.ctx.h, factor.n, _lib.ptr(W_dev), _lib.ptr(nonpos))
                if not np.isfinite(nonpos[0]):
                    raise FactorizationError(f"{name} diagonal part must be positive and finite")
            _lib.call("vl_lowrank_einv", factor.ctx.h, factor.n, kind, _lib.ptr(W_dev),
                      _lib.ptr(dst) if dst is not None else None, _lib.ptr(self.einv))
            _lib.call("vl_lowrank_prepare", factor.ctx.h, factor.h, None if lf is None else lf.h, _lib.ptr(W_dev),
                      _lib.ptr(self.einv), 0 if name == "l2" else 1, C.byref(h), _lib.ptr(out))
        self.h = h
        self.logdet_M = float(out[0])
        self.sumlogW = float(out[1])  # sum log(1/e)
        self.pivots = lf.pivots if lf is not None else np.zeros(0, dtype=int)
        self._sums = None
        self._sumlogWop = None

    @property
    def sumlogWop(self):
        """sum log W of the system (the eq7 log-det split, laplace.py:335)."""
        if self._sumlogWop is None:
            if self.name == "lrac":
                self._sumlogWop = self.sumlogW
            else:
                out = np.zeros(1)
                _lib.call("vl_sum_log", self.factor.ctx.h, self.factor.n, _lib.ptr(self.W_dev), _lib.ptr(out))
                self._sumlogWop = float(out[0])
        return self._sumlogWop

    def logdet(self):
        return -self.sumlogW + self.logdet_M

    @property
    def k(self):
        return self.lf.keff if self.lf is not None else 0

    @property
    def U(self):
        return self.lf.L() if self.lf is not None else np.zeros((self.factor.n, 0))

    def sums(self):
        if self._sums is None:
            out = np.zeros(6)
            _lib.call("vl_factor_sums", self.factor.ctx.h, self.factor.h, _lib.ptr(self.W_dev), _lib.ptr(out))
            self._sums = out
        return self._sums

    def solve_dev(self, r_dev):
        z = dev.empty(self.factor.ctx, *r_dev.shape)
        _lib.call("vl_lrac_apply_inv", self.factor.ctx.h, self.h, int(r_dev.shape[1]), _lib.ptr(r_dev), _lib.ptr(z))
        return z

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().vl_lracw_destroy(self.h)
        except Exception:
            pass


def build_preconditioner(factor, W_dev, cfg):
    _check_supported(cfg)
    if cfg.preconditioner in LOWRANK_VARIANTS:
        lf = None if cfg.preconditioner == "l2" else lrac_factor(factor, cfg)
        return LracPreconditioner(factor, W_dev, lf, cfg.preconditioner)
    return Eq6Preconditioner(factor, W_dev, cfg.preconditioner)


_G_CACHE = []  # (pattern, seed, t, cols, tensor) -- SAA: same probes every evaluation


def base_normals(factor, seed, t, cols=None):
    """G = default_rng(seed).standard_normal((n, t)) in factor order (the
    reference's VADU sample_block draw, preconditioners.py:121-122), uploaded
    once and cached on the device (storage order).  ``cols`` selects a
    contiguous column shard (multi-GPU)."""
    pat = factor.pattern
    key = (seed, t, cols)
    for ent in _G_CACHE:
        if ent[0] is pat and ent[1] == key:
            return ent[2]
    G = np.random.default_rng(seed).standard_normal((factor.n, t))
    if cols is not None:
        G = G[:, cols[0]:cols[1]]
    Gd = pat.to_dev(np.ascontiguousarray(G))
    _G_CACHE.append((pat, key, Gd))
    del _G_CACHE[:-2]
    return Gd


def _lrac_normals(factor, seed, t, k, cols=None):
    """LRAC sample_block draws (preconditioners.py:204-207): g_n (n x t) then
    g_k (k x t) from one default_rng(seed) stream; cached on the device."""
    pat = factor.pattern
    key = ("lrac", seed, t, k, cols)
    for ent in _G_CACHE:
        if ent[0] is pat and ent[1] == key:
            return ent[2]
    rng = np.random.default_rng(seed)
    Gn = rng.standard_normal((factor.n, t))
    Gk = rng.standard_normal((k, t))
    if cols is not None:
        Gn, Gk = Gn[:, cols[0]:cols[1]], Gk[:, cols[0]:cols[1]]
    val = (pat.to_dev(np.ascontiguousarray(Gn)), dev.upload(factor.ctx, np.ascontiguousarray(Gk)) if k else None)
    _G_CACHE.append((pat, key, val))
    del _G_CACHE[:-2]
    return val


def make_probes(factor, state, cfg, cols=None):
    """Fresh N(0, P) probes for the current mode, deterministic in the seed."""
    P = build_preconditioner(factor, state._dev["W"], cfg)
    if cfg.preconditioner in LOWRANK_VARIANTS:
        Gn, Gk = _lrac_normals(factor, cfg.probe_seed, cfg.t, P.k, cols)
        t = int(Gn.shape[1])
        Z = dev.empty(factor.ctx, factor.n, t)
        V = dev.empty(factor.ctx, factor.n, t)
        w = np.zeros(t)
        _lib.call("vl_lrac_probes", factor.ctx.h, P.h, t, _lib.ptr(Gn), _lib.ptr(Gk) if P.k else None,
                  _lib.ptr(Z), _lib.ptr(V), _lib.ptr(w))
        ps = ProbeSet(Z, cfg.probe_seed, P.name, pattern=factor.pattern, psolves_dev=V, weights=w,
                      shard=(0 if cols is None else cols[0], cfg.t))
        return ps, P
    G = base_normals(factor, cfg.probe_seed, cfg.t, cols)
    t = int(G.shape[1])
    Z = dev.empty(factor.ctx, factor.n, t)
    V = dev.empty(factor.ctx, factor.n, t)
    w = np.zeros(t)
    _lib.call("vl_probes_eq6", factor.ctx.h, factor.h, _lib.ptr(P.dinv), P.pkind, t, _lib.ptr(G), _lib.ptr(Z),
              _lib.ptr(V), _lib.ptr(w))
    ps = ProbeSet(Z, cfg.probe_seed, P.name, pattern=factor.pattern, psolves_dev=V, weights=w,
                  shard=(0 if cols is None else cols[0], cfg.t))
    return ps, P


def _given_probes(factor, state, cfg, Zd, seed, cols):
    P = build_preconditioner(factor, state._dev["W"], cfg)
    if cfg.preconditioner in LOWRANK_VARIANTS:
        raise CapabilityError("caller-supplied probes are implemented for the eq6 (vadu-family) preconditioners")
    t = int(Zd.shape[1])
    V = dev.empty(factor.ctx, factor.n, t)
    w = np.zeros(t)
    _lib.call("vl_probes_given", factor.ctx.h, factor.h, _lib.ptr(P.dinv), P.pkind, t, _lib.ptr(Zd), _lib.ptr(V),
              _lib.ptr(w))
    shard = (0 if cols is None else cols[0], cfg.t if cols is not None else t)
    return ProbeSet(Zd, seed, P.name, pattern=factor.pattern, psolves_dev=V, weights=w, shard=shard), P


def probes_from_Z(factor, state, cfg, Z):
    """Inject caller-supplied probes (the reference's ``ProbeSet(Z, seed,
    P.name)`` passed to neg_marginal_loglik / gradient, laplace.py:340, 439;
    e.g. Rademacher probes).  Z is (n, t) in factor order; it is
    uploaded once and P^-1 Z and the SLQ weights z^T P^-1 z are formed on
    the device (two triangular solves, weights fused)."""
    Z = np.ascontiguousarray(np.asarray(Z, dtype=float))
    if Z.ndim != 2 or Z.shape[0] != factor.n:
        raise ConfigError(f"probes must have shape (n, t) with n = {factor.n}")
    return _given_probes(factor, state, cfg, factor.pattern.to_dev(Z), cfg.probe_seed, None)


def rademacher_probes(factor, state, cfg, seed=None, cols=None):
    """Probes with the preconditioner's covariance built from Rademacher base
    draws instead of Gaussian ones: Z = B^T (sqrt(d) o R) for the
    VADU-family sandwich (sqrt(d) o R for diagonal P), the same construction
    as sample_block (preconditioners.py:121-122) with R in place of G.  R is
    drawn on the device: entry (factor row i, column c) is -1 or +1 by the top
    bit of splitmix64(seed * 0x9E3779B97F4A7C15 + i * t + c); ``cols`` selects
    a column shard.  P^-1 Z and the SLQ weights follow as in make_probes."""
    if cfg.preconditioner in LOWRANK_VARIANTS:
        raise CapabilityError("Rademacher probes are implemented for the eq6 (vadu-family) preconditioners")
    seed = cfg.probe_seed if seed is None else int(seed)
    c0, c1 = (0, cfg.t) if cols is None else cols
    t = c1 - c0
    P = build_preconditioner(factor, state._dev["W"], cfg)
    R = dev.empty(factor.ctx, factor.n, t)
    _lib.call("vl_probes_rademacher", factor.ctx.h, factor.pattern.h, t, cfg.t, c0, seed & 0xFFFFFFFFFFFFFFFF,
              _lib.ptr(R))
    Z = dev.empty(factor.ctx, factor.n, t)
    V = dev.empty(factor.ctx, factor.n, t)
    w = np.zeros(t)
    _lib.call("vl_probes_eq6", factor.ctx.h, factor.h, _lib.ptr(P.dinv), P.pkind, t, _lib.ptr(R), _lib.ptr(Z),
              _lib.ptr(V), _lib.ptr(w))
    return ProbeSet(Z, seed, P.name, pattern=factor.pattern, psolves_dev=V, weights=w, shard=(c0, cfg.t)), P


def _run_probe_solves(factor, state, P, cfg, probes):
    """CG-solve every probe at mode_cg_tol, capturing tridiagonals (laplace.py:290-309)."""
    if probes.solves_dev is not None and len(probes.tridiags) == probes.t:
        return
    t = probes.t
    U = dev.empty(factor.ctx, factor.n, t)
    cap = int(cfg.cg_max_iter)
    its = np.zeros(t, dtype=np.int32)
    conv = np.zeros(t, dtype=np.int32)
    res = np.zeros(t)
    al = np.zeros((max(cap, 1), t))
    be = np.zeros((max(cap, 1), t))
    if cfg.preconditioner in LOWRANK_VARIANTS:
        _lib.call("vl_lrac_pcg", factor.ctx.h, P.h, t, _lib.ptr(probes.Z_dev), _lib.ptr(U), float(cfg.mode_cg_tol),
                  int(cfg.cg_max_iter), 1, _lib.ptr(its), _lib.ptr(conv), _lib.ptr(res), _lib.ptr(al), _lib.ptr(be),
                  max(cap, 1))
    else:
        _lib.call("vl_pcg_eq6", factor.ctx.h, factor.h, _lib.ptr(state._dev["W"]), _lib.ptr(P.dinv), P.pkind, t,
                  _lib.ptr(probes.Z_dev), _lib.ptr(U), float(cfg.mode_cg_tol), int(cfg.cg_max_iter), 1,
                  _lib.ptr(its), _lib.ptr(conv), _lib.ptr(res), _lib.ptr(al), _lib.ptr(be), max(cap, 1))
    probes.solves_dev = U
    probes.iters = its
    probes.tridiags = [tridiag_from_cg(al[:, c], be[:, c], int(its[c])) for c in range(t)]


def solve_system(factor, state, rhs_dev, cfg, tol=None, P=None):
    """u = (W + SigmaTilde^-1)^-1 rhs for device rhs (n x k): eq6 with VADU,
    or the eq7 form with LRAC (laplace.py:168-182)."""
    tol = cfg.cg_tol if tol is None else tol
    k = int(rhs_dev.shape[1])
    u = dev.empty(factor.ctx, factor.n, k)
    its = np.zeros(k, dtype=np.int32)
    if cfg.preconditioner in LOWRANK_VARIANTS:
        P = P if P is not None else build_preconditioner(factor, state._dev["W"], cfg)
        _lib.call("vl_lrac_solve_system", factor.ctx.h, P.h, k, _lib.ptr(rhs_dev), _lib.ptr(u), float(tol),
                  int(cfg.cg_max_iter), _lib.ptr(its))
        return u, its
    conv = np.zeros(k, dtype=np.int32)
    res = np.zeros(k)
    P = P if P is not None else build_preconditioner(factor, state._dev["W"], cfg)
    _lib.call("vl_pcg_eq6", factor.ctx.h, factor.h, _lib.ptr(state._dev["W"]), _lib.ptr(P.dinv), P.pkind, k,
              _lib.ptr(rhs_dev), _lib.ptr(u), float(tol), int(cfg.cg_max_iter), 0, _lib.ptr(its), _lib.ptr(conv),
              _lib.ptr(res), None, None, 1)
    return u, its


def slq_parts(probes):
    """Per-probe SLQ terms w_i e1^T log(T_i) e1 (summed by the caller)."""
    out = np.zeros(probes.t)
    for i, tri in enumerate(probes.tridiags):
        if tri.order:
            out[i] = float(probes.weights[i]) * tri.quadrature_logdet()
    return out


def logdet_system(factor, state, cfg, probes=None, P=None, comm=None):
    """log det(SigmaTilde W + I) = sum log D + log det P + SLQ (laplace.py:318-337)."""
    _check_supported(cfg)
    if P is None or probes is None:
        probes, P = make_probes(factor, state, cfg)
    if probes.precond_tag != P.name:
        raise ConfigError("probes were drawn against a different preconditioner")
    _run_probe_solves(factor, state, P, cfg, probes)
    parts = slq_parts(probes)
    if comm is not None:
        parts = comm.allgather_cols(parts, probes.shard)
    slq = float(sum(parts[i] for i in range(len(parts)))) / len(parts)
    if cfg.resolved_split() == "eq7":
        return P.sumlogWop + P.logdet() + slq
    sums = P.sums()
    return float(sums[0]) + P.logdet() + slq


def neg_marginal_loglik(state, factor, cfg, probes=None, P=None, comm=None):
    """Approximate negative log-marginal likelihood at the converged mode."""
    if not state.converged:
        raise ConvergenceError("state is not converged", last_state=state)
    return -state.logp + 0.5 * state.quad + 0.5 * logdet_system(factor, state, cfg, probes=probes, P=P, comm=comm)


def gradient(state, factor, lik, X, cfg, probes=None, P=None, comm=None):
    """Full gradient: d theta (2,), d beta (p,), d xi (r,) (laplace.py:439-580)."""
    if not state.converged:
        raise ConvergenceError("state is not converged", last_state=state)
    _check_supported(cfg)
    X = np.asarray(X, dtype=float)
    if X.ndim == 1:
        X = X[:, None]
    pat, ctx, n = factor.pattern, factor.ctx, factor.n
    if P is None or probes is None:
        probes, P = make_probes(factor, state, cfg)
    _run_probe_solves(factor, state, P, cfg, probes)
    dv = state._dev
    t = probes.t
    gamma = lik.n_xi > 0
    md3x = None
    if gamma:
        md3x = dev.empty(ctx, n, 1)
        junk = np.zeros(3)
        _lib.call("vl_gamma_xi_terms", ctx.h, factor.h, _lib.ptr(dv["y"]), _lib.ptr(dv["F"]), _lib.ptr(dv["b"]),
                  _lib.ptr(dv["W"]), _lib.ptr(dv["b"]), _lib.ptr(md3x), _lib.ptr(junk))
    s = dev.empty(ctx, n, 1)
    cols = np.zeros((4, t))
    xicols = np.zeros((2, t))
    if cfg.preconditioner in ("lrac", "l2"):
        return _gradient_lrac(state, factor, lik, X, cfg, probes, P, comm, md3x, s)
    plain = 0 if cfg.preconditioner in CV_VARIANTS else 1
    if comm is not None and (comm.world > 1 or getattr(comm, "force_split", False)):
        s, cols, xicols = comm.grad_probe_pass(factor, state, probes, md3x, plain=plain)
    else:
        _lib.call("vl_grad_probe_pass", ctx.h, factor.h, _lib.ptr(dv["W"]), _lib.ptr(dv["d3"]),
                  _lib.ptr(probes.solves_dev), _lib.ptr(probes.psolves_dev), t, _lib.ptr(s), _lib.ptr(cols),
                  _lib.ptr(md3x) if gamma else None, _lib.ptr(xicols) if gamma else None, plain)
    tvec, tvec_its = solve_system(factor, state, s, cfg, tol=cfg.mode_cg_tol, P=P)
    probes.tvec_iters = int(tvec_its[0])
    terms = np.zeros(4)
    _lib.call("vl_grad_scalar_terms", ctx.h, factor.h, _lib.ptr(dv["b"]), _lib.ptr(tvec), _lib.ptr(terms))
    sums = P.sums()
    dtheta = np.empty(2)
    for k in (0, 1):
        ex = float(sums[2 + k])
        dPt = float(sums[4 + k])
        h, r = cols[2 * k], cols[2 * k + 1]
        ste = ste_combine(h, None if plain else r, dPt)  # plain STE for variants without dP (laplace.py:509-536)
        dtheta[k] = 0.5 * terms[2 * k] + 0.5 * (ex + ste) - terms[2 * k + 1]
    dxi = np.empty(lik.n_xi)
    if gamma:
        g3 = np.zeros(3)
        _lib.call("vl_gamma_xi_terms", ctx.h, factor.h, _lib.ptr(dv["y"]), _lib.ptr(dv["F"]), _lib.ptr(dv["b"]),
                  _lib.ptr(dv["W"]), _lib.ptr(tvec), _lib.ptr(md3x), _lib.ptr(g3))
        a = lik.shape
        dlogp = n * (np.log(a) + 1.0 - digamma(a)) + g3[0]
        ste = ste_combine(xicols[0], None if plain else xicols[1], float(g3[2]))
        dxi[0] = -dlogp + 0.5 * (0.0 + ste) + g3[1]
    p = X.shape[1]
    dbeta = np.zeros(p)
    if p:
        Xd = pat.to_dev(np.ascontiguousarray(X))
        _lib.call("vl_grad_dbeta", ctx.h, n, _lib.ptr(dv["d1"]), _lib.ptr(s), _lib.ptr(dv["W"]), _lib.ptr(tvec),
                  _lib.ptr(Xd), p, _lib.ptr(dbeta))
    return {"dtheta": dtheta, "dbeta": dbeta, "dxi": dxi}


def _gradient_lrac(state, factor, lik, X, cfg, probes, P, comm, md3x, s):
    """eq7 + LRAC branch of laplace.py:439-580: d logdet/d mu with the LRAC
    control variate (421-431), dA_op = -SigmaTilde dQ SigmaTilde, ex = 0,
    dP from d L (369-386, 527-533); xi: ex = sum m3/W, dA = dP = -m3/W^2."""
    ctx, n, dv, t = factor.ctx, factor.n, state._dev, probes.t
    gamma = md3x is not None
    plain = 0 if cfg.preconditioner == "lrac" else 1
    if comm is not None and (comm.world > 1 or getattr(comm, "force_split", False)):
        s, hcols, rcols, dPt, xicols, xis = comm.lrac_grad_pass(factor, state, probes, P, md3x, plain=plain)
    else:
        hcols = np.zeros((2, t))
        rcols = np.zeros((2, t))
        dPt = np.zeros(2)
        xicols = np.zeros((2, t))
        xis = np.zeros(2)
        _lib.call("vl_lrac_grad", ctx.h, P.h, t, _lib.ptr(probes.solves_dev), _lib.ptr(probes.psolves_dev),
                  _lib.ptr(dv["d3"]), _lib.ptr(md3x) if gamma else None, _lib.ptr(s), _lib.ptr(hcols),
                  _lib.ptr(rcols), _lib.ptr(dPt), _lib.ptr(xicols), _lib.ptr(xis), plain)
    tvec, tvec_its = solve_system(factor, state, s, cfg, tol=cfg.mode_cg_tol, P=P)
    probes.tvec_iters = int(tvec_its[0])
    terms = np.zeros(4)
    _lib.call("vl_grad_scalar_terms", ctx.h, factor.h, _lib.ptr(dv["b"]), _lib.ptr(tvec), _lib.ptr(terms))
    dtheta = np.empty(2)
    for k in (0, 1):
        ste = ste_combine(hcols[k], None if plain else rcols[k], float(dPt[k]))
        dtheta[k] = 0.5 * terms[2 * k] + 0.5 * (0.0 + ste) - terms[2 * k + 1]
    dxi = np.empty(lik.n_xi)
    if gamma:
        g3 = np.zeros(3)
        _lib.call("vl_gamma_xi_terms", ctx.h, factor.h, _lib.ptr(dv["y"]), _lib.ptr(dv["F"]), _lib.ptr(dv["b"]),
                  _lib.ptr(dv["W"]), _lib.ptr(tvec), _lib.ptr(md3x), _lib.ptr(g3))
        a = lik.shape
        dlogp = n * (np.log(a) + 1.0 - digamma(a)) + g3[0]
        ex = float(xis[1])
        ste = ste_combine(xicols[0], None if plain else xicols[1], float(xis[0] - xis[1]))
        dxi[0] = -dlogp + 0.5 * (ex + ste) + g3[1]
    X = np.asarray(X, dtype=float)
    if X.ndim == 1:
        X = X[:, None]
    p = X.shape[1]
    dbeta = np.zeros(p)
    if p:
        Xd = factor.pattern.to_dev(np.ascontiguousarray(X))
        _lib.call("vl_grad_dbeta", ctx.h, n, _lib.ptr(dv["d1"]), _lib.ptr(s), _lib.ptr(dv["W"]), _lib.ptr(tvec),
                  _lib.ptr(Xd), p, _lib.ptr(dbeta))
    return {"dtheta": dtheta, "dbeta": dbeta, "dxi": dxi}
