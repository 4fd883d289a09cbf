"""Vecchia factor on the device: ordering, neighbour sets, B/D build, products
and triangular solves.

Mirrors the reference module vlgp/vecchia.py (same function names, argument
meaning and errors): order_random (vecchia.py:39-43), find_neighbors (59-98),
build_factor (220-283), VecchiaFactor (139-217), factor_gradient (286-337),
apply_dprecision (340-354), quad_dprecision (357-361), make_factor (444-449).

The factor values live in HBM in the library's storage order; numpy views
(``B``, ``D``) are materialised on request only (tests, diagnostics).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from . import device as dev
from .covariance import K_RHO, K_SIGMA2, Locations
from .errors import ConfigError

#: storage orders of the device layout (vl_pattern_create order_kind)
ORDER_FACTOR, ORDER_SPATIAL, ORDER_LEVEL = 0, 1, 2
DEFAULT_ORDER = ORDER_SPATIAL


def order_random(n, seed):
    """Uniformly random permutation of [0, n), reproducible from ``seed``."""
    if n < 1:
        raise ConfigError("n must be >= 1")
    return np.random.default_rng(seed).permutation(n)


def _coords(locs):
    c = locs.coords if isinstance(locs, Locations) else np.atleast_2d(np.asarray(locs, dtype=float))
    if c.ndim == 2 and c.shape[0] == 1 and c.shape[1] > 1 and not isinstance(locs, Locations):
        # a single row of coordinates is ambiguous; the reference treats 1-D input as one point
        pass
    return np.ascontiguousarray(c, dtype=float)


def _knn_on_device(d, m, where):
    if where == "host":
        return False
    if where == "device":
        return True
    return 1 <= d <= 3 and m <= 256 and dev.torch().cuda.is_available()


def neighbor_array(locs, perm, m, n_threads=0, where="auto"):
    """Exact nearest-preceding neighbours as an (n, m) int32 array padded with -1
    (same definition as find_neighbors).  ``where``: "device" (the grid search
    kernels, knn.cu), "host" (the native multi-threaded grid search) or
    "auto" (device when a GPU is present and 1 <= d <= 3, m <= 256)."""
    if m < 0:
        raise ConfigError("m must be >= 0")
    xy = np.ascontiguousarray(_coords(locs)[np.asarray(perm, dtype=int)])
    n, d = xy.shape
    out = np.full((n, max(m, 0)), -1, dtype=np.int32)
    if m > 0 and n > 1:
        if _knn_on_device(d, m, where):
            _lib.call("vl_knn_previous_dev", dev.context().h, _lib.ptr(xy), n, d, m, _lib.ptr(out))
        else:
            _lib.call("vl_knn_previous", _lib.ptr(xy), n, d, m, _lib.ptr(out), int(n_threads))
    return out


def knn_query(train_coords, query_coords, m):
    """The min(m, n) nearest training points of every query point, nearest
    first, ties to the smaller training index (vecchia.py:411-421), on the
    device.  Returns (idx (n_q, take) int64, dmin (n_q,) distance to the nearest)."""
    train = np.ascontiguousarray(np.atleast_2d(np.asarray(train_coords, dtype=float)))
    q = np.ascontiguousarray(np.atleast_2d(np.asarray(query_coords, dtype=float)))
    n, d = train.shape
    if q.shape[1] != d:
        raise ConfigError("prediction coordinates must have the training dimension")
    if m < 1:
        raise ConfigError("prediction requires m >= 1")
    nq = q.shape[0]
    take = min(m, n)
    out = np.full((nq, take), -1, dtype=np.int32)
    dmin = np.empty(nq)
    if nq:
        _lib.call("vl_knn_query", dev.context().h, _lib.ptr(train), n, _lib.ptr(q), nq, d, take, _lib.ptr(out),
                  _lib.ptr(dmin))
    return out.astype(np.int64), dmin


def find_neighbors(locs, perm, m):
    """Nearest-preceding-neighbour sets along the permuted ordering.

    For permuted position i the set N(i) holds the min(i, m) points among
    positions 0..i-1 closest in Euclidean distance, ties broken by the
    smaller permuted index (vecchia.py:59-98).  Returns a list of int arrays.
    """
    nb = neighbor_array(locs, perm, m)
    return [row[row >= 0].astype(int) for row in nb]


def _as_nbr_array(neighbors, n):
    if isinstance(neighbors, np.ndarray) and neighbors.ndim == 2:
        return np.ascontiguousarray(neighbors, dtype=np.int32)
    if len(neighbors) != n:
        raise ConfigError("neighbor sets must have one entry per point")
    m = max((len(x) for x in neighbors), default=0)
    out = np.full((n, m), -1, dtype=np.int32)
    for i, x in enumerate(neighbors):
        out[i, : len(x)] = x
    return out


def _content_key(a):
    """Exact content digest of an array (shape, dtype and bytes)."""
    import hashlib
    a = np.ascontiguousarray(a)
    h = hashlib.blake2b(digest_size=16)
    h.update(repr((a.shape, a.dtype.str)).encode())
    h.update(a.reshape(-1).view(np.uint8))
    return h.hexdigest()


_FP_W = {}


def _coords_fingerprint(xy):
    """Cheap content fingerprint of a coordinate array (a fixed pseudo-random
    projection, ~1 ms at n = 1e6): detects coordinates that differ from the
    ones a Pattern was built from."""
    flat = np.ascontiguousarray(xy, dtype=float).reshape(-1)
    w = _FP_W.get(flat.size)
    if w is None:
        w = np.random.default_rng(0x5EED).uniform(0.5, 1.5, size=flat.size)
        _FP_W.clear()
        _FP_W[flat.size] = w
    return (xy.shape, float(flat @ w), float(flat[::7].sum()))


class Pattern:
    """Device-resident sparsity pattern + solve schedules (once per dataset)."""

    def __init__(self, xy, nbr, order_kind=DEFAULT_ORDER, ctx=None):
        self.ctx = ctx or dev.context()
        xy = np.ascontiguousarray(xy, dtype=float)
        nbr = np.ascontiguousarray(nbr, dtype=np.int32)
        self.coords_fp = _coords_fingerprint(xy)
        self.n, self.d = xy.shape
        self.m = nbr.shape[1] if nbr.ndim == 2 else 0
        if nbr.shape[0] != self.n:
            raise ConfigError("neighbor sets must have one entry per point")
        h = C.c_void_p()
        _lib.call("vl_pattern_create", self.ctx.h, self.n, self.d, self.m, _lib.ptr(xy),
                  _lib.ptr(nbr) if self.m else None, int(order_kind), C.byref(h))
        self.h = h
        self.nbr = nbr
        self.sperm = np.empty(self.n, dtype=np.int32)
        _lib.call("vl_pattern_perm", self.h, _lib.ptr(self.sperm))
        self.siperm = np.empty(self.n, dtype=np.int64)
        self.siperm[self.sperm] = np.arange(self.n)
        info = (C.c_int64 * 10)()
        _lib.call("vl_pattern_info", self.h, info)
        self.head_levels, self.head_rows = int(info[8]), int(info[9])
        self.nnz_off = int(info[3])
        self.n_levels = int(info[4])
        self.n_levels_T = int(info[5])
        self.max_children = int(info[6])
        self._sperm_t = None

    def solve_order(self, transpose=False):
        """Storage rows in the order the multi-column solves walk them when x does not fit
        in L2 (tile-blocked topological order, csrc/pattern.cpp); empty when the pattern
        keeps the level order."""
        ln = C.c_int64(0)
        _lib.call("vl_pattern_solve_order", self.h, int(bool(transpose)), C.byref(ln), None)
        out = np.empty(ln.value, dtype=np.int32)
        if ln.value:
            _lib.call("vl_pattern_solve_order", self.h, int(bool(transpose)), C.byref(ln), _lib.ptr(out))
        return out

    def max_count(self):
        """Largest neighbour count (VecchiaFactor.m), computed once per pattern."""
        if getattr(self, "_max_count", None) is None:
            self._max_count = int((self.nbr >= 0).sum(axis=1).max()) if self.m else 0
        return self._max_count

    # factor-order numpy <-> storage-order device tensors
    def to_dev(self, v):
        """Permute to storage order into a pinned staging buffer and copy H2D
        asynchronously on the library stream."""
        v = np.asarray(v, dtype=float)
        T = dev.torch()
        key = v.shape
        ent = self._staging.get(key) if hasattr(self, "_staging") else None
        if not hasattr(self, "_staging"):
            self._staging = {}
        if ent is None:
            ent = [T.empty(key, dtype=T.float64, pin_memory=True), None]
            self._staging[key] = ent
        buf, ev = ent
        if ev is not None:
            ev.synchronize()          # previous copy out of this buffer finished
        np.take(v, self.sperm, axis=0, out=buf.numpy())
        out = buf.to(self.ctx.tdev, non_blocking=True)
        ev = T.cuda.Event()
        ev.record()
        ent[1] = ev
        return out

    def from_dev(self, x):
        a = dev.download(x)
        out = np.empty_like(a)
        out[self.sperm] = a
        return out

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().vl_pattern_destroy(self.h)
        except Exception:
            pass


_PATTERNS = []  # small LRU of (content key, Pattern)


def pattern_for(xy, neighbors, order_kind=DEFAULT_ORDER):
    """Device pattern for (coords, neighbour sets), reused across theta when the
    same coordinates and neighbour sets come back (keyed on their full
    contents, so an in-place edit of either builds a fresh pattern)."""
    nbr = _as_nbr_array(neighbors, xy.shape[0])
    key = (_content_key(xy), _content_key(nbr), order_kind)
    for ent in _PATTERNS:
        if ent[0] == key:
            return ent[1]
    pat = Pattern(xy, nbr, order_kind)
    _PATTERNS.append((key, pat))
    del _PATTERNS[:-4]
    return pat


@dataclass
class VecchiaGradient:
    """theta_k-derivatives of the factor: dB (pattern of B's off-diagonal), dD."""

    dB: sp.csr_matrix
    dD: np.ndarray
    k: int


class VecchiaFactor:
    """Device-resident Vecchia factor (B, D) with d/d theta (vecchia.py:139-217)."""

    def __init__(self, coords, spec, neighbors, perm, pattern, handle, m):
        self.coords = coords
        self.spec = spec
        self._neighbors = neighbors
        self._perm = None if perm is None else np.asarray(perm, dtype=int)
        self._iperm = None
        self.pattern = pattern
        self.h = handle
        self.m = m
        self.cache = {}
        self._B = None
        self._D = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                _lib.lib().vl_factor_destroy(self.h)
        except Exception:
            pass

    # perm / iperm (vecchia.py:139-217 attributes), materialised on first use
    @property
    def perm(self):
        if self._perm is None:
            self._perm = np.arange(self.pattern.n)
        return self._perm

    @property
    def iperm(self):
        if self._iperm is None:
            self._iperm = np.argsort(self.perm)
        return self._iperm

    @property
    def ctx(self):
        return self.pattern.ctx

    @property
    def n(self):
        return self.pattern.n

    @property
    def neighbors(self):
        nb = self._neighbors
        if isinstance(nb, np.ndarray):
            nb = [row[row >= 0].astype(int) for row in nb]
            self._neighbors = nb
        return nb

    def _get(self, which, size):
        out = np.empty(size, dtype=float)
        _lib.call("vl_factor_get", self.ctx.h, self.h, which, _lib.ptr(out))
        return out

    def _to_factor_order(self, a):
        out = np.empty_like(a)
        out[self.pattern.sperm] = a
        return out

    def set_values(self, B=None, D=None):
        """Replay externally computed factor values (factor-order CSR with the
        reference layout, diagonal last) into the device factor."""
        P = self.pattern
        if D is not None:
            Ds = np.ascontiguousarray(np.asarray(D, dtype=float)[P.sperm])
            _lib.call("vl_factor_set", self.ctx.h, self.h, 0, _lib.ptr(Ds))
            self._D = np.asarray(D, dtype=float).copy()
        if B is not None and P.m:
            B = B.tocsr()
            n, m = self.n, P.m
            ell = np.zeros((n, m))
            cnt = np.diff(B.indptr) - 1
            for i in range(n):
                lo = B.indptr[i]
                ell[i, :cnt[i]] = B.data[lo:lo + cnt[i]]
            ell = np.ascontiguousarray(ell[P.sperm])
            _lib.call("vl_factor_set", self.ctx.h, self.h, 3, _lib.ptr(ell))
            self._B = None

    @property
    def D(self):
        if self._D is None:
            self._D = self._to_factor_order(self._get(0, self.n))
        return self._D

    def _ell_csr(self, which):
        P = self.pattern
        n, m = self.n, P.m
        vals = self._get(which, n * m).reshape(n, m) if m else np.zeros((n, 0))
        vals = vals[P.siperm]  # factor order rows
        nbr = P.nbr
        cnt = (nbr >= 0).sum(axis=1) if m else np.zeros(n, dtype=int)
        indptr = np.zeros(n + 1, dtype=np.int64)
        indptr[1:] = np.cumsum(cnt + 1)
        indices = np.empty(indptr[-1], dtype=np.int64)
        data = np.empty(indptr[-1])
        mask = np.zeros((n, m + 1), dtype=bool)
        if m:
            mask[:, :m] = nbr >= 0
        # diagonal slot placed right after the last neighbour
        mask_diag = np.zeros((n, m + 1), dtype=bool)
        mask_diag[np.arange(n), cnt] = True
        full_idx = np.concatenate([nbr.astype(np.int64), np.zeros((n, 1), np.int64)], axis=1)
        full_val = np.concatenate([vals, np.zeros((n, 1))], axis=1)
        full_idx[mask_diag] = np.arange(n)
        full_val[mask_diag] = 1.0 if which == 3 else 0.0
        keep = mask | mask_diag
        indices[:] = full_idx[keep]
        data[:] = full_val[keep]
        return sp.csr_matrix((data, indices, indptr), shape=(n, n))

    @property
    def B(self):
        """B as scipy CSR in factor order, diagonal last (vecchia.py:272-282)."""
        if self._B is None:
            self._B = self._ell_csr(3)
        return self._B

    @property
    def _B_csc(self):
        return self.B.tocsc()

    # --- products / solves on numpy inputs (compatibility surface) ----------
    def _apply(self, name, v, *args):
        v = np.asarray(v, dtype=float)
        vec = v.ndim == 1
        V = v[:, None] if vec else v
        outs = []
        for c0 in range(0, V.shape[1], 128):  # the kernels take <= 128 columns per call
            blk = np.ascontiguousarray(V[:, c0:c0 + 128])
            t = blk.shape[1]
            x = self.pattern.to_dev(blk)
            y = dev.empty(self.ctx, self.n, t)
            _lib.call(name, self.ctx.h, self.h, *args, t, _lib.ptr(x), _lib.ptr(y))
            outs.append(self.pattern.from_dev(y))
        out = np.concatenate(outs, axis=1) if outs else np.zeros_like(V)
        return out[:, 0] if vec else out

    def B_matvec(self, v):
        return self._apply("vl_spmm", v, 0)

    def BT_matvec(self, v):
        return self._apply("vl_spmm", v, 1)

    def solve_B(self, v, transpose=False):
        """B^{-1} v, or B^{-T} v when ``transpose``; v may be a matrix."""
        return self._apply("vl_sptrsv", v, 1 if transpose else 0)

    def apply_precision(self, v):
        """(B^T D^{-1} B) v."""
        t = self.B_matvec(v)
        t = t / (self.D if t.ndim == 1 else self.D[:, None])
        return self.BT_matvec(t)

    def apply_sigma_tilde(self, v):
        """SigmaTilde v = B^{-1} D B^{-T} v."""
        x = self.solve_B(v, transpose=True)
        x = x * (self.D if x.ndim == 1 else self.D[:, None])
        return self.solve_B(x)

    def logdet_sigma_tilde(self):
        return float(np.log(self.D).sum())

    def dense_sigma_tilde(self):
        Binv = self.solve_B(np.eye(self.n))
        return (Binv * self.D) @ Binv.T


def build_factor(locs, spec, neighbors, perm=None, want_grad=True, order_kind=DEFAULT_ORDER):
    """Assemble the factor (B, D) -- and d/d theta -- on the device.

    Raises FactorizationError if a neighbour submatrix is not positive
    definite or D_i < 1e-10 * sigma2 (vecchia.py:220-283).
    """
    coords = _coords(locs)
    if perm is None:  # identity order: no host copy (the fit loop's per-theta call)
        xy = coords
    else:
        perm = np.asarray(perm, dtype=int)
        xy = np.ascontiguousarray(coords[perm])
    n = xy.shape[0]
    pat = neighbors if isinstance(neighbors, Pattern) else pattern_for(xy, neighbors, order_kind)
    if pat.n != n:
        raise ConfigError("neighbor sets must have one entry per point")
    if isinstance(neighbors, Pattern) and _coords_fingerprint(xy) != pat.coords_fp:
        # the factor is assembled from the pattern's device copy of the coordinates
        raise ConfigError("locations differ from the ones the Pattern was built from")
    m = pat.max_count()
    h = C.c_void_p()
    _lib.call("vl_factor_build", pat.ctx.h, pat.h, float(spec.sigma2), float(spec.rho), float(spec.nu),
              1 if want_grad else 0, C.byref(h))
    return VecchiaFactor(xy, spec, pat.nbr if isinstance(neighbors, Pattern) else neighbors, perm, pat, h, m)


def factor_gradient(factor, k):
    """d B / d theta_k and d D / d theta_k with the pattern of B (host copies)."""
    if k not in (K_SIGMA2, K_RHO):
        raise ConfigError(f"parameter index must be 0 or 1, got {k}")
    if k == K_SIGMA2:
        dB = factor.B.copy()
        dB.data = np.zeros_like(dB.data)
        return VecchiaGradient(dB, factor._to_factor_order(factor._get(1, factor.n)), k)
    return VecchiaGradient(factor._ell_csr(4), factor._to_factor_order(factor._get(2, factor.n)), k)


def make_factor(locs, spec, m, ordering_seed):
    """Convenience: random ordering, neighbour search, factor assembly."""
    locs = locs if isinstance(locs, Locations) else Locations(locs)
    perm = order_random(locs.n, ordering_seed)
    neighbors = neighbor_array(locs, perm, m)
    return build_factor(locs, spec, neighbors, perm)
