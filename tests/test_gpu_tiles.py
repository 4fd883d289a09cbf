"""Row order of the multi-column solves (csrc/pattern.cpp): the tile-blocked order is a
topological order of the dependency graph that holds every row outside the head block once,
and the solves that walk it (with the late dependencies listed last) agree with the oracle."""

import os

import numpy as np
import pytest

from oracle import vl_oracle as O

pytestmark = pytest.mark.gpu

ENV = {"VL_TILE_MIN_N": "0", "VL_TILE_MIN_ROWS": "256", "VL_TILE_MIN_MB": "0"}


def _pattern(xy, nbr, **env):
    from paper_2310_12000_b200.vecchia import Pattern
    env = {**ENV, **{k: str(v) for k, v in env.items()}}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return Pattern(xy, nbr, 1)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def pat_levels(nbr, transpose):
    """Dependency level (forward) or height (backward) of every factor row."""
    n = nbr.shape[0]
    lev = np.zeros(n, dtype=np.int64)
    if not transpose:
        for i in range(n):
            r = nbr[i][nbr[i] >= 0]
            if r.size:
                lev[i] = lev[r].max() + 1
    else:
        for i in range(n - 1, -1, -1):
            r = nbr[i][nbr[i] >= 0]
            if r.size:
                lev[r] = np.maximum(lev[r], lev[i] + 1)
    return lev


@pytest.fixture(scope="module")
def data():
    import paper_2310_12000_b200 as vg
    rng = np.random.default_rng(77)
    n, m = 30000, 20
    xy = rng.uniform(size=(n, 2))
    nbr = vg.vecchia.neighbor_array(xy, np.arange(n), m)
    return vg, xy, nbr


@pytest.mark.parametrize("K,S", [(4, 5), (64, 6), (1, 16)])
def test_tile_order_is_topological(data, K, S):
    vg, xy, nbr = data
    pat = _pattern(xy, nbr, VL_TILE_K=K, VL_TILE_S=S)
    n = pat.n
    spos = pat.siperm                       # factor row -> storage position
    par = np.where(nbr >= 0, spos[np.maximum(nbr, 0)], -1)   # factor row x m: storage rows of the parents
    for transpose in (False, True):
        order = pat.solve_order(transpose)
        # runs of one level are padded to 32 positions with -1: the rows one warp takes
        # together (32 / G of them, from an aligned group) then share a level
        assert order.size % 32 == 0
        lvl = pat_levels(nbr, transpose)[pat.sperm]          # level / height by storage row
        grp = order.reshape(-1, 32)
        for g in grp[:: max(1, grp.shape[0] // 500)]:
            assert np.unique(lvl[g[g >= 0]]).size <= 1
        order = order[order >= 0]
        assert order.size == n - pat.head_rows
        assert np.unique(order).size == order.size
        pos = np.full(n, -1, dtype=np.int64)
        pos[order] = np.arange(order.size)
        child = np.repeat(spos[:, None], nbr.shape[1], axis=1)
        ok = (par >= 0) & (pos[np.maximum(par, 0)] >= 0) & (pos[child] >= 0)   # neither end in the head
        pp, pc = pos[par[ok]], pos[child[ok]]
        assert np.all(pc < pp) if transpose else np.all(pp < pc)
    # rows of the head block are exactly the ones left out
    assert np.count_nonzero(pos < 0) == pat.head_rows


@pytest.mark.parametrize("t", [3, 8, 13, 25, 50, 64])
def test_tile_order_solves_vs_oracle(data, t):
    vg, xy, nbr = data
    spec = vg.CovarianceSpec(1.0, 0.05, 1.5)
    pat = _pattern(xy, nbr, VL_TILE_K=4, VL_TILE_S=5)
    assert pat.solve_order(False).size > 0
    f = vg.vecchia.build_factor(xy, spec, pat)
    flat = vg.vecchia.build_factor(xy, spec, _pattern(xy, nbr, VL_TILE_K=0, VL_CHILD_LATE=0))
    assert flat.pattern.solve_order(False).size == 0
    fo = O.Factor(xy, nbr, 1.0, 0.05, 1.5, f.B, f.D)
    X = np.random.default_rng(t).standard_normal((xy.shape[0], t))
    for tr in (False, True):
        got, lvl, want = f.solve_B(X, tr), flat.solve_B(X, tr), fo.solve_B(X, tr)
        assert np.abs(got - want).max() <= 1e-11 * np.abs(want).max()
        # same rows, same dependencies: only the summation order inside a row differs
        assert np.abs(got - lvl).max() <= 1e-13 * np.abs(want).max()
    # products read the factor in the reference's in-row order whatever the solve order is
    assert np.array_equal(f.B_matvec(X), flat.B_matvec(X))


def test_single_rhs_solves_with_late_dependencies_last(data):
    vg, xy, nbr = data
    spec = vg.CovarianceSpec(1.0, 0.05, 1.5)
    f = vg.vecchia.build_factor(xy, spec, _pattern(xy, nbr, VL_CHILD_LATE=16))
    flat = vg.vecchia.build_factor(xy, spec, _pattern(xy, nbr, VL_CHILD_LATE=0))
    fo = O.Factor(xy, nbr, 1.0, 0.05, 1.5, f.B, f.D)
    x = np.random.default_rng(3).standard_normal(xy.shape[0])
    for tr in (False, True):
        want = fo.solve_B(x, tr)
        assert np.abs(f.solve_B(x, tr) - want).max() <= 1e-11 * np.abs(want).max()
        assert np.abs(f.solve_B(x, tr) - flat.solve_B(x, tr)).max() <= 1e-13 * np.abs(want).max()
    assert np.abs(f.BT_matvec(x) - fo.BTmul(x)).max() <= 1e-12 * np.abs(x).max()
