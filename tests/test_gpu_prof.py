"""The in-library kernel profiler bench.py reads its live roofline from:
per-tag CUDA-event times, the tag filter (events only on one tag) and the
launch counter, which counts every launch either way."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _table(L, ctx):
    buf = C.create_string_buffer(1 << 16)
    nl = C.c_int64(0)
    assert L.vl_prof_report(ctx.h, buf, 1 << 16, C.byref(nl)) == 0
    rows = {}
    for ln in buf.value.decode().splitlines():
        tag, cnt, ms, by = ln.split("\t")
        rows[tag] = (int(cnt), float(ms), float(by))
    return rows, int(nl.value)


def test_tag_filter_and_launch_counter():
    import paper_2310_12000_b200 as vg
    from paper_2310_12000_b200 import _lib
    from paper_2310_12000_b200.vecchia import build_factor, neighbor_array
    rng = np.random.default_rng(3)
    n = 4000
    xy = rng.uniform(size=(n, 2))
    perm = vg.order_random(n, 1)
    f = build_factor(xy, vg.CovarianceSpec(1.0, 0.1, 1.5), neighbor_array(xy, perm, 10), perm, want_grad=False)
    lik = vg.get_likelihood("bernoulli-logit")
    y = (rng.uniform(size=n) < 0.5).astype(float)
    cfg = vg.BackendConfig(t=4)
    L = _lib.lib()
    L.vl_prof_enable.argtypes = [C.c_void_p, C.c_int]
    L.vl_prof_reset.argtypes = [C.c_void_p]
    L.vl_prof_only.argtypes = [C.c_void_p, C.c_char_p]
    L.vl_prof_report.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_int64)]
    ctx = f.ctx
    assert L.vl_prof_only(ctx.h, None) == 0
    assert L.vl_prof_reset(ctx.h) == 0 and L.vl_prof_enable(ctx.h, 1) == 0
    st = vg.find_mode(f, lik, y[perm], np.zeros(n), cfg)
    full, n_full = _table(L, ctx)
    assert "cg1_trsv_Bt" in full and "cg1_trsv_B" in full and n_full > 0
    assert full["cg1_trsv_Bt"][0] >= sum(st.cg_iters)   # one backward solve per CG iteration (+ initial residuals)
    # same work, events on one tag only: that tag's launch count is unchanged, nothing else is timed
    assert L.vl_prof_only(ctx.h, b"cg1_trsv_Bt") == 0 and L.vl_prof_reset(ctx.h) == 0
    vg.find_mode(f, lik, y[perm], np.zeros(n), cfg)
    only, n_only = _table(L, ctx)
    assert set(only) == {"cg1_trsv_Bt"}
    assert only["cg1_trsv_Bt"][0] == full["cg1_trsv_Bt"][0]
    assert n_only == n_full
    assert L.vl_prof_only(ctx.h, None) == 0 and L.vl_prof_enable(ctx.h, 0) == 0
