"""Diagnose the dependency-driven solve: per-row completion timestamps ->
per-level finish times and hop latency (row done - max(dep done))."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_12000_b200 as vg  # noqa: E402
from paper_2310_12000_b200 import _lib  # noqa: E402
from paper_2310_12000_b200.vecchia import Pattern, build_factor, neighbor_array  # noqa: E402

n, m = int(os.environ.get("KP_N", 1000000)), 20
xy = np.random.default_rng(0).uniform(size=(n, 2))
perm = np.random.default_rng(1).permutation(n)
nbr = neighbor_array(xy, perm, m)
xyp = np.ascontiguousarray(xy[perm])
pat = Pattern(xyp, nbr, 1)
f = build_factor(xyp, vg.CovarianceSpec(1.0, 0.02, 1.5), pat, want_grad=False)
L = _lib.lib()
L.vl_debug_set_tstamp.argtypes = [C.c_void_p, C.c_void_p]
ts = torch.zeros(n, dtype=torch.int64, device="cuda")
# levels in factor order
nb = nbr
TR = int(os.environ.get("KP_TR", "0"))
lev = np.zeros(n, dtype=np.int64)
if not TR:
    for i in range(n):
        row = nb[i][nb[i] >= 0]
        if row.size:
            lev[i] = lev[row].max() + 1
else:  # heights (levels of the B^T solve)
    for i in range(n - 1, -1, -1):
        row = nb[i][nb[i] >= 0]
        if row.size:
            lev[row] = np.maximum(lev[row], lev[i] + 1)
for t in [int(x) for x in os.environ.get("KP_TS", "1,50").split(",")]:
    X = torch.randn(n, t, dtype=torch.float64, device="cuda") / 20
    Y = torch.empty_like(X)
    _lib.call("vl_sptrsv", f.ctx.h, f.h, TR, t, _lib.ptr(X), _lib.ptr(Y))
    torch.cuda.synchronize()
    L.vl_debug_set_tstamp(f.ctx.h, C.c_void_p(ts.data_ptr()))
    _lib.call("vl_sptrsv", f.ctx.h, f.h, TR, t, _lib.ptr(X), _lib.ptr(Y))
    torch.cuda.synchronize()
    L.vl_debug_set_tstamp(f.ctx.h, None)
    tsf = np.empty(n, dtype=np.int64)
    tsf[pat.sperm] = ts.cpu().numpy()  # factor order
    t0 = tsf[tsf > 0].min()
    tsf = np.where(tsf > 0, tsf - t0, 0)
    nl = lev.max() + 1
    lev_end = np.full(nl, -1, dtype=np.int64)
    np.maximum.at(lev_end, lev, tsf)
    size = np.bincount(lev, minlength=nl)
    # hop latency: own done - max(dep done)
    depmax = np.zeros(n, dtype=np.int64)
    for k in range(m):
        col = nb[:, k]
        ok = col >= 0
        if not TR:
            depmax[ok] = np.maximum(depmax[ok], tsf[col[ok]])
        else:
            np.maximum.at(depmax, col[ok], tsf[np.flatnonzero(ok)])
    hop = tsf - depmax
    print(f"t={t} total={tsf.max()/1e3:.1f}us levels={nl}")
    print("  hop latency us: p50 %.2f p90 %.2f p99 %.2f max %.2f" % tuple(np.percentile(hop[lev > 0], [50, 90, 99, 100]) / 1e3))
    marks = [0, 10, 20, 50, 100, 150, 200, 250, 300, 330, nl - 1]
    print("  " + " ".join(f"L{Lv}({size[Lv]}):{lev_end[Lv]/1e3:.0f}" for Lv in marks if Lv < nl))
    # critical chain: from the last-finished row follow the latest-finishing dependency
    if not TR:
        cur = int(np.argmax(tsf))
        chain = []
        while True:
            row = nb[cur][nb[cur] >= 0]
            if row.size == 0:
                break
            j = int(row[np.argmax(tsf[row])])
            chain.append((lev[cur], tsf[cur] - tsf[j]))
            cur = j
        hops = np.array([h for _, h in chain])
        print("  critical chain: %d hops, sum %.1fus, hop p50 %.2f p90 %.2f max %.2f us" %
              (len(hops), hops.sum() / 1e3, *(np.percentile(hops, [50, 90, 100]) / 1e3)))
        print("  chain (level:hop_ns) " + " ".join(f"{lv}:{h}" for lv, h in chain))
    print("  level end (us): " + " ".join(f"{Lv}:{lev_end[Lv]/1e3:.1f}" for Lv in range(0, nl, 5)))
