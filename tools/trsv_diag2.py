"""Per-row timeline of the single-column forward solve (needs the VL_TS_EXT
diagnostic build): item start, dependencies-in (pend cleared), store, poll
rounds; summarised per level band."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_12000_b200 as vg  # noqa: E402
from paper_2310_12000_b200 import _lib  # noqa: E402
from paper_2310_12000_b200.vecchia import Pattern, build_factor, neighbor_array  # noqa: E402

n, m = 1000000, 20
xy = np.random.default_rng(0).uniform(size=(n, 2))
perm = np.random.default_rng(1).permutation(n)
nbr = neighbor_array(xy, perm, m)
xyp = np.ascontiguousarray(xy[perm])
pat = Pattern(xyp, nbr, 1)
f = build_factor(xyp, vg.CovarianceSpec(1.0, 0.02, 1.5), pat, want_grad=False)
L = _lib.lib()
L.vl_debug_set_tstamp.argtypes = [C.c_void_p, C.c_void_p]
ts = torch.zeros(5 * n, dtype=torch.int64, device="cuda")
lev = np.zeros(n, dtype=np.int64)
for i in range(n):
    row = nbr[i][nbr[i] >= 0]
    if row.size:
        lev[i] = lev[row].max() + 1
X = torch.randn(n, 1, dtype=torch.float64, device="cuda") / 20
Y = torch.empty_like(X)
for _ in range(3):
    _lib.call("vl_sptrsv", f.ctx.h, f.h, 0, 1, _lib.ptr(X), _lib.ptr(Y))
torch.cuda.synchronize()
L.vl_debug_set_tstamp(f.ctx.h, C.c_void_p(ts.data_ptr()))
_lib.call("vl_sptrsv", f.ctx.h, f.h, 0, 1, _lib.ptr(X), _lib.ptr(Y))
torch.cuda.synchronize()
L.vl_debug_set_tstamp(f.ctx.h, None)
a = ts.cpu().numpy().reshape(5, n)
done, start, ready, rounds, slab = (np.empty(n, dtype=np.int64) for _ in range(5))
for arr, k in ((done, 0), (start, 1), (ready, 2), (rounds, 3), (slab, 4)):
    arr[pat.sperm] = a[k]
ok = start > 0
t0 = start[ok].min()
depmax = np.zeros(n, dtype=np.int64)
for k in range(m):
    col = nbr[:, k]
    g = col >= 0
    depmax[g] = np.maximum(depmax[g], done[col[g]])
nl = lev.max() + 1
print("band      rows   start-dep  ready-dep  done-ready  rounds  (us, medians; start-dep<0 = started early)")
for lo in range(150, nl, 20):
    sel = ok & (lev >= lo) & (lev < lo + 20) & (depmax > 0)
    if sel.sum() == 0:
        continue
    sd = (start[sel] - depmax[sel]) / 1e3
    rd = (ready[sel] - depmax[sel]) / 1e3
    dr = (done[sel] - ready[sel]) / 1e3
    ss = (slab[sel] - start[sel]) / 1e3          # item start -> slab entries in registers
    r1 = sel & (rounds == 1)
    rs = (ready[r1] - slab[r1]) / 1e3 if r1.sum() else np.zeros(1)   # gathers + rhs (no polling needed)
    tot = (done[sel] - start[sel]) / 1e3
    print(f"L{lo:3d}-{lo+19:3d} {sel.sum():7d}  {np.median(sd):9.2f}  {np.median(rd):9.2f}  {np.median(dr):9.2f}  "
          f"{np.median(rounds[sel]):6.0f}   p90 ready-dep {np.percentile(rd, 90):.2f}  slab-start {np.median(ss):.2f} "
          f"ready-slab(rounds=1) {np.median(rs):.2f} item {np.median(tot):.2f}")
