"""One launch of each hot kernel at n=1e6 (for ncu capture)."""
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
pat = Pattern(xyp, nbr, int(os.environ.get("KP_ORDER", 1)))
f = build_factor(xyp, vg.CovarianceSpec(1.0, 0.02, 1.5), pat, want_grad=True)
for t in (50, 1):
    X = torch.randn(n, t, dtype=torch.float64, device="cuda") / 20
    Y = torch.empty_like(X)
    for fn, a in [("vl_spmm", 0), ("vl_spmm", 1), ("vl_sptrsv", 0), ("vl_sptrsv", 1)]:
        _lib.call(fn, f.ctx.h, f.h, a, t, _lib.ptr(X), _lib.ptr(Y))
torch.cuda.synchronize()
print("ok")
