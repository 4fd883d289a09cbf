"""Newton diagnostics at the bench configuration."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("VL_DEBUG_NEWTON", "1")
import bench  # noqa: E402
import paper_2310_12000_b200 as vg  # noqa: E402
from paper_2310_12000_b200.vecchia import Pattern, build_factor, neighbor_array  # noqa: E402

n = int(os.environ.get("KP_N", 1000000))
rho = float(os.environ.get("KP_RHO", 0.02))
class A: pass
a = A(); a.n = n; a.seed = 2310; a.rho = rho
coords, _ = bench.synth(a)
b_true = bench.latent_field(coords, rho, a.seed)
y = (np.random.default_rng(a.seed + 4).uniform(size=n) < 1 / (1 + np.exp(-b_true))).astype(float)
perm = np.random.default_rng(a.seed + 3).permutation(n)
nbr = neighbor_array(coords, perm, 20)
xy = np.ascontiguousarray(coords[perm])
pat = Pattern(xy, nbr, 1)
f = build_factor(xy, vg.CovarianceSpec(1.0, rho, 1.5), pat)
D = f.D
print("D min %.3e median %.3e" % (D.min(), np.median(D)), flush=True)
cfg = vg.BackendConfig(t=50, cg_tol=1e-3, newton_max_iter=int(os.environ.get("KP_NEWTON", 30)))
t0 = time.time()
try:
    st = vg.find_mode(f, vg.get_likelihood("bernoulli-logit"), y[perm], np.zeros(n), cfg)
    print("converged", st.newton_iters, st.cg_iters, time.time() - t0)
except vg.ConvergenceError as e:
    print("not converged", e, time.time() - t0)
