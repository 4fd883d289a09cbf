import faulthandler, sys, time
faulthandler.dump_traceback_later(150, exit=True)
sys.path.insert(0, '.')
import numpy as np
import paper_2310_12000_b200 as vg
from paper_2310_12000_b200.vecchia import build_factor, neighbor_array
rng = np.random.default_rng(11)
n = n_p = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
t0=time.time()
xy = rng.uniform(size=(n + n_p, 2))
perm = vg.order_random(n, 5)
spec = vg.CovarianceSpec(1.0, 0.05, 1.5)
f = build_factor(xy[:n], spec, neighbor_array(xy[:n], perm, 10), perm, want_grad=False)
print('factor', time.time()-t0, flush=True)
lik = vg.get_likelihood("poisson")
y = lik.sample(0.3 * rng.standard_normal(n), rng)
cfg = vg.BackendConfig(preconditioner="vadu", t=4)
st = vg.find_mode(f, lik, y[perm], np.zeros(n), cfg)
print('mode', time.time()-t0, st.newton_iters, flush=True)
blocks = vg.prediction_blocks(f, xy[n:])
print('blocks', time.time()-t0, flush=True)
for variant in ("none","l1","l2"):
    var, order = vg.latent_var_lanczos(st, f, blocks, 31, variant=variant, cfg=cfg)
    print(variant, order, var[:3], time.time()-t0, flush=True)
