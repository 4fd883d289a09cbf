"""Time the device neighbour search against the native host search at n=1e6."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_12000_b200.vecchia import neighbor_array, order_random  # noqa: E402

n, m = int(os.environ.get("KN_N", 1000000)), 20
xy = np.random.default_rng(2310).uniform(size=(n, 2))
perm = order_random(n, 7)
neighbor_array(xy[:5000], perm[perm < 5000] if False else np.arange(5000), m, where="device")  # warm
t0 = time.perf_counter(); a = neighbor_array(xy, perm, m, where="device"); t1 = time.perf_counter()
b = neighbor_array(xy, perm, m, where="host"); t2 = time.perf_counter()
print(f"n={n} m={m} device {t1-t0:.3f}s host {t2-t1:.3f}s equal={np.array_equal(a, b)}")
