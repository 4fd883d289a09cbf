"""numpy statement of the device Rademacher probe generator
(vl_probes_rademacher, csrc/laplace.cu): entry (factor row i, column c) is -1
if the top bit of splitmix64(seed * 0x9E3779B97F4A7C15 + i * t + c) is set,
else +1.  Test infrastructure: used to build the Z injected into the
reference (make_golden_scale.py rademacher) and to check the device draw."""
import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)


def _splitmix64(z):
    z = z + _GOLD
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def rademacher(n, t, seed):
    with np.errstate(over="ignore"):
        i = np.arange(n, dtype=np.uint64)[:, None]
        c = np.arange(t, dtype=np.uint64)[None, :]
        key = np.uint64(seed) * _GOLD + i * np.uint64(t) + c
        top = _splitmix64(key) >> np.uint64(63)
    return np.where(top == 1, -1.0, 1.0)
