"""Helpers to load the reference-generated fixtures in tests/golden/."""

import os

import numpy as np
import scipy.sparse as sp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

LAPLACE_CASES = ["logit_vadu_n400", "logit_vadu_n1500", "logit_vadu_cov_n300",
                 "probit_vadu_n300", "gamma_vadu_n300", "logit_lrac_n300",
                 "gamma_lrac_cov_n300", "poisson_vadu_n300", "logit_lva_n300", "logit_diag_n300",
                 "logit_identity_n300", "logit_pcholprec_n300", "logit_rowsel_n300", "gamma_l2_n300"]


def load(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)
    return {k: z[k] for k in z.files}


def csr(g, prefix):
    n = int(g["n"])
    return sp.csr_matrix((g[f"{prefix}_data"], g[f"{prefix}_indices"], g[f"{prefix}_indptr"]),
                         shape=(n, n))


def tridiags(g):
    out, a, b = [], 0, 0
    for k in g["tri_len"]:
        k = int(k)
        out.append((g["tri_diag"][a:a + k], g["tri_off"][b:b + max(k - 1, 0)]))
        a += k
        b += max(k - 1, 0)
    return out


def scal(g, key):
    v = g[key]
    return v.item() if v.ndim == 0 else v
