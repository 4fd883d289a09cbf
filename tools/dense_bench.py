"""Hand-written fp64 GEMM (csrc/dense.cu) vs cuBLAS (torch.matmul) on the
shapes of the low-rank paths at config 2 (n = 1e5, k = 1000, t = 1 / 50):
ms and fp64 TFLOP/s per call.  VL_DGEMM_TC=0 forces the FMA tiles."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_12000_b200 as vg  # noqa: E402,F401
from paper_2310_12000_b200 import _lib  # noqa: E402
from paper_2310_12000_b200 import device as dev  # noqa: E402

ctx = dev.context()
n, k = 100_000, 1000
g = torch.Generator(device="cuda").manual_seed(0)
L = torch.randn(n, k, dtype=torch.float64, device="cuda", generator=g)       # row-major n x k
W = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
Kk = torch.randn(k, k, dtype=torch.float64, device="cuda", generator=g)


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def ours(ta, tb, m, nn, kk, A, lda, B, ldb, C, ldc, kw=None, lower=0):
    return lambda: _lib.call("vl_dgemm", ctx.h, ta, tb, m, nn, kk, 1.0, _lib.ptr(A), lda, _lib.ptr(B), ldb, 0.0,
                             _lib.ptr(C), ldc, _lib.ptr(kw) if kw is not None else None, lower)


cases = []
M = torch.empty(k, k, dtype=torch.float64, device="cuda")
cases.append(("syrk_LtWL k=1000 n=1e5 (lower)", ours(0, 1, k, k, n, L, k, L, k, M, k, W, 1),
              lambda: torch.matmul(L.T, W[:, None] * L), n * k * k))
for t in (1, 50):
    X = torch.randn(n, t, dtype=torch.float64, device="cuda", generator=g)
    w = torch.empty(k, t, dtype=torch.float64, device="cuda")
    cases.append((f"Lt_x t={t}", ours(0, 1, k, t, n, L, k, X, t, w, k), lambda X=X: torch.matmul(L.T, X),
                  2 * n * k * t))
    u = torch.randn(t, k, dtype=torch.float64, device="cuda", generator=g)   # column-major k x t
    y = torch.empty(n, t, dtype=torch.float64, device="cuda")
    cases.append((f"L_u t={t}", ours(1, 0, t, n, k, u, k, L, k, y, t), lambda u=u: torch.matmul(L, u.T),
                  2 * n * k * t))
Y = torch.empty(n, k, dtype=torch.float64, device="cuda")
cases.append(("kxk_times_kxn (dL chain)", ours(0, 0, k, n, k, Kk, k, L, k, Y, k), lambda: torch.matmul(L, Kk.T),
              2 * n * k * k))
C3 = torch.empty(k, k, dtype=torch.float64, device="cuda")
cases.append(("kxk_kxk", ours(0, 0, k, k, k, Kk, k, Kk, k, C3, k), lambda: torch.matmul(Kk, Kk), 2 * k ** 3))
for name, f_ours, f_ref, flops in cases:
    a, b = timeit(f_ours), timeit(f_ref)
    print(json.dumps({"case": name, "ours_ms": round(a, 4), "cublas_ms": round(b, 4),
                      "ours_tflops": round(flops / a / 1e9, 2), "cublas_tflops": round(flops / b / 1e9, 2),
                      "tc": os.environ.get("VL_DGEMM_TC", "1")}), flush=True)
