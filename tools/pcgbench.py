"""PCG microbench at n = 1e6: fixed-iteration VADU PCG solves (t = 1 and
t = 50) through vl_pcg_vadu, per-kernel time per iteration from the
in-library profiler.  VLGPX_LIB selects a library variant."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_12000_b200 as vg  # noqa: E402
from paper_2310_12000_b200 import _lib  # noqa: E402
from paper_2310_12000_b200.vecchia import Pattern, build_factor, neighbor_array  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--ts", default="1,50")
    ap.add_argument("--iters", default="120,20")
    ap.add_argument("--label", default=os.environ.get("VLGPX_LIB", "default"))
    a = ap.parse_args()
    n = a.n
    xy = np.random.default_rng(0).uniform(size=(n, 2))
    perm = np.random.default_rng(1).permutation(n)
    nbr = neighbor_array(xy, perm, 20)
    xyp = np.ascontiguousarray(xy[perm])
    pat = Pattern(xyp, nbr, 1)
    f = build_factor(xyp, vg.CovarianceSpec(1.0, 0.02, 1.5), pat, want_grad=False)
    ctx = f.ctx
    L = _lib.lib()
    L.vl_prof_enable.argtypes = [_lib.c_void_p, _lib.c_int]
    L.vl_prof_reset.argtypes = [_lib.c_void_p]
    L.vl_prof_report.argtypes = [_lib.c_void_p, _lib.C.c_char_p, _lib.c_int, _lib.P_int64]
    g = torch.Generator(device="cuda").manual_seed(3)
    W = (0.05 + 0.2 * torch.rand(n, dtype=torch.float64, device="cuda", generator=g)).contiguous()
    for t, it in zip([int(x) for x in a.ts.split(",")], [int(x) for x in a.iters.split(",")]):
        Bm = torch.randn(n, t, dtype=torch.float64, device="cuda", generator=g).contiguous()
        U = torch.empty_like(Bm)
        iters = np.zeros(t, dtype=np.int32)
        conv = np.zeros(t, dtype=np.int32)
        res = np.zeros(t)

        def run():
            _lib.call("vl_pcg_vadu", ctx.h, f.h, _lib.ptr(W), t, _lib.ptr(Bm), _lib.ptr(U), 1e-30, it, 0,
                      iters.ctypes.data, conv.ctypes.data, res.ctypes.data, None, None, 0)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 2
        _lib.check(L.vl_prof_reset(ctx.h))
        _lib.check(L.vl_prof_enable(ctx.h, 1))
        run()
        torch.cuda.synchronize()
        buf = _lib.C.create_string_buffer(1 << 16)
        nl = _lib.C.c_int64(0)
        _lib.check(L.vl_prof_report(ctx.h, buf, 1 << 16, _lib.C.byref(nl)))
        _lib.check(L.vl_prof_enable(ctx.h, 0))
        ker = {}
        for ln in buf.value.decode().splitlines():
            tg, cnt, tms, by = ln.split("\t")
            ker[tg] = round(float(tms) / it, 4)
        print(json.dumps({"label": os.path.basename(a.label), "t": t, "iters": int(iters.max()),
                          "ms_per_iter": round(ms / it, 4), "per_iter_ms": ker,
                          "u_sum": float(U.sum())}), flush=True)


if __name__ == "__main__":
    main()
