"""Reference runs at the BASELINE.json configurations -- fixture generator.

Run in the build container (where /root/reference exists); the GPU box only
reads what this writes:

    python tests/golden/make_golden_scale.py data3      # config-3 dataset (cached under /tmp)
    python tests/golden/make_golden_scale.py c3         # reference evaluation at config 3
    python tests/golden/make_golden_scale.py c3mode6    # reference find_mode at newton_grad_tol=1e-6
    python tests/golden/make_golden_scale.py c1 c2 c2lrac replay

Every number is produced by the REFERENCE package itself (``vlgp`` imported
from /root/reference/pkg/src) through its public API: ``find_neighbors``,
``build_factor``, ``find_mode``, ``make_probes``, ``neg_marginal_loglik``,
``gradient``.  ``vlgp.laplace.pcg_solve`` is wrapped (the original is called)
only to record the CG iteration counts of each phase.

Datasets:
* c1: n=1e4, rho=0.05, dense-Cholesky latent field (as pkg/tests/util.py).
* c2: n=1e5, rho=0.05, Vecchia-sampled latent field (m_sim=30).
* c3: n=1e6, rho=0.02, the exact bench.py dataset (seed 2310): coords, the
  Vecchia-sampled latent field and y are produced by the same recipe as
  ``bench.latent_field`` but with the reference's functions; the bench checks
  the sha256 of its own y against the one stored here before reporting parity.
* replay: n=2e4, t=50 -- large enough that the GPU's dense head block is
  active and the t=50 (G=32) PCG bodies run; stores W, b*, tridiagonals and
  projections of the probe solves.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
CACHE = "/tmp/vlgp_c3"


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import vlgp  # noqa: F401
    return vlgp


class CGLog:
    """Records (phase, iterations, tol) of every reference pcg_solve call."""

    def __init__(self, live=None):
        import vlgp.laplace as L
        self.L = L
        self.orig = L.pcg_solve
        self.phase = "mode"
        self.calls = []
        self.live = live

        def wrapped(*a, **k):
            t0 = time.perf_counter()
            res = self.orig(*a, **k)
            tol = a[3] if len(a) > 3 else k.get("tol")
            self.calls.append((self.phase, int(res.iterations), float(tol)))
            if self.live:
                print(f"[{time.strftime('%H:%M:%S')}] {self.phase} pcg its={res.iterations} tol={tol:.3e} "
                      f"conv={res.converged} {time.perf_counter() - t0:.1f}s", file=self.live, flush=True)
            return res

        L.pcg_solve = wrapped

    def its(self, phase):
        return [c[1] for c in self.calls if c[0] == phase]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def nbr_array(nb, m):
    out = np.full((len(nb), m), -1, dtype=np.int32)
    for i, s in enumerate(nb):
        out[i, : len(s)] = s
    return out


def vecchia_latent(coords, rho, seed, m_sim=30):
    """b ~ N(0, SigmaTilde_sim): b = B^-1 (sqrt(D) g) in a separate random
    ordering (seed+1), normals from seed+2 -- bench.latent_field's recipe."""
    from vlgp.covariance import CovarianceSpec
    from vlgp.vecchia import build_factor, find_neighbors
    n = coords.shape[0]
    perm = np.random.default_rng(seed + 1).permutation(n)
    nb = find_neighbors(coords, perm, m_sim)
    f = build_factor(coords, CovarianceSpec(1.0, rho, 1.5), nb, perm)
    g = np.random.default_rng(seed + 2).standard_normal(n)
    b_perm = f.solve_B(np.sqrt(f.D) * g)
    b = np.empty_like(b_perm)
    b[perm] = b_perm
    return b


def bench_dataset(n, rho, seed):
    """bench.synth + bench.latent_field + the Bernoulli draw, reference side."""
    coords = np.random.default_rng(seed).uniform(size=(n, 2))
    b = vecchia_latent(coords, rho, seed)
    p = 1.0 / (1.0 + np.exp(-b))
    y = (np.random.default_rng(seed + 4).uniform(size=n) < p).astype(float)
    return coords, b, y


def dense_dataset(n, rho, seed):
    """pkg/tests/util.py:18-22 recipe (dense Cholesky draw), Bernoulli-logit."""
    from vlgp.covariance import CovarianceSpec, cov_matrix
    from vlgp.likelihoods import get_likelihood
    rng = np.random.default_rng(seed)
    coords = rng.uniform(size=(n, 2))
    K = cov_matrix(CovarianceSpec(1.0, rho, 1.5), coords)
    b = np.linalg.cholesky(K) @ rng.standard_normal(n)
    del K
    y = get_likelihood("bernoulli-logit").sample(b, rng)
    return coords, b, y


def evaluate(coords, y, rho, m, t, ordering_seed, probe_seed, precond="vadu", rank=None,
             newton_grad_tol=1e-6, nbr=None, live=None, keep=False):
    """One reference evaluation (estimate.py:125-150 sequence) with timings."""
    from vlgp.covariance import CovarianceSpec
    from vlgp.laplace import BackendConfig, find_mode, gradient, make_probes, neg_marginal_loglik
    from vlgp.likelihoods import get_likelihood
    from vlgp.vecchia import build_factor, find_neighbors, order_random

    n = coords.shape[0]
    log = CGLog(live)
    tm = {}
    t0 = time.perf_counter()
    perm = order_random(n, ordering_seed)
    if nbr is None:
        nb = find_neighbors(coords, perm, m)
    else:
        nb = [r[r >= 0].astype(int) for r in nbr]
    tm["knn_s"] = time.perf_counter() - t0
    cfg = BackendConfig(preconditioner=precond, t=t, cg_tol=1e-3, probe_seed=probe_seed, rank=rank,
                        newton_grad_tol=newton_grad_tol)
    lik = get_likelihood("bernoulli-logit")
    theta = np.array([1.0, rho])
    t0 = time.perf_counter()
    f = build_factor(coords, CovarianceSpec(1.0, rho, 1.5), nb, perm)
    tm["factor_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    st = find_mode(f, lik, y[perm], np.zeros(n), cfg)
    tm["mode_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    log.phase = "probes"
    pr, P = make_probes(f, st, cfg)
    nll = neg_marginal_loglik(st, f, cfg, probes=pr, P=P)
    tm["nll_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    log.phase = "grad"
    g = gradient(st, f, lik, np.zeros((n, 0)), cfg, probes=pr, P=P)
    tm["grad_s"] = time.perf_counter() - t0
    tm["eval_s"] = tm["factor_s"] + tm["mode_s"] + tm["nll_s"] + tm["grad_s"]
    log.L.pcg_solve = log.orig
    out = dict(n=n, m=m, t=t, rho=rho, precond=precond, rank=-1 if rank is None else rank,
               ordering_seed=ordering_seed, probe_seed=probe_seed, newton_grad_tol=newton_grad_tol,
               nll=float(nll), dtheta=[float(v) for v in g["dtheta"]],
               grad_log_theta=[float(v) for v in g["dtheta"] * theta],
               newton_iters=int(st.newton_iters), newton_cg=log.its("mode"),
               probe_cg=[int(tr.order) for tr in pr.tridiags], grad_cg=log.its("grad"),
               logp=float(st.logp), quad=float(st.quad), logdet_P=float(P.logdet()),
               b_norm=float(np.linalg.norm(st.b)), b_sum=float(st.b.sum()), W_sum=float(st.W.sum()),
               nbr_sha256=sha(nbr_array(nb, m)), timings=tm,
               threads=os.environ.get("OMP_NUM_THREADS", "default"))
    if keep:
        return out, dict(f=f, st=st, pr=pr, P=P, nb=nb, perm=perm)
    return out, None


def _dump_json(name, d):
    with open(os.path.join(HERE, name), "w") as fh:
        json.dump(d, fh, indent=1)
    print(name, json.dumps({k: d[k] for k in ("nll", "dtheta", "newton_iters") if k in d}))


def data3():
    os.makedirs(CACHE, exist_ok=True)
    t0 = time.perf_counter()
    coords, b, y = bench_dataset(1_000_000, 0.02, 2310)
    np.savez(os.path.join(CACHE, "data.npz"), coords=coords, b=b, y=y)
    print(f"data3: {time.perf_counter() - t0:.0f}s, y sum {y.sum()}, sha {sha(y.astype(np.uint8))}")


def c3(tol=1e-5):
    z = np.load(os.path.join(CACHE, "data.npz"))
    coords, y = z["coords"], z["y"]
    with open(os.path.join(CACHE, f"c3_tol{tol:g}.log"), "w") as live:
        out, _ = evaluate(coords, y, 0.02, 20, 50, ordering_seed=2313, probe_seed=2315,
                          newton_grad_tol=tol, live=live)
    out.update(seed=2310, y_sha256=sha(y.astype(np.uint8)), y_sum=float(y.sum()),
               source="reference vlgp (/root/reference/pkg/src) run in the build container by "
                      "tests/golden/make_golden_scale.py c3")
    _dump_json("c3_reference.json", out)


def c3mode6():
    """The reference's find_mode at its DEFAULT newton_grad_tol=1e-6 on the
    config-3 dataset: record whether it converges (DESIGN 6)."""
    from vlgp.covariance import CovarianceSpec
    from vlgp.errors import ConvergenceError
    from vlgp.laplace import BackendConfig, find_mode
    from vlgp.likelihoods import get_likelihood
    from vlgp.vecchia import build_factor, find_neighbors, order_random

    z = np.load(os.path.join(CACHE, "data.npz"))
    coords, y = z["coords"], z["y"]
    n = coords.shape[0]
    logp = os.path.join(HERE, "..", "..", "profiles", "r2_c3_reference_newton_tol1e-6.log")
    with open(logp, "w") as live:
        print("reference vlgp find_mode at config 3 (n=1e6, rho=0.02, m=20, logit, VADU), "
              "BackendConfig defaults (newton_grad_tol=1e-6); every pcg_solve call logged", file=live, flush=True)
        log = CGLog(live)
        perm = order_random(n, 2313)
        nb = find_neighbors(coords, perm, 20)
        f = build_factor(coords, CovarianceSpec(1.0, 0.02, 1.5), nb, perm)
        print(f"D_min={f.D.min():.4e}", file=live, flush=True)
        cfg = BackendConfig(t=50, cg_tol=1e-3, probe_seed=2315)
        trace = []
        t0 = time.perf_counter()
        try:
            st = find_mode(f, get_likelihood("bernoulli-logit"), y[perm], np.zeros(n), cfg, trace=trace)
            print(f"CONVERGED newton_iters={st.newton_iters} in {time.perf_counter() - t0:.0f}s", file=live, flush=True)
        except ConvergenceError as e:
            print(f"ConvergenceError: {e} after {time.perf_counter() - t0:.0f}s", file=live, flush=True)
            st = e.last_state
            gn = float(np.abs(st.d1 - f.apply_precision(st.b)).max())
            print(f"last state: grad sup-norm {gn:.3e} objective {st.objective!r}", file=live, flush=True)
        print("objective trace:", json.dumps(trace), file=live, flush=True)
        print("newton cg iterations:", json.dumps(log.its("mode")), file=live, flush=True)


def c1():
    coords, b, y = dense_dataset(10_000, 0.05, 101)
    out, keep = evaluate(coords, y, 0.05, 20, 50, ordering_seed=102, probe_seed=103, keep=True)
    st = keep["st"]
    np.savez_compressed(os.path.join(HERE, "c1_n1e4.npz"), coords=coords, y=y.astype(np.uint8),
                        b=st.b, W=st.W, meta=json.dumps(out))
    print("c1", json.dumps({k: out[k] for k in ("nll", "dtheta", "newton_iters", "timings")}))


def c2(precond="vadu"):
    coords, b, y = bench_dataset(100_000, 0.05, 201)
    rank = 1000 if precond == "lrac" else None
    tol = 1e-6
    try:
        out, keep = evaluate(coords, y, 0.05, 20, 50, ordering_seed=202, probe_seed=203, precond=precond,
                             rank=rank, newton_grad_tol=tol, keep=True)
    except Exception as e:  # ConvergenceError at the fp64 floor (DESIGN 6): record it, retry at 1e-5
        print(f"c2 {precond} at newton_grad_tol=1e-6: {type(e).__name__}: {e}")
        tol = 1e-5
        out, keep = evaluate(coords, y, 0.05, 20, 50, ordering_seed=202, probe_seed=203, precond=precond,
                             rank=rank, newton_grad_tol=tol, keep=True)
        out["note_tol1e-6"] = f"{type(e).__name__}: {e}"
    st = keep["st"]
    out.update(seed=201, y_sha256=sha(y.astype(np.uint8)))
    np.savez_compressed(os.path.join(HERE, f"c2_{precond}_n1e5.npz"), y_bits=np.packbits(y.astype(np.uint8)),
                        b_stride=st.b[::97].copy(), W_stride=st.W[::97].copy(), meta=json.dumps(out))
    print("c2", precond, json.dumps({k: out[k] for k in ("nll", "dtheta", "newton_iters", "timings")}))


def replay():
    """n=2e4, t=50 end-to-end + CG replay material (head block active on the GPU)."""
    coords, b, y = bench_dataset(20_000, 0.05, 301)
    out, keep = evaluate(coords, y, 0.05, 20, 50, ordering_seed=302, probe_seed=303, keep=True)
    st, pr = keep["st"], keep["pr"]
    c = np.random.default_rng(304).standard_normal(coords.shape[0])
    tri = pr.tridiags
    np.savez_compressed(os.path.join(HERE, "replay_n2e4_t50.npz"), y=y.astype(np.uint8), b=st.b, W=st.W,
                        Z_proj=c @ pr.Z, Z_norm=np.linalg.norm(pr.Z, axis=0),
                        U_proj=c @ pr.solves, U_norm=np.linalg.norm(pr.solves, axis=0),
                        U_head=pr.solves[:64].copy(), V_proj=c @ pr.psolves,
                        tri_len=np.array([tr.order for tr in tri]),
                        tri_diag=np.concatenate([tr.diag for tr in tri]),
                        tri_off=np.concatenate([tr.off for tr in tri]), meta=json.dumps(out))
    print("replay", json.dumps({k: out[k] for k in ("nll", "dtheta", "newton_iters", "probe_cg")}))


def rademacher_case():
    """The reference's ProbeSet injection (laplace.py:340) with probes built from
    Rademacher base draws R (tests/golden/rademacher.py) on the logit_vadu_n1500
    dataset: Z = B^T (sqrt(d) o R), the sample_block construction
    (preconditioners.py:121-122) with R for the Gaussian draws.  vadu (d = W + 1/D)
    and lva (d = 1/D).  With R_i^2 = 1 the VADU per-row control variate divides
    rounding noise by rounding noise (Var_t((BV)_i^2) = Var_t(1 / d_i) = 0), so only
    its NLL is a meaningful comparison; lva's plain estimator gives the gradient."""
    from vlgp.covariance import CovarianceSpec
    from vlgp.iterative import ProbeSet
    from vlgp.laplace import BackendConfig, build_preconditioner, find_mode, gradient, neg_marginal_loglik
    from vlgp.likelihoods import get_likelihood
    from vlgp.vecchia import build_factor
    sys.path.insert(0, HERE)
    from rademacher import rademacher
    g = np.load(os.path.join(HERE, "logit_vadu_n1500.npz"))
    n, t, seed = int(g["n"]), 16, 4242
    nb = [r[r >= 0].astype(int) for r in g["nbr"]]
    f = build_factor(g["coords"], CovarianceSpec(float(g["sigma2"]), float(g["rho"]), float(g["nu"])), nb, g["perm"])
    lik = get_likelihood("bernoulli-logit")
    R = rademacher(n, t, seed)
    out, arrays = {"case": "logit_vadu_n1500", "t": t, "seed": seed}, {}
    for pc in ("vadu", "lva"):
        cfg = BackendConfig(preconditioner=pc, t=t, probe_seed=seed)
        st = find_mode(f, lik, g["y"][g["perm"]], g["F"][g["perm"]], cfg)
        P = build_preconditioner(f, st.W, cfg)
        d = st.W + 1.0 / f.D if pc == "vadu" else 1.0 / f.D
        Z = f.B.T @ (np.sqrt(d)[:, None] * R)
        pr = ProbeSet(Z, seed, P.name)
        nll = neg_marginal_loglik(st, f, cfg, probes=pr, P=P)
        gr = gradient(st, f, lik, np.zeros((n, 0)), cfg, probes=pr, P=P)
        out[pc] = dict(nll=float(nll), dtheta=[float(v) for v in gr["dtheta"]],
                       probe_cg=[int(tr.order) for tr in pr.tridiags])
        arrays[f"Z_{pc}"] = Z
    np.savez_compressed(os.path.join(HERE, "rademacher_n1500.npz"), meta=json.dumps(out), **arrays)
    print("rademacher", json.dumps(out)[:400])


def main():
    _ref()
    for job in sys.argv[1:]:
        {"data3": data3, "c3": c3, "c3mode6": c3mode6, "c1": c1, "c2": c2,
         "c2lrac": lambda: c2("lrac"), "replay": replay, "rademacher": rademacher_case}[job]()


if __name__ == "__main__":
    main()
