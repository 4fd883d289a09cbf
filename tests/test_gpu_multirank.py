"""Probe sharding through the real device path with two ranks.

Two processes share cuda:0 and talk through gloo (host collectives only: no
kernel of one rank waits on the other, so sharing one GPU is safe).  Each
rank runs make_probes / neg_marginal_loglik / gradient with a ProbeComm on
its contiguous column shard; the results must equal the single-process
evaluation to 1e-10 (probe-ordered sums make them independent of the rank
count).  Covers VADU (row-statistics allreduce rounds) and LRAC.

Bar: NLL 1e-12 (probe-ordered SLQ sums are exact across shardings); gradient
1e-8 -- the per-row control-variate sums are added rank by rank
instead of in one warp tree, which moves dtheta by <= 6.3e-10 relative
(measured, gamma/LRAC cases) because c_i = cov_i / var_i amplifies rounding."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _evaluate(name, comm):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from _golden import load, scal

    import paper_2310_12000_b200 as vg
    from paper_2310_12000_b200.vecchia import build_factor
    g = load(name)
    spec = vg.CovarianceSpec(scal(g, "sigma2"), scal(g, "rho"), scal(g, "nu"))
    f = build_factor(g["coords"], spec, g["nbr"], g["perm"])
    fam = str(g["family"])
    lik = vg.get_likelihood(fam, **({"shape": float(g["shape"])} if fam == "gamma" else {}))
    rank = int(g["rank"])
    cfg = vg.BackendConfig(preconditioner=str(g["precond"]), t=int(g["t"]), probe_seed=int(g["probe_seed"]),
                           rank=None if rank < 0 else rank)
    perm = g["perm"]
    st = vg.find_mode(f, lik, g["y"][perm], g["F"][perm], cfg)
    cols = comm.shard(cfg.t) if comm is not None else None
    pr, P = vg.make_probes(f, st, cfg, cols=cols)
    nll = vg.neg_marginal_loglik(st, f, cfg, probes=pr, P=P, comm=comm)
    gr = vg.gradient(st, f, lik, g["X"][perm], cfg, probes=pr, P=P, comm=comm)
    return nll, gr


def _worker(rank, world, port, names, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_12000_b200.distributed import ProbeComm
        comm = ProbeComm()
        for name in names:
            nll, gr = _evaluate(name, comm)
            out[(rank, name)] = (nll, [float(v) for v in gr["dtheta"]], [float(v) for v in gr["dbeta"]],
                                 [float(v) for v in gr["dxi"]])
    finally:
        dist.destroy_process_group()


CASES = ["logit_vadu_n1500", "gamma_vadu_n300", "logit_lrac_n300", "gamma_lrac_cov_n300"]


def test_probe_sharded_device_path_world2():
    import torch.multiprocessing as mp
    ref = {name: _evaluate(name, None) for name in CASES}
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), CASES, out), nprocs=world, join=True)
    for name in CASES:
        nll0, g0 = ref[name]
        for r in range(world):
            nll, dth, dbe, dxi = out[(r, name)]
            assert abs(nll - nll0) <= 1e-12 * abs(nll0), (name, r, nll, nll0)
            np.testing.assert_allclose(dth, g0["dtheta"], rtol=1e-8, atol=1e-12, err_msg=name)
            np.testing.assert_allclose(dbe, g0["dbeta"], rtol=1e-8, atol=1e-12, err_msg=name)
            np.testing.assert_allclose(dxi, g0["dxi"], rtol=1e-8, atol=1e-12, err_msg=name)
