"""Multi-process (world_size 2, gloo, CPU) checks of the probe-sharded path:
column sharding, probe-ordered gathers, and the two-round row-statistics
allreduce that reproduces the single-process control-variate weights
(laplace.py:401-419) -- computed here with the CPU oracle as the per-rank
compute (test infrastructure only)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_12000_b200.distributed import ProbeComm, shard_bounds
        comm = ProbeComm()
        t = 11
        c0, c1 = comm.shard(t)
        assert (c0, c1) == shard_bounds(t, world, rank)
        # per-probe values gathered in probe order
        full = comm.allgather_cols(np.arange(c0, c1, dtype=float) * 10.0, (c0, t))
        assert np.array_equal(full, np.arange(t) * 10.0)
        # row statistics: H, R for n rows x t probes (same seeded data on every rank)
        rng = np.random.default_rng(0)
        n = 257
        H = rng.standard_normal((n, t))
        R = rng.standard_normal((n, t)) ** 2 + 0.1
        h, r = H[:, c0:c1], R[:, c0:c1]
        rowA = torch.tensor(np.stack([h.sum(1), r.sum(1)], axis=1))
        comm.allreduce_(rowA)
        hbar, rbar = rowA[:, 0].numpy() / t, rowA[:, 1].numpy() / t
        rowB = torch.tensor(np.stack([((h - hbar[:, None]) * (r - rbar[:, None])).sum(1),
                                      ((r - rbar[:, None]) ** 2).sum(1)], axis=1))
        comm.allreduce_(rowB)
        c = rowB[:, 0].numpy() / rowB[:, 1].numpy()
        mean_term = (rowA[:, 0].numpy() - c * rowA[:, 1].numpy()) / t
        # single-process reference formula (oracle _cv_rows + mean(H - cR))
        from oracle import vl_oracle as O
        c_ref = O._cv_rows(H, R, t)
        m_ref = (H - c_ref[:, None] * R).mean(axis=1)
        out[rank] = (float(np.abs(c - c_ref).max()), float(np.abs(mean_term - m_ref).max()))
    finally:
        dist.destroy_process_group()


def test_probe_sharding_gloo_world2():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        dc, dm = out[r]
        assert dc < 1e-12 and dm < 1e-12, (r, dc, dm)


def test_shard_bounds_cover():
    from paper_2310_12000_b200.distributed import shard_bounds
    for t in (1, 7, 50, 64):
        for w in (1, 2, 3, 8):
            b = [shard_bounds(t, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == t
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            assert max(c1 - c0 for c0, c1 in b) - min(c1 - c0 for c0, c1 in b) <= 1
