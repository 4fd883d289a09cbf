"""Probe sharding over ranks (one process per GPU, torch.distributed).

The t probe columns are split contiguously over the ranks; the
factor, the Newton mode and the tvec solve are replicated (deterministic, no
broadcast needed).  Collectives per evaluation:
  * allgather of the t per-probe SLQ terms (summed in probe order, so the
    result does not depend on the number of ranks);
  * allgather of the per-probe STE (h, r) pairs;
  * two rounds of n-vector allreduce for the per-row control-variate
    statistics (sum H, sum R; then the centred cross/square sums).
"""

from __future__ import annotations

import numpy as np



def shard_bounds(t, world, rank):
    """Contiguous split of t columns: the first t % world ranks get one extra."""
    base, extra = divmod(t, world)
    c0 = rank * base + min(rank, extra)
    c1 = c0 + base + (1 if rank < extra else 0)
    return c0, c1


class ProbeComm:
    def __init__(self, group=None, force_split=False):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.force_split = force_split  # use the sharded gradient path even at world == 1 (tests)

    def shard(self, t):
        return shard_bounds(t, self.world, self.rank)

    def _device(self):
        import torch
        return torch.device("cuda", torch.cuda.current_device()) if self.dist.get_backend(self.group) == "nccl" \
            else torch.device("cpu")

    def allgather_cols(self, parts, shard):
        """Gather per-probe values of every rank's column shard into the full
        probe-ordered vector (t = shard[1] global probes)."""
        import torch
        t = int(shard[1])
        parts = np.asarray(parts, dtype=float)
        dev = self._device()
        full = torch.zeros(t, dtype=torch.float64, device=dev)
        c0 = int(shard[0])
        full[c0:c0 + parts.size] = torch.as_tensor(parts, dtype=torch.float64, device=dev)
        self.dist.all_reduce(full, group=self.group)   # disjoint supports: sum == gather
        return full.cpu().numpy()

    def allreduce_(self, tensor):
        """In-place sum over ranks (device tensors through NCCL; with a CPU
        backend such as gloo the data is staged through host memory)."""
        if getattr(tensor, "is_cuda", False) and self.dist.get_backend(self.group) != "nccl":
            host = tensor.cpu()
            self.dist.all_reduce(host, group=self.group)
            tensor.copy_(host)
            return tensor
        self.dist.all_reduce(tensor, group=self.group)
        return tensor

    def grad_probe_pass(self, factor, state, probes, md3x, plain=0):
        """Sharded gradient probe pass: local row sums -> allreduce -> centred
        sums -> allreduce -> s; STE (h, r) per probe gathered in probe order."""
        from . import _lib
        from . import device as dev
        ctx, n = factor.ctx, factor.n
        dv = state._dev
        t = probes.t
        t_glob = int(probes.shard[1])
        rowA = dev.empty(ctx, n, 2)
        rowB = dev.empty(ctx, n, 2)
        s = dev.empty(ctx, n, 1)
        cols = np.zeros((4, t))
        xicols = np.zeros((2, t))
        gamma = md3x is not None
        args = (ctx.h, factor.h)
        common = (_lib.ptr(dv["W"]), _lib.ptr(dv["d3"]), _lib.ptr(probes.solves_dev), _lib.ptr(probes.psolves_dev),
                  t, t_glob, _lib.ptr(rowA), _lib.ptr(rowB), _lib.ptr(s))
        _lib.call("vl_grad_probe_pass_split", *args, 1, *common, _lib.ptr(cols),
                  _lib.ptr(md3x) if gamma else None, _lib.ptr(xicols) if gamma else None, int(plain))
        self.allreduce_(rowA)
        if not plain:  # the centred sums only feed the control-variate weights
            _lib.call("vl_grad_probe_pass_split", *args, 2, *common, None, None, None, 0)
            self.allreduce_(rowB)
        _lib.call("vl_grad_probe_pass_split", *args, 3, *common, None, None, None, int(plain))
        full = np.stack([self.allgather_cols(cols[k], probes.shard) for k in range(4)])
        xfull = np.stack([self.allgather_cols(xicols[k], probes.shard) for k in range(2)]) if gamma else np.zeros((2, t_glob))
        return s, full, xfull

    def lrac_grad_pass(self, factor, state, probes, P, md3x, plain=0):
        """Sharded LRAC gradient pass (eq7): the mu-derivative's per-row
        control variate through two row-sum allreduce rounds; the per-probe
        h / r columns gathered in probe order; dP_trace and the xi scalars
        do not depend on the probes and are identical on every rank."""
        from . import _lib
        from . import device as dev
        ctx, n = factor.ctx, factor.n
        dv = state._dev
        t = probes.t
        t_glob = int(probes.shard[1])
        rowA = dev.empty(ctx, n, 2)
        rowB = dev.empty(ctx, n, 2)
        s = dev.empty(ctx, n, 1)
        hcols, rcols, xicols = np.zeros((2, t)), np.zeros((2, t)), np.zeros((2, t))
        dPt, xis = np.zeros(2), np.zeros(2)
        gamma = md3x is not None
        head = (ctx.h, P.h)
        bufs = (_lib.ptr(probes.solves_dev), _lib.ptr(probes.psolves_dev), _lib.ptr(dv["d3"]),
                _lib.ptr(md3x) if gamma else None, _lib.ptr(rowA), _lib.ptr(rowB), _lib.ptr(s))
        outs = (_lib.ptr(hcols), _lib.ptr(rcols), _lib.ptr(dPt), _lib.ptr(xicols), _lib.ptr(xis))
        _lib.call("vl_lrac_grad_split", *head, 1, t, t_glob, *bufs, *outs, int(plain))
        self.allreduce_(rowA)
        if not plain:
            _lib.call("vl_lrac_grad_split", *head, 2, t, t_glob, *bufs, *outs, int(plain))
            self.allreduce_(rowB)
        _lib.call("vl_lrac_grad_split", *head, 3, t, t_glob, *bufs, *outs, int(plain))
        gather = lambda a: np.stack([self.allgather_cols(a[k], probes.shard) for k in range(2)])  # noqa: E731
        return s, gather(hcols), gather(rcols), dPt, gather(xicols) if gamma else np.zeros((2, t_glob)), xis
