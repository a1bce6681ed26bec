"""The two per-step collectives of the member-sharded scheme.

With members sharded contiguously over ranks (one GPU each), a time-step
needs exactly two exchanges, both over the whole process group:

  1. allreduce SUM of the member-summed fields [sum_j v_j | sum_j w_j]
     (2 n_vel doubles) -> every rank gets the ensemble means that drive the
     shared matrices and the fluctuations (`ensemble.py:216-224`);
  2. allreduce MAX of the per-rank maxima max_j |z'_j(x_q)|^2 at every
     quadrature point for both families (2 nt 7 doubles) -> the eddy
     viscosity nu_T of both shared matrices (`ensemble.py:227-238`).

Everything else (right-hand sides, the replicated matrix assembly and
factorisation, the column-batched solve) is rank-local.  Over NCCL on one
B200 node these run on the NVLink/NVSwitch fabric; the same calls run over
gloo on CPU tensors in the tests.
"""

from __future__ import annotations

import torch.distributed as dist


def member_slice(J_total: int, rank: int, world: int):
    """(first member, count) of a rank's contiguous shard."""
    base, extra = divmod(J_total, world)
    j0 = rank * base + min(rank, extra)
    return j0, base + (1 if rank < extra else 0)


def allreduce_member_sums(sums, comm=None):
    """In place: sums <- sum over ranks (exchange 1)."""
    if comm is not None:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=comm)
    return sums


def allreduce_eddy_max(maxsq, comm=None):
    """In place: maxsq <- max over ranks (exchange 2)."""
    if comm is not None:
        dist.all_reduce(maxsq, op=dist.ReduceOp.MAX, group=comm)
    return maxsq


def allreduce_max_scalar(value: float, comm=None, device=None) -> float:
    return allreduce_max_values([value], comm, device)[0]


_SCALAR_BUFS = {}


def allreduce_max_values(values, comm=None, device=None):
    """Elementwise max over ranks of a few host scalars (one small collective).

    Persistent pinned host / device buffers per (device, count): one async H2D, the
    collective, one async D2H and a single stream synchronisation."""
    if comm is None:
        return list(values)
    import torch
    if device is None or torch.device(device).type != "cuda":   # gloo / CPU tensors (tests)
        t = torch.tensor(list(values), dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=comm)
        return [float(x) for x in t.tolist()]
    n = len(values)
    key = (str(device), n)
    bufs = _SCALAR_BUFS.get(key)
    if bufs is None:
        bufs = (torch.zeros(n, dtype=torch.float64, pin_memory=True),
                torch.zeros(n, dtype=torch.float64, device=device),
                torch.zeros(n, dtype=torch.float64, pin_memory=True))
        _SCALAR_BUFS[key] = bufs
    h_in, d, h_out = bufs
    h_in.numpy()[:] = values
    d.copy_(h_in, non_blocking=True)
    dist.all_reduce(d, op=dist.ReduceOp.MAX, group=comm)
    h_out.copy_(d, non_blocking=True)
    torch.cuda.current_stream(d.device).synchronize()
    return [float(x) for x in h_out.numpy()]
