"""Process-group plumbing for the z-slab decomposition (torch.distributed only).

The data path (ghost-plane exchange per RK stage, diagnostics all-gather) runs
inside libosbli.so over NCCL; torch.distributed is used only to start the
processes and to broadcast the 128-byte NCCL unique id from rank 0.

``slab_bounds`` mirrors the partition rule of ``osbli_create_dist`` (near-equal
slabs, the first nz % nranks ranks one plane larger); ``ghost_exchange_plan``
states which planes travel where, and ``exchange_ghosts_torch`` executes that
plan with torch.distributed point-to-point calls — used by the CPU (gloo)
tests to check the decomposition logic without a GPU.
"""
from __future__ import annotations

import os


def slab_bounds(nz: int, nranks: int, rank: int):
    """(z0, nz_local) of `rank` for a global nz split over `nranks`."""
    base, extra = divmod(nz, nranks)
    nzl = base + (1 if rank < extra else 0)
    z0 = rank * base + min(rank, extra)
    return z0, nzl


def ghost_exchange_plan(rank: int, nranks: int, nz_local: int, m: int):
    """List of (peer, send_planes, recv_planes) per direction, in local plane
    coordinates (ghosts are planes -m..-1 and nz_local..nz_local+m-1)."""
    up, dn = (rank + 1) % nranks, (rank - 1) % nranks
    return [
        (dn, (0, m), (nz_local, nz_local + m)),          # my low planes -> below; above's low -> my top ghosts
        (up, (nz_local - m, nz_local), (-m, 0)),         # my high planes -> above; below's high -> my low ghosts
    ]


def exchange_ghosts_torch(q_ghosted, m: int, rank: int, nranks: int):
    """Execute the plan on a [nz_local + 2m, ...] torch tensor (ghost planes at
    both ends) with torch.distributed (any backend).  Test utility."""
    import torch.distributed as dist
    nzl = q_ghosted.shape[0] - 2 * m
    up, dn = (rank + 1) % nranks, (rank - 1) % nranks
    lo = q_ghosted[m:2 * m].contiguous()
    hi = q_ghosted[nzl:nzl + m].contiguous()
    recv_top = q_ghosted[nzl + m:].clone()
    recv_bot = q_ghosted[:m].clone()
    # rank parity orders the blocking calls so that ring exchanges cannot deadlock
    ops = [dist.P2POp(dist.isend, lo, dn), dist.P2POp(dist.irecv, recv_top, up),
           dist.P2POp(dist.isend, hi, up), dist.P2POp(dist.irecv, recv_bot, dn)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    q_ghosted[nzl + m:] = recv_top
    q_ghosted[:m] = recv_bot
    return q_ghosted


def init_distributed():
    """Initialise torch.distributed from the torchrun environment and return
    (rank, world_size, local_rank, nccl_unique_id or None)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world == 1:
        return rank, world, local, None
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if not dist.is_initialized():
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        dist.init_process_group(backend=backend)
    uid = None
    if rank == 0:
        from .native import nccl_unique_id
        uid = nccl_unique_id()
    obj = [uid]
    dist.broadcast_object_list(obj, src=0)
    return rank, world, local, obj[0]
