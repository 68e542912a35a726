"""Process-group plumbing for the z-slab decomposition (torch.distributed only).

The data path (ghost-plane exchange per RK stage, diagnostics all-gather) runs
inside libosbli.so over NCCL; torch.distributed is used only to start the
processes and to broadcast the 128-byte NCCL unique id from rank 0.

The partition rule and the ghost plan live in the C library
(``osbli_slab_bounds``, ``osbli_ghost_plan``; host-only functions);
``exchange_ghosts_torch`` executes that plan with torch.distributed
point-to-point calls — used by the CPU (gloo) tests to check the
decomposition logic without a GPU.
"""
from __future__ import annotations

import os


def exchange_ghosts_torch(q_ghosted, m: int, rank: int, nranks: int, symz: bool = False):
    """Execute the library's ghost plan (osbli_ghost_plan_sym) on a
    [nz_local + 2m, 5, ...] torch tensor (ghost planes at both ends) with
    torch.distributed point-to-point calls (any backend); with symmetry in z the
    outer faces get the mirrored own planes (field 3, rho u_z, negated), as the
    library's mirror kernel does.  The CPU (gloo) tests use it to check the
    decomposition logic of the C library."""
    import torch.distributed as dist

    from .native import ghost_plan
    nzl = q_ghosted.shape[0] - 2 * m
    plan = ghost_plan(rank, nranks, nzl, m, symz)
    ops, recvs = [], []
    for send_peer, send_plane, recv_peer, recv_plane in plan:
        if send_peer >= 0:
            buf = q_ghosted[send_plane + m:send_plane + 2 * m].contiguous()
            ops.append(dist.P2POp(dist.isend, buf, send_peer))
        if recv_peer >= 0:
            rbuf = q_ghosted[recv_plane + m:recv_plane + 2 * m].clone()
            ops.append(dist.P2POp(dist.irecv, rbuf, recv_peer))
            recvs.append((recv_plane, rbuf))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    for recv_plane, rbuf in recvs:
        q_ghosted[recv_plane + m:recv_plane + 2 * m] = rbuf
    sign = None
    for side, (_, _, recv_peer, _) in ((1, plan[0]), (0, plan[1])):
        if recv_peer >= 0:
            continue
        if sign is None:
            sign = q_ghosted.new_ones(q_ghosted.shape[1:])
            sign[3] = -1.0
        for k in range(1, m + 1):  # ghost -k <- k-1 (low), nzl-1+k <- nzl-k (high)
            g, i = (m - k, m + k - 1) if side == 0 else (m + nzl - 1 + k, m + nzl - k)
            q_ghosted[g] = sign * q_ghosted[i]
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
