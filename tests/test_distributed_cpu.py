"""Host logic of the z-slab decomposition, on the CPU (no GPU): the C library's
partition rule and ghost-exchange plan (osbli_slab_bounds, osbli_ghost_plan),
executed with torch.distributed (gloo, world size 2 and 3)."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_slab_partition_covers_every_plane_once():
    from paper_1609_01277_b200 import slab_bounds
    for nz in (1, 7, 64, 255, 256, 1024):
        for nranks in (1, 2, 3, 4, 7, 8):
            if nranks > nz:
                continue
            owned = []
            sizes = []
            for r in range(nranks):
                z0, n = slab_bounds(nz, nranks, r)
                owned.extend(range(z0, z0 + n))
                sizes.append(n)
            assert owned == list(range(nz))
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("nranks", [2, 3, 5, 8])
def test_ghost_plan_is_a_consistent_ring(nranks):
    """Rank r's transfer-t send goes to the peer whose transfer-t receive names r,
    and the planes sent are the ones the receiver's ghosts stand for."""
    from paper_1609_01277_b200 import ghost_plan, slab_bounds
    nz, m = 8 * nranks + 3, 4
    sizes = [slab_bounds(nz, nranks, r)[1] for r in range(nranks)]
    z0s = [slab_bounds(nz, nranks, r)[0] for r in range(nranks)]
    plans = [ghost_plan(r, nranks, sizes[r], m) for r in range(nranks)]
    for r in range(nranks):
        for t in range(2):
            sp, splane, _, _ = plans[r][t]
            _, _, rp, rplane = plans[sp][t]
            assert rp == r
            # global plane index of what is sent == what the receiver's ghost represents
            sent_global = (z0s[r] + splane) % nz
            ghost_global = (z0s[sp] + rplane) % nz
            assert sent_global == ghost_global


def _worker(rank, world, port, nz, m, q, symz=False):
    import torch
    import torch.distributed as dist

    from paper_1609_01277_b200 import exchange_ghosts_torch, slab_bounds
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    rng = np.random.default_rng(1234)
    glob = rng.standard_normal((nz, 5, 6, 7))  # plane-major [z][f][y][x], same on all ranks
    z0, nzl = slab_bounds(nz, world, rank)
    loc = torch.full((nzl + 2 * m, 5, 6, 7), float("nan"), dtype=torch.float64)
    loc[m:m + nzl] = torch.from_numpy(glob[z0:z0 + nzl])
    exchange_ghosts_torch(loc, m, rank, world, symz)
    if symz:
        # mirror about the domain faces: rho u_z (field 3) odd
        exp = []
        for k in range(-m, nzl + m):
            g = z0 + k
            src, s = (-1 - g, -1.0) if g < 0 else ((2 * nz - 1 - g, -1.0) if g >= nz else (g, 1.0))
            plane = glob[src].copy()
            plane[3] *= s
            exp.append(plane)
        ok = bool(np.array_equal(loc.numpy(), np.stack(exp)))
    else:
        idx = [(z0 + k) % nz for k in range(-m, nzl + m)]
        ok = bool(np.array_equal(loc.numpy(), glob[idx]))
    q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nz,m", [(2, 24, 6), (3, 31, 4), (2, 12, 6)])
def test_gloo_ghost_exchange_matches_periodic_neighbours(world, nz, m):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nz, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


@pytest.mark.parametrize("world,nz,m", [(2, 24, 6), (3, 31, 4), (4, 40, 2)])
def test_gloo_ghost_exchange_with_symmetry_in_z(world, nz, m):
    """The symmetric-z plan (osbli_ghost_plan_sym): no transfer across the periodic
    wrap (sends and receives still pair up), the outer faces mirrored."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nz, m, q, True))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
