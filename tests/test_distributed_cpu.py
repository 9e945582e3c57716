"""Multi-process (world_size 2 and 4, gloo, CPU) check of the multi-GPU decomposition in
paper_2302_08251_b200/distributed.py: shard ranges and the n-body positions-only exchange.

Each rank updates only its own i-range (oracle arithmetic stands in for the kernels, which
need a GPU) against the gathered positions G[world][3][S] and masses M[n], packs its new
positions into its slot, and one all-gather per step refreshes G; the result must equal a
single-process run bit for bit."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT, R32

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, steps, outdir):
    """One rank of the positions-only exchange protocol (distributed.py) with the
    oracle arithmetic standing in for the update / move kernels: own i-range only, j from the
    gathered exchange buffer G[world][3][S] and the once-gathered masses M[n]."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import lamina_oracle as O
    from paper_2302_08251_b200.distributed import all_gather_slot, exchange_shape
    S = exchange_shape(n, 1, world)
    lo, hi = rank * S, (rank + 1) * S
    init = O.nbody_init_values(42, n).astype(np.float32)  # x, y, z, m per particle
    own_pos = init[lo:hi, :3].copy()
    own_vel = np.zeros((S, 3), np.float32)
    G = torch.zeros(world * 3 * S, dtype=torch.float32)
    M = torch.zeros(n, dtype=torch.float32)
    G[rank * 3 * S:(rank + 1) * 3 * S] = torch.from_numpy(own_pos.T.reshape(-1).copy())
    M[lo:hi] = torch.from_numpy(init[lo:hi, 3].copy())
    all_gather_slot(M, rank, world)
    all_gather_slot(G, rank, world)
    for _ in range(steps):
        pos_all = G.numpy().reshape(world, 3, S).transpose(0, 2, 1).reshape(n, 3)
        vel_all = np.zeros((n, 3), np.float32)
        vel_all[lo:hi] = own_vel
        vel = O.nbody_update(pos_all, vel_all, M.numpy())
        own_vel = vel[lo:hi]
        own_pos = O.nbody_move(pos_all[lo:hi], own_vel)
        G[rank * 3 * S:(rank + 1) * 3 * S] = torch.from_numpy(np.ascontiguousarray(own_pos.T).reshape(-1))
        all_gather_slot(G, rank, world)
    vels = [torch.zeros(S * 3) for _ in range(world)]
    dist.all_gather(vels, torch.from_numpy(own_vel.reshape(-1).copy()))
    if rank == 0:
        np.savez(os.path.join(outdir, "dist.npz"), G=G.numpy(), M=M.numpy(),
                 V=np.concatenate([v.numpy().reshape(S, 3) for v in vels]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_positions_only_exchange_matches_single(tmp_path, world):
    import torch.multiprocessing as mp
    from oracle import lamina_oracle as O
    n, steps = 256, 3
    mp.spawn(_worker, args=(world, _free_port(), n, steps, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "dist.npz")
    pos, vel, mass, _ = O.nbody_run(n, steps, seed=42)
    S = n // world
    g_pos = got["G"].reshape(world, 3, S).transpose(0, 2, 1).reshape(n, 3)
    assert np.array_equal(g_pos.view(np.uint32), pos.astype(np.float32).view(np.uint32))
    assert np.array_equal(got["V"].view(np.uint32), vel.astype(np.float32).view(np.uint32))
    assert np.array_equal(got["M"].view(np.uint32), mass.astype(np.float32).view(np.uint32))


def test_exchange_pointers_address_the_slots():
    """x_r + j*elem addresses G[r][0][j - rS] for j in rank r's range, y/z follow by S, and
    every pointer lies inside G (distributed.exchange_pointers)."""
    from paper_2302_08251_b200.distributed import exchange_pointers, exchange_shape
    for n, world, elem in [(128 * 1024, 8, 4), (4096, 2, 8), (1024, 4, 4)]:
        S = exchange_shape(n, 4, world)
        base, mass = 1 << 40, 1 << 41
        ptrs = exchange_pointers(base, n, world, elem, mass)
        for r, p in enumerate(ptrs):
            for j in (r * S, r * S + S // 2, (r + 1) * S - 1):
                for d in range(3):
                    assert p[d] + j * elem == base + (3 * r * S + d * S + (j - r * S)) * elem
            assert all(x % 16 == 0 for x in p) and base <= p[0] < base + 3 * world * S * elem
            assert p[3:] == [mass] * 4
    with pytest.raises(ValueError):
        exchange_shape(1000, 32, 3)


def test_shard_ranges_partition():
    from paper_2302_08251_b200.distributed import shard_range
    for n, unit, world in [(1000, 32, 3), (128 * 1024, 32, 8), (5, 4, 2), (1 << 26, 4, 8)]:
        cuts = [shard_range(n, unit, r, world) for r in range(world)]
        assert cuts[0][0] == 0 and cuts[-1][1] == n
        for (a, b), (c, d) in zip(cuts, cuts[1:]):
            assert b == c and a % unit == 0
