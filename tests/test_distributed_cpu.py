"""Multi-process (world_size 2, gloo, CPU) check of the multi-GPU decomposition in
paper_2302_08251_b200/distributed.py: shard ranges + all-gather of blob-stream regions.

Each rank updates only its own i-range of the n-body state (oracle arithmetic stands in
for the kernels, which need a GPU), then the ranks all-gather their regions; the
replicated blobs must equal a single-process run byte for byte."""
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


def _worker(rank, world, port, layout, n, steps, outdir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import lamina_oracle as O
    from paper_2302_08251_b200 import lamina as L
    from paper_2302_08251_b200.distributed import allgather_regions, shard_range
    lay = L.Layout(R32, f"i64:[{n}]", layout)
    m = O.make(R32, f"i64:[{n}]", layout)
    init = O.nbody_init_values(42, n)
    vals = np.zeros((n, 7), np.float32)
    vals[:, :3] = init[:, :3]
    vals[:, 6] = init[:, 3]
    blobs_np = O.zero_blobs(m)
    O.write_all(m, blobs_np, vals.view(np.uint32).astype(np.uint64))
    blobs = [torch.from_numpy(b) for b in blobs_np]
    lo, hi = shard_range(n, lay.shard_unit, rank, world)
    for _ in range(steps):
        cur = O.read_all(m, [b.numpy() for b in blobs]).astype(np.uint32).view(np.float32)
        vel = O.nbody_update(cur[:, :3], cur[:, 3:6], cur[:, 6])
        nxt = cur.copy()
        nxt[lo:hi, 3:6] = vel[lo:hi]
        nxt[lo:hi, :3] = O.nbody_move(cur[lo:hi, :3], vel[lo:hi])
        O.write_all(m, [b.numpy() for b in blobs], nxt.view(np.uint32).astype(np.uint64))
        allgather_regions(lay, blobs, world)
    if rank == 0:
        np.savez(os.path.join(outdir, "dist.npz"), *[b.numpy() for b in blobs])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("layout", ["aos-packed", "soa-mb", "aosoa:8", "soa-sb"])
def test_sharded_nbody_allgather_matches_single(tmp_path, layout):
    import torch.multiprocessing as mp
    from oracle import lamina_oracle as O
    n, steps = 256, 2
    mp.spawn(_worker, args=(2, _free_port(), layout, n, steps, str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "dist.npz")
    pos, vel, mass, _ = O.nbody_run(n, steps, seed=42)
    m = O.make(R32, f"i64:[{n}]", layout)
    want = O.zero_blobs(m)
    v = np.concatenate([pos, vel, mass[:, None]], axis=1).astype(np.float32)
    O.write_all(m, want, v.view(np.uint32).astype(np.uint64))
    for k, b in enumerate(want):
        assert np.array_equal(got[f"arr_{k}"], b), f"blob {k}"


def test_shard_ranges_partition():
    from paper_2302_08251_b200.distributed import shard_range
    for n, unit, world in [(1000, 32, 3), (128 * 1024, 32, 8), (5, 4, 2), (1 << 26, 4, 8)]:
        cuts = [shard_range(n, unit, r, world) for r in range(world)]
        assert cuts[0][0] == 0 and cuts[-1][1] == n
        for (a, b), (c, d) in zip(cuts, cuts[1:]):
            assert b == c and a % unit == 0
