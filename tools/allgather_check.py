"""Run under torchrun (ranks may share a GPU; gloo stages the all-gather through the host):
nbody_distributed(transport="allgather") -- the positions-only exchange with the real kernels --
against a single-view run.  Exact mode: the gathered positions and every rank's own shard
(all 7 leaves) are bit-identical; fast mode: within the n-body fast tolerance.
Rank 0 prints OK or FAIL."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2302_08251_b200 import lamina as L  # noqa: E402
from paper_2302_08251_b200.distributed import nbody_distributed  # noqa: E402

dist.init_process_group(os.environ.get("LAMB_DIST_BACKEND", "gloo"))
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
layout, n, steps, mode = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
view, (G, M) = nbody_distributed(layout, n, steps, mode=mode, seed=42, transport="allgather")
S = n // world
lo, hi = rank * S, (rank + 1) * S
R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"
ref = L.View(L.Layout(R32, f"i64:[{n}]", layout))
ref.nbody_init(42)
for _ in range(steps):
    ref.nbody_update(mode)
    ref.nbody_move()
idx = np.arange(lo, hi)
leaves = np.arange(7)
mine = view.read_values(np.repeat(idx, 7), np.tile(leaves, S)).reshape(S, 7).astype(np.uint32).view(np.float32)
want = ref.read_values(np.repeat(idx, 7), np.tile(leaves, S)).reshape(S, 7).astype(np.uint32).view(np.float32)
allp = ref.read_values(np.repeat(np.arange(n), 3), np.tile(np.arange(3), n)).reshape(n, 3).astype(np.uint32)
gpos = G.cpu().numpy().reshape(world, 3, S).transpose(0, 2, 1).reshape(n, 3).view(np.uint32)
if mode == 0:
    ok = np.array_equal(mine.view(np.uint32), want.view(np.uint32)) and np.array_equal(gpos, allp)
else:
    a, b = mine.astype(np.float64), want.astype(np.float64)
    ok = bool((np.abs(a - b) / np.maximum(1.0, np.abs(b))).max() <= 2e-6)
oks = [None] * world
dist.all_gather_object(oks, bool(ok))
if rank == 0:
    print("OK" if all(oks) else f"FAIL {oks}")
dist.destroy_process_group()
