"""Run under torchrun (gloo, ranks may share a GPU): the fused p2p n-body step over CUDA IPC
equals the single-view run bit for bit in exact mode.  Rank 0 prints OK or FAIL."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2302_08251_b200 import lamina as L  # noqa: E402
from paper_2302_08251_b200.distributed import nbody_distributed  # noqa: E402

dist.init_process_group("gloo")
rank = dist.get_rank()
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
layout, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
view, _ = nbody_distributed(layout, n, steps, mode=0, seed=42, transport="p2p")
got = [b.copy() for b in view.download_all()]
R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"
ref = L.View(L.Layout(R32, f"i64:[{n}]", layout))
ref.nbody_init(42)
for _ in range(steps):
    ref.nbody_update(0)
    ref.nbody_move()
ok = all(np.array_equal(a, b) for a, b in zip(got, ref.download_all()))
oks = [None] * dist.get_world_size()
dist.all_gather_object(oks, ok)
if rank == 0:
    print("OK" if all(oks) else f"FAIL {oks}")
dist.destroy_process_group()
