"""Multi-GPU decomposition of the hot path, one process per GPU.

* copy / pack / instrument: every rank owns the element range `shard_range(...)` of every blob;
  no collective (weak scaling, `lam_copy_range`).
* n-body: every rank holds the whole view, updates Vel / moves Pos of its own i-range, then the
  ranks all-gather the byte regions their ranges occupy in each blob stream (NCCL over NVLink on
  GPUs, gloo in the CPU tests).  Per-i arithmetic is independent of the sharding, so the result
  is bit-identical to one GPU in exact mode.
"""
from __future__ import annotations


def shard_range(n: int, unit: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of rank's shard: equal multiples of `unit`, the last rank takes the rest."""
    per = (n // world) // unit * unit
    lo = rank * per
    hi = n if rank == world - 1 else lo + per
    return lo, hi


def stream_regions(layout, lo: int, hi: int):
    """[(nr, byte_lo, byte_hi)] per blob stream for elements [lo, hi)."""
    return [layout.stream_region(s, lo, hi) for s in range(layout.stream_count)]


def allgather_regions(layout, blobs, world: int, group=None):
    """All-gather every rank's shard regions into the replicated blobs (torch uint8 tensors).

    Needs equal shards: element count a multiple of world * shard_unit.
    """
    import torch.distributed as dist
    n = layout.element_count
    unit = layout.shard_unit
    if n % (world * unit):
        raise ValueError(f"n-body all-gather needs n ({n}) to be a multiple of world*shard_unit ({world * unit})")
    per = n // world
    rank = dist.get_rank(group)
    for s in range(layout.stream_count):
        nr, a0, _ = layout.stream_region(s, 0, per)
        _, _, b_last = layout.stream_region(s, (world - 1) * per, n)
        _, lo, hi = layout.stream_region(s, rank * per, (rank + 1) * per)
        if hi <= lo:
            continue
        out = blobs[nr][a0:b_last]
        piece = blobs[nr][lo:hi]
        if out.numel() != world * piece.numel():
            raise ValueError("stream regions are not equal per rank")
        dist.all_gather_into_tensor(out, piece.clone() if out.device.type == "cpu" else piece, group=group)


def nbody_distributed(layout_text: str, n: int, steps: int, mode: int = 0, seed: int = 42, f64: bool = False,
                      group=None, transport: str = "allgather"):
    """Run the n-body benchmark with the particles sharded over the process group.

    transport "allgather": every rank updates and moves its i-shard, then the shards' blob
    regions are all-gathered (NCCL over NVLink).  transport "p2p": the fused step -- every
    rank maps its peers' views (CUDA IPC) and the update kernel reads their positions over
    NVLink directly (lam_nbody_update_multi); a barrier separates update and move.

    Returns (view, blobs): the view holds the whole replicated state after the last step.
    """
    if transport == "p2p":
        return _nbody_p2p(layout_text, n, steps, mode, seed, f64, group)
    import torch
    import torch.distributed as dist

    from . import lamina as L
    t = "f64" if f64 else "f32"
    schema = f"Record{{Pos:Record{{x:{t},y:{t},z:{t}}},Vel:Record{{x:{t},y:{t},z:{t}}},Mass:{t}}}"
    lay = L.Layout(schema, f"i64:[{n}]", layout_text)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = torch.cuda.current_device()
    blobs = [torch.zeros(max(16, s), dtype=torch.uint8, device="cuda") for s in lay.blob_sizes]
    view = L.View(lay, device=dev, blobs=[b.data_ptr() for b in blobs], blob_bytes=lay.blob_sizes)
    view.nbody_init(seed)
    lo, hi = shard_range(n, lay.shard_unit, rank, world)
    stream = torch.cuda.current_stream()
    for _ in range(steps):
        view.nbody_update(mode, lo, hi, stream=stream)
        view.nbody_move(lo, hi, stream=stream)
        allgather_regions(lay, blobs, world, group)
    torch.cuda.synchronize()
    return view, blobs


def _nbody_p2p(layout_text, n, steps, mode, seed, f64, group):
    import torch
    import torch.distributed as dist

    from . import lamina as L
    t = "f64" if f64 else "f32"
    schema = f"Record{{Pos:Record{{x:{t},y:{t},z:{t}}},Vel:Record{{x:{t},y:{t},z:{t}}},Mass:{t}}}"
    lay = L.Layout(schema, f"i64:[{n}]", layout_text)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = torch.cuda.current_device()
    view = L.View(lay, device=dev)  # cudaMalloc'd blobs: IPC handles cover them exactly
    view.nbody_init(seed)
    torch.cuda.synchronize()
    handles = [L.ipc_handle(view.blob_ptr(nr)) for nr in range(lay.blob_count) if lay.blob_sizes[nr]]
    everyone = [None] * world
    dist.all_gather_object(everyone, handles, group=group)
    ranges = [shard_range(n, lay.shard_unit, r, world) for r in range(world)]
    peers, mapped = {}, []
    for r in range(world):
        if r == rank:
            continue
        ptrs = [L.ipc_open(h, dev) for h in everyone[r]]
        mapped += ptrs
        peers[r] = L.View(lay, device=dev, blobs=ptrs, blob_bytes=[s for s in lay.blob_sizes if s])
    sources = [(view if r == rank else peers[r], lo, hi) for r, (lo, hi) in enumerate(ranges)]
    lo, hi = ranges[rank]
    for _ in range(steps):
        view.nbody_update_from(sources, mode, lo, hi)
        torch.cuda.synchronize()
        dist.barrier(group=group)  # every rank has read the positions before anyone moves
        view.nbody_move(lo, hi)
        torch.cuda.synchronize()
        dist.barrier(group=group)
    for r, pv in peers.items():  # replicate the final state locally (NVLink reads)
        L.copy_view_range(pv, view, *ranges[r])
    torch.cuda.synchronize()
    dist.barrier(group=group)
    del peers
    for p in mapped:
        L.ipc_close(p)
    return view, None
