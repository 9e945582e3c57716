"""Multi-GPU decomposition of the hot path, one process per GPU.

* copy / pack / instrument: every rank owns the element range `shard_range(...)` of every blob;
  no collective (weak scaling, `lam_copy_range`).
* n-body (transport "allgather", the SURVEY §8e plan): every rank owns the i-range
  [r*S, (r+1)*S) of the particles in the chosen mapping.  Per step it updates Vel of its
  i-range against all j, moves its Pos, packs its positions as SoA x,y,z (12 B/particle for
  f32) into its slot of a replicated exchange buffer G[world][3][S], and ONE all-gather
  (NCCL over NVLink) refreshes G everywhere.  Mass is constant: gathered once at init into
  M[n].  The update reads j from G and M through one soa-mb view per rank slot (blob
  pointers into G, `exchange_pointers`), visited in global j order, so exact mode is
  bit-identical to one GPU.
* transport "p2p": the fused step -- peers' blobs are mapped with CUDA IPC and read over
  NVLink inside the update kernel (`lam_nbody_update_multi`), no gathered copy.
"""
from __future__ import annotations

import math


def shard_range(n: int, unit: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of rank's shard: equal multiples of `unit`, the last rank takes the rest."""
    per = (n // world) // unit * unit
    lo = rank * per
    hi = n if rank == world - 1 else lo + per
    return lo, hi


def exchange_shape(n: int, unit: int, world: int) -> int:
    """Particles per rank S of the positions-only exchange (equal shards, S a multiple of the
    layout's shard unit and of 4 so every slot pointer stays 16-byte aligned)."""
    u = unit * 4 // math.gcd(unit, 4)
    if n % (world * u):
        raise ValueError(f"n-body all-gather needs n ({n}) to be a multiple of world*unit ({world * u})")
    return n // world


def exchange_pointers(base: int, n: int, world: int, elem: int, mass_base: int):
    """Blob pointers of the soa-mb j-view of rank slot r of G[world][3][S] (S = n/world):
    x_r = G + (3rS - rS)*elem, so x_r + j*elem addresses G[r][0][j - rS] for j in [rS, (r+1)S);
    y_r = x_r + S*elem, z_r = x_r + 2S*elem.  Vel (never read by the update) and Mass point
    at M[n].  Every pointer stays inside G."""
    S = n // world
    out = []
    for r in range(world):
        x = base + 2 * r * S * elem
        out.append([x, x + S * elem, x + 2 * S * elem, mass_base, mass_base, mass_base, mass_base])
    return out


def world_rank(group=None) -> tuple[int, int]:
    """(world size, rank) of the group; (1, 0) without an initialised process group."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def all_gather_slot(buf, rank: int, world: int, group=None):
    """In-place all-gather of rank's equal slot of `buf` (1-D tensor) into every slot: NCCL
    all-gather on CUDA tensors; staged through host memory for gloo (CPU tests)."""
    import torch.distributed as dist
    if world == 1:
        return
    per = buf.numel() // world
    slot = buf[rank * per:(rank + 1) * per]
    if buf.device.type == "cuda" and dist.get_backend(group) == "nccl":
        # a separate send buffer (per * elem bytes, 1.5 MiB / world at 128K) rather than relying
        # on NCCL's in-place convention through a view of the output
        dist.all_gather_into_tensor(buf, slot.clone(), group=group)
        return
    host = buf.cpu()
    dist.all_gather_into_tensor(host, host[rank * per:(rank + 1) * per].clone(), group=group)
    buf.copy_(host)


def nbody_distributed(layout_text: str, n: int, steps: int, mode: int = 0, seed: int = 42, f64: bool = False,
                      group=None, transport: str = "allgather", timing: dict | None = None):
    """Run the n-body benchmark with the particles sharded over the process group.

    transport "allgather": positions-only exchange (module docstring), one all-gather per step.
    transport "p2p": the fused step over CUDA IPC (see `_nbody_p2p`).
    With `timing` (a dict), per-step CUDA-event times are recorded: update_ms, move_ms,
    exchange_ms (pack + all-gather), step_ms.

    Returns (view, exchange): the view's own i-range [r*S, (r+1)*S) holds the rank's final
    state; for "allgather" exchange = (G, M), the replicated final positions and masses.
    """
    if transport == "p2p":
        return _nbody_p2p(layout_text, n, steps, mode, seed, f64, group)
    import torch

    from . import lamina as L
    t = "f64" if f64 else "f32"
    schema = f"Record{{Pos:Record{{x:{t},y:{t},z:{t}}},Vel:Record{{x:{t},y:{t},z:{t}}},Mass:{t}}}"
    lay = L.Layout(schema, f"i64:[{n}]", layout_text)
    world, rank = world_rank(group)
    dev = torch.cuda.current_device()
    S = exchange_shape(n, lay.shard_unit, world)
    lo, hi = rank * S, (rank + 1) * S
    dtype = torch.float64 if f64 else torch.float32
    elem = 8 if f64 else 4
    view = L.View(lay, device=dev)
    view.nbody_init(seed)
    stream = torch.cuda.current_stream()
    G = torch.empty(world * 3 * S, dtype=dtype, device="cuda")
    M = torch.empty(n, dtype=dtype, device="cuda")
    tmp = torch.empty(4 * S, dtype=dtype, device="cuda")
    view.nbody_pack_positions(lo, hi, tmp.data_ptr(), with_mass=True, stream=stream)
    G[rank * 3 * S:(rank + 1) * 3 * S].copy_(tmp[:3 * S])
    M[lo:hi].copy_(tmp[3 * S:])
    del tmp
    all_gather_slot(M, rank, world, group)  # Mass once
    all_gather_slot(G, rank, world, group)
    soa = L.Layout(schema, f"i64:[{n}]", "soa-mb")
    jviews = [L.View(soa, device=dev, blobs=p, blob_bytes=[n * elem] * 7)
              for p in exchange_pointers(G.data_ptr(), n, world, elem, M.data_ptr())]
    sources = [(jviews[r], r * S, (r + 1) * S) for r in range(world)]
    slot = G[rank * 3 * S:(rank + 1) * 3 * S]
    ev = []
    for _ in range(steps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timing is not None else None
        if e:
            e[0].record(stream)
        view.nbody_update_from(sources, mode, lo, hi, stream=stream)
        if e:
            e[1].record(stream)
        view.nbody_move(lo, hi, stream=stream)
        if e:
            e[2].record(stream)
        view.nbody_pack_positions(lo, hi, slot.data_ptr(), stream=stream)
        all_gather_slot(G, rank, world, group)
        if e:
            e[3].record(stream)
            ev.append(e)
    torch.cuda.synchronize()
    if timing is not None and ev:
        k = len(ev)
        timing["update_ms"] = sum(e[0].elapsed_time(e[1]) for e in ev) / k
        timing["move_ms"] = sum(e[1].elapsed_time(e[2]) for e in ev) / k
        timing["exchange_ms"] = sum(e[2].elapsed_time(e[3]) for e in ev) / k
        timing["step_ms"] = sum(e[0].elapsed_time(e[3]) for e in ev) / k
        timing["exchange_bytes_per_step"] = 3 * n * elem
    del jviews
    return view, (G, M)


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
