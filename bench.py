#!/usr/bin/env python
"""Benchmark of the B200 layout-copy hot path (BASELINE.json config C2).

Step = one pass of lamina::copyView over all 25 ordered pairs of
{aos-packed, soa-sb, soa-mb, aosoa:8, aosoa:32} on 2^26 n-body records
(Record{Pos{x,y,z},Vel{x,y,z},Mass}, 7 x f32 = 28 B) per GPU.  5 pairs take the
reference's blob-memcpy path (view.cpp:175-181), 20 the fieldwise layout transpose.
Algorithmic bytes = source leaf bytes read + destination leaf bytes written
= 56 B per record per pair.

  value  : whole-job GB/s, device-resident views, CUDA events, max over ranks
  e2e    : same metric through lam_copy_host (host pinned blobs in and out, H2D/D2H
           inside the timed region)
  roofline: dominant kernel k_vec_transpose<7,4>, algorithmic bytes / mean launch time vs
           the measured HBM copy peak (MEASURED_PEAKS.json)
  parity : after the timed region, every pair's destination is checked bit-exactly against the
           reference copyView on three 2^20-record ranges (checker leg)
  cpu_baseline: the reference itself (oracle/_ref, compiled from /root/reference) on a
           bounded sample (2^24 records x 25 pairs), all host threads

--impl reference : the reference's copyView (oracle/_ref) on the SAME workload (2^26 records x
                   25 pairs per step), all host threads over disjoint index ranges.
--suite          : additionally time configs C1, C3, C5 and n-body (C4) on this GPU.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"
R64 = "Record{Pos:Record{x:f64,y:f64,z:f64},Vel:Record{x:f64,y:f64,z:f64},Mass:f64}"
C2_LAYOUTS = ["aos-packed", "soa-sb", "soa-mb", "aosoa:8", "aosoa:32"]
METRIC = "layout-copy and bitpack GB/s (frac of HBM peak) at 1/2/4/8 B200; n-body interactions/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p.get("hbm_gbs", 6650.0)), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled through NVML every 20 ms during
    the timed region (same fields as `nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.*`)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.sm, self.mask, self.max = [], 0, None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self._physical_index())
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._nv = None
        return self

    def _physical_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[self.gpu])
            except (ValueError, IndexError):
                pass
        return self.gpu

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.mask |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            time.sleep(0.02)

    def __exit__(self, *a):
        self._stop.set()
        if getattr(self, "_nv", None):
            self._t.join(timeout=1)

    def summary(self):
        reasons = sorted(k for k, bit in self.REASONS.items() if self.mask & bit)
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None,
                "sm_max_mhz": float(self.max) if self.max else None, "reasons": reasons, "samples": len(self.sm)}


def dist_setup():
    """One process per GPU (torchrun env).  LAMB_DIST_BACKEND=gloo with more ranks than GPUs
    (ranks share devices round-robin) exercises the multi-rank path on a one-GPU box; the
    numbers are then not a scaling measurement."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = os.environ.get("LAMB_DIST_BACKEND", "nccl")
        if backend != "nccl":
            local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


SPECIAL_U32 = (0x7FC00000, 0xFFC00000, 0x7F800001, 0xFFA00001, 0x7F800000, 0xFF800000, 0x00000001, 0x80000001,
               0x007FFFFF, 0x80000000, 0x00000000)


def fill_source(L, view, n, seed):
    """Synthetic source content: full-range random u32 patterns per (i, f), with about 1 in 50
    values replaced by NaN / sNaN / +-0 / denormal / Inf patterns (a layout copy is a byte
    permutation, so every pattern must survive).  Generated in aos-packed on the device, then
    copied into `view` by the library; device-synchronised on both sides, so the zero-fill of
    the view (lam_view_alloc), the generator and the copy never overlap."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    raw = torch.randint(-2**31, 2**31, (n * 7,), device="cuda", dtype=torch.int32, generator=g)
    pick = torch.randint(0, 50, (n * 7,), device="cuda", generator=g) == 0
    special = torch.tensor([x - 2**32 if x >= 2**31 else x for x in SPECIAL_U32], device="cuda", dtype=torch.int32)
    raw = torch.where(pick, special[torch.randint(0, len(SPECIAL_U32), (n * 7,), device="cuda", generator=g)], raw)
    raw = raw.view(torch.uint8)
    aos = L.Layout(R32, f"i32:[{n}]", "aos-packed")
    torch.cuda.synchronize()
    tmp = L.View(aos, blobs=[raw.data_ptr()], blob_bytes=[raw.numel()])
    L.copy_view(tmp, view)
    torch.cuda.synchronize()
    del tmp, raw


def run_c2(L, n, steps, warmup, world, local):
    import torch
    stream = torch.cuda.Stream()
    ext = f"i32:[{n}]"
    lays = {a: L.Layout(R32, ext, a) for a in C2_LAYOUTS}
    srcs = {a: L.View(lays[a], device=local) for a in C2_LAYOUTS}
    dsts = {a: L.View(lays[a], device=local) for a in C2_LAYOUTS}
    for k, a in enumerate(C2_LAYOUTS):
        fill_source(L, srcs[a], n, 1234 + k)
    pairs = [(a, b) for a in C2_LAYOUTS for b in C2_LAYOUTS]
    bytes_pair = 56 * n
    ev = [{p: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for p in pairs}
          for _ in range(steps)]
    for _ in range(warmup):
        for a, b in pairs:
            L.copy_view(srcs[a], dsts[b], stream=stream)
    torch.cuda.synchronize()
    barrier(world)
    launches0 = L.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier(world)
        e0.record(stream)
        for s in range(steps):
            for p in pairs:
                ev[s][p][0].record(stream)
                L.copy_view(srcs[p[0]], dsts[p[1]], stream=stream)
                ev[s][p][1].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    launches = L.launch_count() - launches0
    total_ms = e0.elapsed_time(e1)
    pair_ms = {p: sum(ev[s][p][0].elapsed_time(ev[s][p][1]) for s in range(steps)) for p in pairs}
    ms_max = max_over_ranks(total_ms / steps, world)
    bytes_step = bytes_pair * len(pairs)
    value = sum_over_ranks(bytes_step, world) / (ms_max * 1e-3) / 1e9
    cross = [p for p in pairs if p[0] != p[1]]
    tile_ms = sum(pair_ms[p] for p in cross) / (steps * len(cross))
    achieved = bytes_pair / (tile_ms * 1e-3) / 1e9
    per_pair = {f"{a}->{b}": round(bytes_pair / (pair_ms[(a, b)] / steps * 1e-3) / 1e9, 1) for a, b in pairs}
    out = {"ms_per_step": ms_max, "value": value, "launches": launches, "clocks": clk.summary(),
           "achieved_tile": achieved, "tile_ms": tile_ms, "per_pair_gbs": per_pair, "bytes_step": bytes_step,
           "wall_ms_per_step": total_ms / steps, "views": (srcs, dsts)}
    return out


def run_c2_e2e(L, n, steps, local, world=1):
    """Same workload through lam_copy_host: pinned host blobs, H2D + copy + D2H per pair.

    Every rank runs it at once on its own GPU and host buffers; the step time is the max over
    ranks (barrier on both sides) and the value is all ranks' bytes over that time.  Host
    buffers are shared between the source and destination roles of a layout (the timing does
    not depend on the values), so one rank pins 5 x 28 B x n.
    """
    import torch
    ext = f"i32:[{n}]"
    lays = {a: L.Layout(R32, ext, a) for a in C2_LAYOUTS}
    rng = np.random.default_rng(7 + local)
    host = {}
    for a in C2_LAYOUTS:
        blobs = []
        for s in lays[a].blob_sizes:
            t = torch.empty(s, dtype=torch.uint8, pin_memory=True)
            arr = t.numpy()
            arr[:] = rng.integers(0, 256, s, dtype=np.uint8)
            blobs.append((t, arr))
        host[a] = blobs
    pairs = [(a, b) for a in C2_LAYOUTS for b in C2_LAYOUTS]
    h2d = sum(sum(lays[a].blob_sizes) for a, b in pairs)
    d2h = sum(sum(lays[b].blob_sizes) for a, b in pairs)

    def step():
        for a, b in pairs:
            if a == b:  # same-layout copyView into a second buffer set would double the pinning;
                src = [x for _, x in host[a]]  # the memcpy path streams blob -> blob in place
                L.copy_view_host(lays[a], src, lays[b], src, device=local)
            else:
                L.copy_view_host(lays[a], [x for _, x in host[a]], lays[b], [x for _, x in host[b]], device=local)
    step()  # warm-up: one untimed pass over every pair (pipeline slots, per-pair device images)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = max_over_ranks((time.perf_counter() - t0) / steps, world)
    link = pcie_bandwidth(local)
    moved = (h2d + d2h) / dt / 1e9
    return {"value": 56 * n * len(pairs) * world / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": int(h2d) * world,
            "d2h_bytes_per_step": int(d2h) * world, "s_per_step": dt, "records_per_gpu": n,
            "api": "lam_copy_host (pinned host blobs), all ranks concurrently, max over ranks",
            "host_link_GBps": link, "transfer_GBps_per_gpu": moved,
            "frac_of_link": moved / link["bidirectional"] if link.get("bidirectional") else None}


def pcie_bandwidth(local, nbytes=1 << 30):
    """Host link roofline of the e2e number: pinned H2D, D2H and both at once (copy engines)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{local}")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{local}")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    t_h2d = timed(lambda: d.copy_(h, non_blocking=True))
    t_d2h = timed(lambda: h2.copy_(d2, non_blocking=True))
    t_bi = timed(both)
    return {"h2d": nbytes / t_h2d / 1e9, "d2h": nbytes / t_d2h / 1e9, "bidirectional": 2 * nbytes / t_bi / 1e9}


class RefC2:
    """The reference's copyView (oracle/_ref, the unmodified lamina library) over the 25 C2
    pairs on resident reference views of n records: 5 sources (random u32 patterns, aos-packed
    drawn once and copied into the other layouts by the reference) and 5 destinations.  One
    step = 25 copyView calls; nthreads > 1 runs the loop body over disjoint index ranges
    (SURVEY 8(d) variant ii; the same-layout pairs take the blob-memcpy path split by bytes)."""

    def __init__(self, n, nthreads, seed=3):
        from oracle import ref
        ext = f"i32:[{n}]"
        self.n, self.nthreads = n, nthreads
        self.src = {a: ref.RefView(R32, ext, a) for a in C2_LAYOUTS}
        self.dst = {a: ref.RefView(R32, ext, a) for a in C2_LAYOUTS}
        rng = np.random.default_rng(seed)
        blob = self.src["aos-packed"].blobs[0].view(np.uint32)
        step = 1 << 24
        for lo in range(0, blob.size, step):
            blob[lo:lo + step] = rng.integers(0, 2**32, min(step, blob.size - lo), dtype=np.uint32)
        for a in C2_LAYOUTS[1:]:
            self.src[a].copy_from(self.src["aos-packed"], nthreads)

    def step(self):
        """Seconds of the 25 copyView calls (wall clock of each call, summed)."""
        return sum(self.dst[b].copy_from(self.src[a], self.nthreads)[0] for a in C2_LAYOUTS for b in C2_LAYOUTS)


def check_c2_parity(L, srcs, dsts, n, nthreads, chunk=1 << 20):
    """Bit-exact check of the timed workload (checker leg, after the timed region).  For every
    pair, the GPU copies the full 2^26-record view again; three record ranges [lo, lo+chunk)
    (first, middle, last) of its destination are compared with the reference copyView of a
    chunk view whose blobs are the same ranges of the GPU source (SURVEY 8(d) slice rules)."""
    from oracle import ref
    cext = f"i32:[{chunk}]"
    checked = 0
    los = (0, (n // 2) // chunk * chunk, n - chunk)
    for a in C2_LAYOUTS:
        chunk_src = {}
        for lo in los:
            ca = ref.RefView(R32, cext, a)
            for g, glo, ghi, cbn, clo, chi in _c2_slices(a, n, lo, chunk):
                ca.blobs[cbn][clo:chi] = srcs[a].download_range(g, glo, ghi - glo)
            chunk_src[lo] = ca
        for b in C2_LAYOUTS:
            L.copy_view(srcs[a], dsts[b])
            for lo in los:
                cb = ref.RefView(R32, cext, b)
                cb.copy_from(chunk_src[lo], nthreads)
                for g, glo, ghi, cbn, clo, chi in _c2_slices(b, n, lo, chunk):
                    got = dsts[b].download_range(g, glo, ghi - glo)
                    if not np.array_equal(got, cb.blobs[cbn][clo:chi]):
                        raise AssertionError(f"bench parity: {a} -> {b} records [{lo}, {lo + chunk}) differ")
                    checked += ghi - glo
    return {"pairs": 25, "ranges_per_pair": len(los), "records_per_range": chunk, "bytes_compared": checked,
            "bit_exact": True, "against": "reference copyView (oracle/_ref) of the same source bytes"}


def _c2_slices(layout, n, a, c):
    if layout == "aos-packed" or layout.startswith("aosoa:"):
        return [(0, 28 * a, 28 * (a + c), 0, 0, 28 * c)]
    if layout == "soa-mb":
        return [(f, 4 * a, 4 * (a + c), f, 0, 4 * c) for f in range(7)]
    return [(0, 4 * n * f + 4 * a, 4 * n * f + 4 * (a + c), 0, 4 * c * f, 4 * c * (f + 1)) for f in range(7)]


def run_c4_strong(L, world, rank, local, steps=10, warmup=5, n=128 * 1024, layout="soa-mb"):
    """C4 strong scaling: 128K particles TOTAL split over the ranks (i-range shards), per step
    update + move + the positions-only all-gather (distributed.py; one collective of 12 B per
    particle, Mass once).  Step time = max over ranks of the per-step CUDA-event time."""
    from paper_2302_08251_b200.distributed import nbody_distributed
    out = {"particles_total": n, "layout": layout, "steps": steps,
           "exchange": "one all-gather of packed x,y,z per step (NCCL); Mass gathered once"}
    for mode, name in ((1, "fast"), (0, "exact")):
        nbody_distributed(layout, n, warmup, mode=mode)  # warm-up: allocation, NCCL rings, caches
        barrier(world)
        t = {}
        with ClockSampler(local) as clk:
            nbody_distributed(layout, n, steps, mode=mode, timing=t)
        step = max_over_ranks(t["step_ms"], world)
        exch = max_over_ranks(t["exchange_ms"], world)
        upd = max_over_ranks(t["update_ms"], world)
        out[name] = {"ms_per_step": step, "update_ms": upd, "exchange_ms": exch, "move_ms": t["move_ms"],
                     "interactions_per_s": n * n / (step * 1e-3),
                     "exchange_bytes_per_step": t["exchange_bytes_per_step"], "clocks": clk.summary()}
    return out


def run_c5_sharded(L, world, rank, local, total=1_000_000_000, reps=3):
    """C5: 1e9 R64 records TOTAL, sharded by index over the ranks (no collective on the data
    path): aos-packed f64 -> FieldAccessCount(changetype:f64=f32:bytesplit:soa-mb), source =
    scalarSample(F64, i*7+f) of the GLOBAL index, generated on each device.  GB/s = 84 B x 1e9
    over the max-over-ranks copy time; write counters summed over ranks must be 1e9 per leaf."""
    import torch
    import torch.distributed as dist
    per = total // world
    lo = rank * per
    n = total - lo if rank == world - 1 else per
    ext = f"i32:[{n}]"
    src_t = torch.empty(n * 7, dtype=torch.float64, device="cuda")
    step = 1 << 26
    for a in range(0, n * 7, step):
        b = min(n * 7, a + step)
        s = torch.arange(lo * 7 + a, lo * 7 + b, dtype=torch.int64, device="cuda")
        h = s * (0x9E3779B97F4A7C15 - 2**64) + 0x2545F4914F6CDD1D
        src_t[a:b] = ((h >> 11) & ((1 << 53) - 1)).to(torch.float64) * 2.0 ** -53 * 4.0 - 2.0
    torch.cuda.synchronize()
    src = L.View(L.Layout(R64, ext, "aos-packed"), device=local, blobs=[src_t.data_ptr()], blob_bytes=[n * 56])
    dst = L.View(L.Layout(R64, ext, "changetype:f64=f32:bytesplit:soa-mb", wrap=1), device=local)
    torch.cuda.synchronize()
    L.copy_view(src, dst)
    torch.cuda.synchronize()
    dst.reset_counters()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    e0.record()
    for _ in range(reps):
        L.copy_view(src, dst)
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / reps, world)
    _, w = dst.counters()
    wt = torch.tensor([int(x) for x in w], dtype=torch.int64, device="cuda")
    if world > 1:
        dist.all_reduce(wt)
    writes = [int(x) // reps for x in wt.tolist()]
    del src, dst, src_t
    torch.cuda.synchronize()
    return {"records_total": total, "records_per_gpu": per, "ms": ms, "GB/s": 84 * total / (ms * 1e-3) / 1e9,
            "GB/s_per_gpu": 84 * total / world / (ms * 1e-3) / 1e9, "writes_per_leaf_total": writes,
            "counters_ok": writes == [total] * 7, "layout": "aos-packed(R64) -> FAC(changetype:f64=f32:bytesplit:soa-mb)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--records", type=int, default=1 << 26)
    ap.add_argument("--cpu-records", type=int, default=1 << 24)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--suite", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the C4 strong / C5 sharded keys")
    ap.add_argument("--c4-particles", type=int, default=128 * 1024)
    ap.add_argument("--c5-records", type=int, default=1_000_000_000)
    args = ap.parse_args()
    if args.impl == "reference":
        # the reference arm is CPU-only: no process group, rank 0 alone works and prints
        world, rank, local = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    else:
        world, rank, local = dist_setup()
    n = args.records
    config = {"workload": "C2: copyView over all 25 ordered pairs of {aos-packed, soa-sb, soa-mb, aosoa:8, aosoa:32}",
              "record": "n-body Record{Pos{x,y,z},Vel{x,y,z},Mass} 7 x f32 = 28 B", "records_per_gpu": n,
              "extents": f"i32:[{n}]", "bytes_per_record_pair": 56, "pairs": 25,
              "l2": "no flush needed: every view is 28 B x 2^26 = 1.88 GB >> 126 MB L2",
              "parallelism": f"weak: {world} independent shard(s), no collective"}

    if args.impl == "reference":
        if rank != 0:
            return
        from oracle import ref
        if not ref.available():
            ref.build()
        threads = os.cpu_count() or 1
        t0 = time.perf_counter()
        rc2 = RefC2(n, threads)
        setup_s = time.perf_counter() - t0
        for _ in range(args.warmup):
            rc2.step()
        samples = [rc2.step() for _ in range(args.steps)]
        total = float(sum(samples))
        value = 56 * n * 25 * args.steps / total / 1e9
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (random u32 bit patterns)",
                "impl": "reference", "config": config,
                "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "reference",
                                 "sample": f"the full workload: 25 pairs x {n} records per step, reference copyView "
                                           f"(oracle/_ref) on resident reference views, {threads} threads over "
                                           f"disjoint index ranges; view setup {setup_s:.1f} s untimed"},
                "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    torch.cuda.set_device(local)
    from paper_2302_08251_b200 import lamina as L
    res = run_c2(L, n, args.steps, max(3, args.warmup), world, local)
    peak, peak_kind = peaks()
    line = {"metric": METRIC, "value": res["value"], "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (random u32 bit patterns)",
            "config": config, "gpu_launches": res["launches"], "clocks": res["clocks"]}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "vec_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("bytes_per_launch")
        except Exception:
            traffic = None
    line["roofline"] = {"bound": "hbm", "kernel": "k_vec_transpose<7,4> (the 20 cross-layout pairs)",
                        "achieved": res["achieved_tile"], "peak": peak, "unit": "GB/s",
                        "frac": res["achieved_tile"] / peak, "traffic": traffic,
                        "traffic_source": "committed ncu constant (profiles/vec_traffic.json: dram__bytes_read.sum + "
                                          "dram__bytes_write.sum of one k_vec_transpose<7,4> launch at 2^26 records, "
                                          "ncu --set full; re-captured whenever that kernel changes)",
                        "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                        "spec_peak_GBps": 8000.0, "frac_of_spec": res["achieved_tile"] / 8000.0,
                        "algorithmic_bytes_per_launch": 56 * n}
    line["per_pair_gbs"] = res["per_pair_gbs"]
    srcs, dsts = res.pop("views")
    if rank == 0 and not args.no_cpu:
        from oracle import ref
        if ref.available():
            # checker: the timed workload's bytes against the reference (first / middle / last ranges)
            line["parity"] = check_c2_parity(L, srcs, dsts, n, os.cpu_count() or 1)
            # cpu_baseline: the reference on a bounded sample of the workload, every host thread
            threads = os.cpu_count() or 1
            rc2 = RefC2(args.cpu_records, threads)
            s = rc2.step()
            line["cpu_baseline"] = {"value": 56 * args.cpu_records * 25 / s / 1e9, "unit": "GB/s", "cores": threads,
                                    "kind": "reference",
                                    "sample": f"25 pairs x {args.cpu_records} records (bounded sample of C2), reference "
                                              f"copyView (oracle/_ref), {threads} threads, {s:.1f} s"}
            del rc2
        else:
            line["cpu_baseline"] = {"value": None, "unit": "GB/s", "cores": 1, "kind": "reference",
                                    "sample": "oracle/_ref not built"}
    del srcs, dsts
    torch.cuda.synchronize()
    if not args.no_e2e:
        # N>1: 2^24 records per GPU for the host leg (5 x 470 MB pinned per rank instead of 9.4 GB)
        e2e = run_c2_e2e(L, n if world == 1 else min(n, 1 << 24), args.e2e_steps, local, world)
        if rank == 0:
            line["e2e"] = e2e
    if not args.no_extra:
        # configs that shard / communicate at N GPUs (informative keys beside the C2 headline)
        line["c4_strong"] = run_c4_strong(L, world, rank, local, n=args.c4_particles)
        line["c5_sharded"] = run_c5_sharded(L, world, rank, local, total=args.c5_records)
    if args.suite and rank == 0:
        from bench_suite import run_suite
        line["suite"] = run_suite(L, local)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
