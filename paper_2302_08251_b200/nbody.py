"""The n-body benchmark runner on the device (proj/tools/nbody/runner.hpp, runner.cpp).

Mirrors the reference's `nbody::BenchConfig` / `nbody::runBenchmark`: same options, same
validation messages (runner.cpp:441-466), same CSV rows on stdout
(`layout,phase,simd_width,seconds_per_step,checksum`, runner.cpp:88-103), and with
`trace_fields` / `heatmap_granularity` the same report files (`fields_update.csv`,
`fields_move.csv`, `heatmap_update.csv`, `heatmap_move.csv`, runner.cpp:344-436), counters
accumulated per phase over the steps.  The arithmetic runs in the sm_100a n-body kernels
(exact mode by default: bit-identical to the reference, so the checksum text matches).

`manual-aos` / `manual-soa` (the reference's hand-written baselines, steps.hpp:124-230,
runner.cpp:239-323) run separate hand-written device kernels over a plain struct array /
seven plain arrays (csrc/nbody_manual.cu, no mapping, no accessor), so the
library-vs-hand-written ratio of paper Fig. 3 is measured; in exact mode their checksum text
equals the library layouts' (acceptance.cpp:744-766).
"""
from __future__ import annotations

import os
import sys
from dataclasses import dataclass

import numpy as np

from .lamina import (NBODY_EXACT, WRAP_FIELD_ACCESS_COUNT, WRAP_HEATMAP, Layout, ManualNbody, View,
                     field_access_csv, heatmap_csv)

SCHEMA = {
    "f32": "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}",
    "f64": "Record{Pos:Record{x:f64,y:f64,z:f64},Vel:Record{x:f64,y:f64,z:f64},Mass:f64}",
}
MANUAL = ("manual-aos", "manual-soa")


@dataclass
class BenchConfig:
    """runner.hpp:9-22 (plus `mode`: the device arithmetic mode, exact by default)."""
    layout: str = "aos-packed"
    n: int = 16384
    steps: int = 5
    simd_width: int = 1
    precision: str = "f64"
    seed: int = 42
    trace_fields: bool = False
    heatmap_granularity: int = 0
    aosoa_nested: bool = False
    csv_path: str = ""
    report_dir: str = "."
    mode: int = NBODY_EXACT
    device: int = 0


def _usage(msg: str) -> int:
    print(f"error: {msg}", file=sys.stderr)
    return 2


def _time_ms(fn) -> float:
    import torch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b)


def _write_csv(cfg: BenchConfig, update_s: float, move_s: float, checksum: float) -> None:
    rows = ("layout,phase,simd_width,seconds_per_step,checksum\n"
            f"{cfg.layout},update,{cfg.simd_width},{update_s!r},{_g17(checksum)}\n"
            f"{cfg.layout},move,{cfg.simd_width},{move_s!r},{_g17(checksum)}\n")
    sys.stdout.write(rows)
    if cfg.csv_path:
        with open(cfg.csv_path, "w") as f:
            f.write(rows)


def _g17(x: float) -> str:
    """std::ostream << double at precision 17 (runner.cpp:91): %.17g."""
    return f"{x:.17g}"


def _run_manual(cfg: BenchConfig) -> int:
    """runManual (runner.cpp:239-323): warm-up on a copy, then the measured steps, checksum."""
    try:
        f64 = cfg.precision == "f64"
        warm = ManualNbody(cfg.layout, cfg.n, f64, cfg.seed, cfg.device)
        warm.update(cfg.mode)
        warm.move()
        del warm
        m = ManualNbody(cfg.layout, cfg.n, f64, cfg.seed, cfg.device)
        upd_t, mov_t = [], []
        for _ in range(cfg.steps):
            upd_t.append(_time_ms(lambda: m.update(cfg.mode)) * 1e-3)
            mov_t.append(_time_ms(lambda: m.move()) * 1e-3)
        _write_csv(cfg, float(np.median(upd_t)), float(np.median(mov_t)), m.checksum())
        return 0
    except Exception as e:  # noqa: BLE001 - runner.cpp:458-462
        print(f"error: {e}", file=sys.stderr)
        return 1


def run_benchmark(cfg: BenchConfig) -> int:
    """runner.cpp:440-466 + runView/runManual on the device; returns the process exit code."""
    if cfg.n < 1:
        return _usage("--n must be >= 1")
    if cfg.steps < 1:
        return _usage("--steps must be >= 1")
    if cfg.simd_width not in (1, 2, 4, 8, 16):
        return _usage("--simd-width must be one of 1, 2, 4, 8, 16")
    if cfg.n % cfg.simd_width != 0:
        return _usage("--n must be a multiple of --simd-width")
    if cfg.precision not in ("f32", "f64"):
        return _usage("--precision must be f32 or f64")
    layout = cfg.layout
    if layout in MANUAL:
        if cfg.simd_width != 1:
            return _usage("manual baselines support --simd-width 1 only")
        if cfg.trace_fields or cfg.heatmap_granularity != 0:
            return _usage("manual baselines have no mapping to instrument")
        return _run_manual(cfg)
    wrap = (WRAP_FIELD_ACCESS_COUNT if cfg.trace_fields else 0) | (WRAP_HEATMAP if cfg.heatmap_granularity else 0)
    if cfg.aosoa_nested and (wrap or not layout.startswith("aosoa:")):
        return _usage("--aosoa-nested requires an uninstrumented aosoa:<L> layout")
    schema, ext = SCHEMA[cfg.precision], f"i64:[{cfg.n}]"
    try:
        lay = Layout(schema, ext, layout, wrap=wrap, granularity=max(1, cfg.heatmap_granularity))
    except Exception as e:  # noqa: BLE001 - mirrors the runner's usage error path
        return _usage(f"invalid layout '{cfg.layout}': {e}")
    try:
        view = View(lay, device=cfg.device)
        view.nbody_init(cfg.seed)
        # warm-up on a separate uninstrumented view of the same layout (runner.cpp:368-375)
        warm = View(Layout(schema, ext, layout), device=cfg.device)
        warm.nbody_init(cfg.seed)
        warm.nbody_update(cfg.mode)
        warm.nbody_move()
        del warm
        if wrap:
            view.reset_counters()
        nleaves = lay.leaf_count
        upd_c = [np.zeros(nleaves, np.uint64), np.zeros(nleaves, np.uint64)]
        mov_c = [np.zeros(nleaves, np.uint64), np.zeros(nleaves, np.uint64)]
        upd_h = [np.zeros(lay.heatmap_blocks(k), np.uint64) for k in range(lay.blob_count)] if cfg.heatmap_granularity else []
        mov_h = [np.zeros(lay.heatmap_blocks(k), np.uint64) for k in range(lay.blob_count)] if cfg.heatmap_granularity else []

        def harvest(counters, blocks):
            if cfg.trace_fields:
                r, w = view.counters()
                counters[0] += r
                counters[1] += w
            if cfg.heatmap_granularity:
                for k in range(lay.blob_count):
                    blocks[k] += view.heatmap(k)
            if wrap:
                view.reset_counters()

        upd_t, mov_t = [], []
        for _ in range(cfg.steps):
            upd_t.append(_time_ms(lambda: view.nbody_update(cfg.mode)) * 1e-3)
            harvest(upd_c, upd_h)
            mov_t.append(_time_ms(lambda: view.nbody_move()) * 1e-3)
            harvest(mov_c, mov_h)
        checksum = view.nbody_checksum()
        _write_csv(cfg, float(np.median(upd_t)), float(np.median(mov_t)), checksum)
        if cfg.trace_fields:
            os.makedirs(cfg.report_dir, exist_ok=True)
            for name, (r, w) in (("fields_update.csv", upd_c), ("fields_move.csv", mov_c)):
                with open(os.path.join(cfg.report_dir, name), "w") as f:
                    f.write(field_access_csv(lay, r, w))
        if cfg.heatmap_granularity:
            os.makedirs(cfg.report_dir, exist_ok=True)
            for name, blocks in (("heatmap_update.csv", upd_h), ("heatmap_move.csv", mov_h)):
                with open(os.path.join(cfg.report_dir, name), "w") as f:
                    f.write(heatmap_csv(cfg.heatmap_granularity, blocks))
        return 0
    except Exception as e:  # noqa: BLE001 - runner.cpp:458-462
        print(f"error: {e}", file=sys.stderr)
        return 1
