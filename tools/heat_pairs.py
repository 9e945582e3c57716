"""Heatmap-instrumented copies at 2^26 records (GB/s of source + destination blob bytes; counters
not counted): the copy kernel plus the closed-form accounting pass k_heat_closed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import _time, _fill, R32
from paper_2302_08251_b200 import lamina as L
from bench import peaks
PEAK = peaks()[0]  # MEASURED_PEAKS.json hbm_gbs
n = 1 << 26
for a, b, sw, dw, g in [("aos-packed", "soa-mb", 0, 2, 64), ("soa-mb", "aos-packed", 2, 0, 64),
                        ("aos-packed", "soa-mb", 0, 2, 4096), ("aos-packed", "soa-mb", 0, 2, 5),
                        ("soa-mb", "aos-packed", 0, 2, 5), ("soa-mb", "aos-packed", 0, 2, 64),
                        ("aos-packed", "bytesplit:soa-mb", 0, 2, 64)]:
    la = L.Layout(R32, f"i32:[{n}]", a, wrap=sw, granularity=g)
    lb = L.Layout(R32, f"i32:[{n}]", b, wrap=dw, granularity=g)
    s, d = L.View(la), L.View(lb)
    _fill(L, s, 1)
    ms = _time(lambda: L.copy_view(s, d), reps=5, warm=2)
    byt = sum(la.blob_sizes) + sum(lb.blob_sizes)
    print(f"heat g={g:<5} {'H(' + a + ')' if sw else a:>16} -> {'H(' + b + ')' if dw else b:<16} {byt / ms / 1e6:7.0f} GB/s  {byt / ms / 1e6 / PEAK:.2f}", flush=True)
    del s, d
