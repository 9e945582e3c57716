"""Spot check of less common compositions at 2^26 records (GB/s of source + destination blob bytes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import _time, _fill, R32, R64
from paper_2302_08251_b200 import lamina as L
from bench import peaks
PEAK = peaks()[0]  # MEASURED_PEAKS.json hbm_gbs
MIXED = "Record{a:f64,b:u16,c:i8,d:f32}"
n = 1 << 26
for schema, a, b in [("Record{v:u16,w:u16}", "soa-mb", "bitpack-int:5"), ("Record{v:u16,w:u16}", "bitpack-int:5", "soa-mb"),
                     (R32, "soa-mb", "bitpack-float:4,3"), (R32, "bitpack-float:4,3", "soa-mb"),
                     (R64, "aos-packed", "changetype:f64=f32:aos-packed"), (R64, "changetype:f64=f32:aos-packed", "soa-mb"),
                     (MIXED, "aos-packed", "bytesplit:soa-sb"), (MIXED, "aosoa:8", "aos-aligned"),
                     (R32, "aosoa:8", "changetype:f32=f64:aosoa:4"), (R32, "soa-sb", "split:Vel:aosoa:8:soa-mb")]:
    la, lb = L.Layout(schema, f"i32:[{n}]", a), L.Layout(schema, f"i32:[{n}]", b)
    s, d = L.View(la), L.View(lb)
    _fill(L, s, 1)
    ms = _time(lambda: L.copy_view(s, d), reps=3, warm=1)
    byt = sum(la.blob_sizes) + sum(lb.blob_sizes)
    print(f"{schema[:22]:22} {a:>32} -> {b:<32} {byt / ms / 1e6:7.0f} GB/s  {byt / ms / 1e6 / PEAK:.2f}", flush=True)
    del s, d
