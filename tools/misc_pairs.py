"""Throughput of compositions outside C2/C3/C5 (which kernel path each takes), 2^26 R32 records."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import _time, _fill, R32, R64
from paper_2302_08251_b200 import lamina as L
n = 1 << 26
PAIRS = [
    (R32, "aos-packed", "bytesplit:soa-mb", 0), (R32, "bytesplit:soa-mb", "aos-packed", 0),
    (R32, "aos-packed", "changetype:f32=f64:soa-mb", 0), (R32, "changetype:f32=f64:soa-mb", "aos-packed", 0),
    (R32, "aos-packed", "split:Pos:soa-mb:aos-packed", 0), (R32, "aos-packed", "aosoa:3", 0),
    (R32, "aos-packed", "aos-aligned", 0), (R32, "soa-mb", "aos-packed", 1), (R32, "aos-packed", "soa-mb", 2),
    (R32, "aos-packed", "bitpack-float:5,10", 0), (R32, "aos-packed", "null", 0),
    ("Record{a:f64,b:u16,c:i8,d:f32}", "aos-packed", "soa-mb", 0),
    # Split compositions (k_vec_multi)
    (R32, "split:Pos:soa-mb:aos-packed", "aos-packed", 0), (R32, "soa-mb", "split:Pos:soa-mb:aos-packed", 0),
    (R32, "aosoa:8", "split:Vel:aosoa:8:soa-mb", 0), (R32, "split:Pos,Mass:aosoa:4:soa-sb", "aos-packed", 0),
    (R32, "aos-packed", "split:Vel:aos-packed:aos-packed", 0), (R64, "aos-packed", "split:Pos:soa-mb:aos-packed", 0),
    # AoSoA with lane counts no vector group fits (k_vec_rows)
    (R32, "aosoa:3", "aos-packed", 0), (R32, "soa-mb", "aosoa:3", 0), (R32, "aosoa:6", "soa-sb", 0),
    (R32, "aosoa:32", "aosoa:3", 0), (R64, "aos-packed", "aosoa:3", 0),
]
for schema, a, b, wrap in PAIRS:
    la, lb = L.Layout(schema, f"i32:[{n}]", a), L.Layout(schema, f"i32:[{n}]", b, wrap=wrap, granularity=64)
    s, d = L.View(la), L.View(lb)
    _fill(L, s, 1)
    c0 = L.launch_count()
    ms = _time(lambda: L.copy_view(s, d), reps=3, warm=1)
    rec = sum(la.leaf(f)[1] for f in range(la.leaf_count))
    print(f"{a:>28} -> {b:<34} wrap={wrap} {2 * rec * n / ms / 1e6:8.0f} GB/s (leaf bytes r+w)", flush=True)
    del s, d
