"""Record-side bit-packing (pack.cu k_rec_pack / k_rec_unpack) at 2^26 records, GB/s of source +
destination blob bytes, against the staged route (LAMB_RECPACK=0 in a second process)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import _time, _fill, R32
from paper_2302_08251_b200 import lamina as L
from bench import peaks
PEAK = peaks()[0]  # MEASURED_PEAKS.json hbm_gbs
I3 = "Record{v:u32,w:i32,x:i32,y:u32,z:i32,p:u32,q:i32}"
n = 1 << 26
tag = "staged" if os.environ.get("LAMB_RECPACK") == "0" else "one-pass"
for schema, a, b in [(R32, "aos-packed", "bitpack-float:5,10"), (R32, "bitpack-float:5,10", "aos-packed"),
                     (R32, "aos-packed", "bitpack-float:8,10"), (R32, "bitpack-float:8,10", "aos-packed"),
                     (R32, "aosoa:8", "bitpack-float:5,10"), (R32, "bitpack-float:5,10", "aosoa:8"),
                     (I3, "aos-packed", "bitpack-int:3"), (I3, "bitpack-int:3", "aos-packed"),
                     (I3, "aos-packed", "bitpack-int:12"), (I3, "bitpack-int:12", "aos-packed"),
                     (I3, "aosoa:16", "bitpack-int:24"), (I3, "bitpack-int:24", "aosoa:16")]:
    la, lb = L.Layout(schema, f"i32:[{n}]", a), L.Layout(schema, f"i32:[{n}]", b)
    s, d = L.View(la), L.View(lb)
    _fill(L, s, 1)
    ms = _time(lambda: L.copy_view(s, d), reps=5, warm=2)
    byt = sum(la.blob_sizes) + sum(lb.blob_sizes)
    print(f"{tag:8} {schema[:14]:14} {a:>20} -> {b:<20} {byt / ms / 1e6:7.0f} GB/s  {byt / ms / 1e6 / PEAK:.2f}", flush=True)
    del s, d
