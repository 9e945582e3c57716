"""k_repack32 vs staging through the SoA scratch (LAMB_REPACK=0) for bit stream -> bit stream pairs, 2^26."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import _time, _fill, R32
from paper_2302_08251_b200 import lamina as L
from bench import peaks
PEAK = peaks()[0]
n = 1 << 26
for schema, a, b in [("Record{v:u32,w:i32}", "bitpack-int:11", "bitpack-int:7"), ("Record{v:u32,w:i32}", "bitpack-int:13", "bitpack-int:13"),
                     ("Record{v:u32,w:i32}", "bitpack-int:3", "bitpack-int:31"), (R32, "bitpack-float:5,10", "bitpack-float:5,10"),
                     (R32, "bitpack-float:4,3", "bitpack-float:5,10"), (R32, "bitpack-float:8,10", "bitpack-float:4,3"), (R32, "bitpack-float:4,3", "bitpack-float:4,3")]:
    la, lb = L.Layout(schema, f"i32:[{n}]", a), L.Layout(schema, f"i32:[{n}]", b)
    s, d = L.View(la), L.View(lb)
    _fill(L, s, 1)
    byt = sum(la.blob_sizes) + sum(lb.blob_sizes)
    row = []
    for rp in ("1", "0"):
        os.environ["LAMB_REPACK"] = rp
        ms = _time(lambda: L.copy_view(s, d), reps=3, warm=1)
        row.append(f"repack={rp}:{byt / ms / 1e6 / PEAK:.2f}")
    print(f"{schema[:20]:20} {a:>20} -> {b:<20}", " ".join(row), flush=True)
    del s, d
