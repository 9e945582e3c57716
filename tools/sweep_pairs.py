"""Every (src, dst) layout pair of two schemas at 2^24 elements: fraction of HBM peak (source +
destination blob bytes), to find the compositions still below 80%.  Three back-to-back copies timed after a warm one (host work per call included)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench_suite import _fill, R32
from paper_2302_08251_b200 import lamina as L
from bench import peaks
PEAK = peaks()[0]
MIXED = "Record{a:i8,b:u16,c:i32,d:u64,e:f32,f:f64,g:bool,h:Record{x:i16,y:f32[3]}}"
LAY = ["aos-packed", "aos-aligned", "soa-sb", "soa-mb", "aosoa:4", "aosoa:8", "aosoa:32", "aosoa:3",
       "bytesplit:soa-mb", "bytesplit:aos-packed", "split:Vel:soa-mb:aos-packed"]
n = int(os.environ.get("SWEEP_N", 1 << 24))
for schema, extra in [(R32, ["changetype:f32=f64:soa-mb", "bitpack-float:5,10", "bitpack-float:4,3"]),
                      (MIXED, ["changetype:f64=f32,i8=i64,u16=u8:aosoa:2", "split:h:bytesplit:soa-mb:aos-aligned"])]:
    lays = LAY + extra
    if schema == MIXED:
        lays = [l.replace("split:Vel:", "split:h:") for l in lays]
    views = {}
    for l in lays:
        lay = L.Layout(schema, f"i32:[{n}]", l)
        v = L.View(lay)
        _fill(L, v, 1)
        views[l] = (lay, v)
    for a in lays:
        row = []
        for b in lays:
            (la, s), (lb, d) = views[a], views[b]
            L.copy_view(s, d)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(3):
                L.copy_view(s, d)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
            row.append((sum(la.blob_sizes) + sum(lb.blob_sizes)) / ms / 1e6 / PEAK)
        print(f"{schema[:12]} {a:>40}: " + " ".join(f"{x:4.2f}" for x in row), flush=True)
    print("columns:", " | ".join(lays), flush=True)
    del views
