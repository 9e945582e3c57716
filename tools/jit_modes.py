"""Staging modes of the generated kernel on selected pairs at 2^24 (fractions of HBM peak)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench_suite import _fill, R32, R64
from paper_2302_08251_b200 import lamina as L
from bench import peaks
PEAK = peaks()[0]
MIXED = "Record{a:i8,b:u16,c:i32,d:u64,e:f32,f:f64,g:bool,h:Record{x:i16,y:f32[3]}}"
n = 1 << 24
PAIRS = [(R32, "aosoa:8", "aosoa:3"), (R32, "aosoa:3", "aosoa:8"), (R32, "soa-mb", "bytesplit:soa-mb"),
         (R32, "bytesplit:soa-mb", "soa-mb"), (MIXED, "aos-packed", "aosoa:3"), (MIXED, "aos-packed", "soa-mb"),
         (MIXED, "soa-mb", "aos-aligned"), (MIXED, "aosoa:32", "aos-aligned"), (MIXED, "aosoa:8", "aosoa:32"),
         (MIXED, "bytesplit:soa-mb", "aosoa:32"), (R64, "aos-packed", "aosoa:3"),
         (MIXED, "aos-packed", "changetype:f64=f32,i8=i64,u16=u8:aosoa:2"), (R32, "changetype:f32=f64:soa-mb", "aosoa:3"),
         (R32, "changetype:f32=f64:soa-mb", "bytesplit:soa-mb"), (R32, "aosoa:3", "changetype:f32=f64:soa-mb"),
         ("Record{a:f64,b:u16,c:i8,d:f32}", "aos-packed", "changetype:f64=f32:soa-mb")]
def t(s, d):
    L.copy_view(s, d)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        L.copy_view(s, d)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 3
for schema, a, b in PAIRS:
    la, lb = L.Layout(schema, f"i32:[{n}]", a), L.Layout(schema, f"i32:[{n}]", b)
    s, d = L.View(la), L.View(lb)
    _fill(L, s, 1)
    byt = sum(la.blob_sizes) + sum(lb.blob_sizes)
    row = []
    for mode in ["a", "1", "s", "d", "0"]:
        os.environ["LAMB_JIT_STAGE"] = mode
        row.append(f"{mode}:{byt / t(s, d) / 1e6 / PEAK:.2f}")
    os.environ["LAMB_JIT"] = "0"
    row.append(f"nojit:{byt / t(s, d) / 1e6 / PEAK:.2f}")
    os.environ["LAMB_JIT"] = "1"
    print(f"{schema[:12]} {a:>18} -> {b:<18}", " ".join(row), flush=True)
    del s, d
