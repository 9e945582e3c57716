"""Which path each weak composition takes (LAMB_TRACE=1) and its fraction of HBM at 2^24."""
import os, sys
os.environ["LAMB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench_suite import _fill, R32
from paper_2302_08251_b200 import lamina as L
from bench import peaks
PEAK = peaks()[0]
MIXED = "Record{a:i8,b:u16,c:i32,d:u64,e:f32,f:f64,g:bool,h:Record{x:i16,y:f32[3]}}"
n = 1 << 24
PAIRS = [(R32, "soa-mb", "aosoa:4"), (R32, "aos-packed", "aosoa:4"), (R32, "aosoa:8", "aosoa:3"), (R32, "aosoa:3", "aosoa:8"),
         (R32, "bytesplit:soa-mb", "aosoa:32"), (R32, "bytesplit:soa-mb", "bytesplit:soa-mb"), (R32, "bytesplit:soa-mb", "soa-mb"),
         (R32, "soa-mb", "bytesplit:soa-mb"), (R32, "changetype:f32=f64:soa-mb", "aosoa:3"),
         (R32, "changetype:f32=f64:soa-mb", "bytesplit:soa-mb"), (R32, "bitpack-float:5,10", "bytesplit:soa-mb"),
         (R32, "aos-packed", "bitpack-float:4,3"), (R32, "soa-mb", "soa-mb"),
         (MIXED, "soa-sb", "soa-mb"), (MIXED, "soa-mb", "aos-aligned"), (MIXED, "aosoa:32", "aos-aligned"),
         (MIXED, "aos-packed", "aosoa:3"), (MIXED, "aosoa:32", "soa-mb"), (MIXED, "aos-packed", "soa-mb"),
         (MIXED, "bytesplit:soa-mb", "aosoa:32"), (MIXED, "aos-packed", "changetype:f64=f32,i8=i64,u16=u8:aosoa:2")]
for schema, a, b in PAIRS:
    la, lb = L.Layout(schema, f"i32:[{n}]", a), L.Layout(schema, f"i32:[{n}]", b)
    s, d = L.View(la), L.View(lb)
    _fill(L, s, 1)
    print(f"=== {schema[:12]} {a} -> {b}", file=sys.stderr, flush=True)
    L.copy_view(s, d)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    os.environ["LAMB_TRACE"] = "0"
    e0.record()
    for _ in range(3):
        L.copy_view(s, d)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"    {(sum(la.blob_sizes) + sum(lb.blob_sizes)) / ms / 1e6 / PEAK:.2f}", file=sys.stderr, flush=True)
    del s, d
