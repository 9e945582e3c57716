"""Host-side cost of one copyView dispatch (small views: the launch path dominates)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2302_08251_b200 import lamina as L
R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"
for n in (1024, 1 << 20):
    for a, b in [("aos-packed", "soa-mb"), ("aos-packed", "bytesplit:soa-mb"), ("soa-mb", "bitpack-float:8,10")]:
        s, d = L.View(L.Layout(R32, f"i32:[{n}]", a)), L.View(L.Layout(R32, f"i32:[{n}]", b))
        for _ in range(20):
            L.copy_view(s, d)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(500):
            L.copy_view(s, d)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(n, a, b, f"host {1e6 * (t1 - t0) / 500:.1f} us/call, total {1e6 * (t2 - t0) / 500:.1f} us/call", flush=True)
