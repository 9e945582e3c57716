"""First-use cost of the generated kernels: first copy (generate + NVRTC compile; at >= 2^22 elements
also the 8-variant autotune) vs the steady-state copy, for a few pairs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench_suite import _fill
from paper_2302_08251_b200 import lamina as L
MIXED = "Record{a:i8,b:u16,c:i32,d:u64,e:f32,f:f64,g:bool,h:Record{x:i16,y:f32[3]}}"
for n in (1 << 16, 1 << 22):
    for a, b in [("aos-packed", "soa-mb"), ("soa-mb", "aosoa:16"), ("aosoa:8", "bytesplit:soa-mb")]:
        la, lb = L.Layout(MIXED, f"i32:[{n}]", a), L.Layout(MIXED, f"i32:[{n}]", b)
        s, d = L.View(la), L.View(lb)
        _fill(L, s, 1)
        torch.cuda.synchronize()
        t0 = time.perf_counter(); L.copy_view(s, d); torch.cuda.synchronize(); first = time.perf_counter() - t0
        t0 = time.perf_counter(); L.copy_view(s, d); torch.cuda.synchronize(); second = time.perf_counter() - t0
        print(f"n=2^{n.bit_length() - 1} {a:>10} -> {b:<18} first {first * 1e3:8.1f} ms   next {second * 1e3:6.2f} ms", flush=True)
        del s, d
