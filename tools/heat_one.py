import os, sys
sys.path.insert(0, os.getcwd())
from bench_suite import _fill, R32
from paper_2302_08251_b200 import lamina as L
import torch
n = 1 << 26
for g in (64, 5):
    la = L.Layout(R32, f"i32:[{n}]", "aos-packed")
    lb = L.Layout(R32, f"i32:[{n}]", "soa-mb", wrap=2, granularity=g)
    s, d = L.View(la), L.View(lb)
    _fill(L, s, 1)
    L.copy_view(s, d)
    torch.cuda.synchronize()
    del s, d
