"""One record-side pack and unpack at 2^26 n-body records (ncu target for k_rec_pack / k_rec_unpack)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import _fill, R32
from paper_2302_08251_b200 import lamina as L
import torch
n = 1 << 26
la, lb = L.Layout(R32, f"i32:[{n}]", "aos-packed"), L.Layout(R32, f"i32:[{n}]", "bitpack-float:5,10")
s, d = L.View(la), L.View(lb)
_fill(L, s, 1)
L.copy_view(s, d)
L.copy_view(d, s)
torch.cuda.synchronize()
print("ok")
