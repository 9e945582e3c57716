"""One copy of a given pair (for ncu launch lists): python tools/one_pair.py SCHEMA SRC DST [N]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import _fill
from paper_2302_08251_b200 import lamina as L
schema, a, b = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 22
s, d = L.View(L.Layout(schema, f"i32:[{n}]", a)), L.View(L.Layout(schema, f"i32:[{n}]", b))
_fill(L, s, 1)
L.copy_view(s, d)
import torch; torch.cuda.synchronize()
