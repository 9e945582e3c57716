"""One generated-kernel copy (for ncu): python tools/jit_one.py SCHEMA SRC DST [n]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import _fill
from paper_2302_08251_b200 import lamina as L
schema, a, b = sys.argv[1:4]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 26
la, lb = L.Layout(schema, f"i32:[{n}]", a), L.Layout(schema, f"i32:[{n}]", b)
s, d = L.View(la), L.View(lb)
_fill(L, s, 1)
for _ in range(3):
    L.copy_view(s, d)
d.sync()
print("bytes", sum(la.blob_sizes) + sum(lb.blob_sizes))
