"""Same-layout copyView (blob copy) rates at the C2 size, for LAMB_BLOB_* experiments."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import _time, R32
from paper_2302_08251_b200 import lamina as L
n = 1 << 26
for lay in ["aos-packed", "soa-mb"]:
    a, b = L.View(L.Layout(R32, f"i32:[{n}]", lay)), L.View(L.Layout(R32, f"i32:[{n}]", lay))
    ms = _time(lambda: L.copy_view(a, b), reps=10, warm=3)
    print(os.environ.get("LAMB_BLOB_U", "4"), os.environ.get("LAMB_BLOB_CTAS", "8"), lay, round(56 * n / ms / 1e6), "GB/s", flush=True)
