"""Uniform pairs the vector transpose cannot take (non-power-of-two AoSoA lanes): k_uniform_direct vs the
generated kernel (LAMB_JIT_UNI=1) under each staging mode, fractions of HBM peak at 2^26."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import _time, _fill, R32, R64
from paper_2302_08251_b200 import lamina as L
from bench import peaks
PEAK = peaks()[0]
n = 1 << 26
for schema, a, b in [(R32, "aos-packed", "aosoa:3"), (R32, "aosoa:3", "aos-packed"), (R32, "soa-mb", "aosoa:3"),
                     (R32, "aosoa:3", "soa-mb"), (R32, "aosoa:6", "soa-sb"), (R32, "aosoa:32", "aosoa:3"),
                     (R64, "aos-packed", "aosoa:3"), (R64, "aosoa:3", "soa-mb"), (R32, "aos-packed", "aosoa:2"),
                     (R32, "aosoa:2", "soa-mb")]:
    la, lb = L.Layout(schema, f"i32:[{n}]", a), L.Layout(schema, f"i32:[{n}]", b)
    s, d = L.View(la), L.View(lb)
    _fill(L, s, 1)
    byt = sum(la.blob_sizes) + sum(lb.blob_sizes)
    row = []
    for uni, st in [("0", "a"), ("1", "a"), ("1", "1"), ("1", "s"), ("1", "d")]:
        os.environ["LAMB_JIT_UNI"], os.environ["LAMB_JIT_STAGE"] = uni, st
        ms = _time(lambda: L.copy_view(s, d), reps=3, warm=1)
        row.append(f"{'jit' if uni == '1' else 'fixed'}/{st}:{byt / ms / 1e6 / PEAK:.2f}")
    print(f"{schema[:16]:16} {a:>12} -> {b:<12}", " ".join(row), flush=True)
    del s, d
