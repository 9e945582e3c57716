"""Staging variants of the generated pair kernels (LAMB_JIT_STAGE = a(uto) / 1 (both) / s / d) at 2^26,
as fractions of HBM peak; the per-span K (16-byte vectors per thread) of each side is in the dump."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import _time, _fill
from paper_2302_08251_b200 import lamina as L
from bench import peaks
from jit_pairs import PAIRS, MIXB
PEAK = peaks()[0]
n = 1 << 26
extra = [(MIXB, "aos-aligned", "soa-mb"), (MIXB, "soa-mb", "aosoa:16"), ("Record{a:f64,b:u16,c:i8,d:f32}", "aosoa:16", "soa-mb"),
         ("Record{a:f64,b:u16,c:i8,d:f32}", "soa-mb", "aos-aligned"), ("Record{a:u8,b:i8,c:u8}", "aos-packed", "soa-mb"),
         ("Record{a:u8,b:i8,c:u8}", "soa-mb", "aos-packed")]
for schema, a, b in [p for p in PAIRS if "Pos" not in p[0]] + extra:
    la, lb = L.Layout(schema, f"i32:[{n}]", a), L.Layout(schema, f"i32:[{n}]", b)
    s, d = L.View(la), L.View(lb)
    _fill(L, s, 1)
    byt = sum(la.blob_sizes) + sum(lb.blob_sizes)
    row = []
    for st in ["a", "1", "s", "d"]:
        os.environ["LAMB_JIT_STAGE"] = st
        ms = _time(lambda: L.copy_view(s, d), reps=3, warm=1)
        row.append(f"{st}:{byt / ms / 1e6 / PEAK:.2f}")
    print(f"{schema[:16]:16} {a:>12} -> {b:<12}", " ".join(row), flush=True)
    del s, d
