"""Small copies through every kernel family, for compute-sanitizer memcheck."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import R32, R64, MIXED, random_values
from paper_2302_08251_b200 import lamina as L

def copy(schema, n, a, b, wa=0, wb=0, g=8):
    la, lb = L.Layout(schema, f"i32:[{n}]", a, wrap=wa, granularity=g), L.Layout(schema, f"i32:[{n}]", b, wrap=wb, granularity=g)
    s, d = L.View(la), L.View(lb)
    L.copy_view(s, d)
    d.download_all()

for n in (1, 37, 4099, 70001):
    for a, b in [("aos-packed", "soa-mb"), ("soa-mb", "aosoa:8"), ("aos-packed", "bytesplit:soa-mb"),
                 ("bytesplit:soa-mb", "aos-packed"), ("aos-packed", "changetype:f32=f64:soa-mb"),
                 ("changetype:f32=f64:soa-mb", "aosoa:32"), ("aos-packed", "split:Pos:soa-mb:aos-packed"),
                 ("aos-packed", "aosoa:3"), ("soa-mb", "bitpack-float:8,10"), ("bitpack-float:5,10", "soa-mb"),
                 ("aos-packed", "null"), ("aos-packed", "aos-packed")]:
        copy(R32, n, a, b)
    copy(R32, n, "aos-packed", "soa-mb", wb=3)
    copy(R32, n, "aos-packed", "bytesplit:aos-packed", wa=2, wb=2)
    copy(R64, n, "aos-packed", "changetype:f64=f32:bytesplit:soa-mb", wb=1)
    copy(R64, n, "changetype:f64=f32:bytesplit:soa-mb", "aos-packed")
    copy(MIXED, n, "aos-packed", "soa-mb")
    copy("Record{v:u32}", n, "soa-mb", "bitpack-int:7")
    copy("Record{v:u32}", n, "bitpack-int:7", "soa-mb", wb=2)
v = L.View(L.Layout(R32, "i64:[700]", "aosoa:8", wrap=3, granularity=16)); v.nbody_init(1); v.nbody_update(0); v.nbody_update(1); v.nbody_move()
print("ok")
