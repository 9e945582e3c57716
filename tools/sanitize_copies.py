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
    # round 2 kernels: packv (1/2/8-byte leaves, > 32-bit fields), compile-time float widths
    copy("Record{v:u16,w:u16}", n, "soa-mb", "bitpack-int:5")
    copy("Record{v:u16,w:u16}", n, "bitpack-int:5", "soa-mb")
    copy("Record{a:i8,b:u8}", n, "soa-mb", "bitpack-int:3")
    copy("Record{v:u64,w:i64}", n, "soa-mb", "bitpack-int:47")
    copy("Record{v:u64,w:i64}", n, "bitpack-int:47", "soa-mb")
    copy(R64, n, "soa-mb", "bitpack-float:11,52")
    copy(R64, n, "bitpack-float:11,52", "soa-mb")
    copy(R32, n, "soa-mb", "bitpack-float:4,3")
    copy(R32, n, "bitpack-float:4,3", "soa-mb")
    copy(R32, n, "soa-mb", "bitpack-float:11,30")
    copy(R32, n, "bitpack-float:11,30", "soa-mb")
v = L.View(L.Layout(R32, "i64:[700]", "aosoa:8", wrap=3, granularity=16)); v.nbody_init(1); v.nbody_update(0); v.nbody_update(1); v.nbody_move()
# exact split kernel (small shards), fast kernel, multi-source update, position packing, manual baselines
w = L.View(L.Layout(R32, "i64:[3000]", "soa-mb")); w.nbody_init(2)
w.nbody_update(0, 0, 1000); w.nbody_update(0); w.nbody_update(1); w.nbody_move()
w.nbody_update_from([(w, 0, 1500), (w, 1500, 3000)], 0, 0, 3000)
import torch
buf = torch.empty(4 * 3000, dtype=torch.float32, device="cuda")
w.nbody_pack_positions(0, 3000, buf.data_ptr(), with_mass=True); torch.cuda.synchronize()
for kind in ("manual-aos", "manual-soa"):
    m = L.ManualNbody(kind, 3000); m.update(0); m.update(1); m.move(); m.checksum()
print("ok")
