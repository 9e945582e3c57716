"""Profiling driver: a few fast-mode n-body updates at N=128K (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_08251_b200 import lamina as L  # noqa: E402

R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"
mode = int(os.environ.get("NBODY_MODE", "1"))
v = L.View(L.Layout(R32, "i64:[131072]", os.environ.get("NBODY_LAYOUT", "soa-mb")))
v.nbody_init(42)
for _ in range(3):
    v.nbody_update(mode)
v.sync()
