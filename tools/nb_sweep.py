"""Sweep the fast n-body j-segment count (LAMB_NB_SEGMENTS) at the C4 shape."""
import os, subprocess, sys
code = r'''
import sys; sys.path.insert(0, ".")
from paper_2302_08251_b200 import lamina as L
from bench_suite import _time
R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"
n = int(sys.argv[1])
for lay in ["aos-packed", "soa-mb"]:
    v = L.View(L.Layout(R32, f"i64:[{n}]", lay)); v.nbody_init(42)
    ms = _time(lambda: v.nbody_update(1), reps=5, warm=2)
    print(lay, round(ms, 3), "ms", round(n * n / ms / 1e9, 3), "e12 int/s", flush=True)
'''
for seg in sys.argv[2:]:
    env = dict(os.environ)
    if seg != "auto":
        env["LAMB_NB_SEGMENTS"] = seg
    print("segments", seg, flush=True)
    subprocess.run([sys.executable, "-c", code, sys.argv[1]], env=env, check=True)
