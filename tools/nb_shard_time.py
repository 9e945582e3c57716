"""Strong-scaling prediction on one GPU: n-body update of an i-shard [0, N/k) against all
N = 128K j-particles (what one of k GPUs computes per step), exact and fast, soa-mb."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import R32, _time  # noqa: E402
from paper_2302_08251_b200 import lamina as L  # noqa: E402

n = 128 * 1024
v = L.View(L.Layout(R32, f"i64:[{n}]", os.environ.get("NB_LAYOUT", "soa-mb")))
v.nbody_init(42)
for mode, name in ((0, "exact"), (1, "fast")):
    base = None
    for k in (1, 2, 4, 8):
        ms = _time(lambda: v.nbody_update(mode, 0, n // k), reps=5, warm=2)
        base = base or ms
        print(f"{name:5} shard 1/{k}: {ms:8.3f} ms  {n * (n // k) / ms / 1e9:7.3f} e12 inter/s  "
              f"predicted speed-up {base / ms:5.2f}x of {k}", flush=True)
