"""Fast n-body update at 128K: the single view vs nbody_distributed at world 1 (j from the
exchange buffer), same process, alternating."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_suite import R32, _time  # noqa: E402
from paper_2302_08251_b200 import lamina as L  # noqa: E402
from paper_2302_08251_b200.distributed import nbody_distributed  # noqa: E402

n = 128 * 1024
v = L.View(L.Layout(R32, f"i64:[{n}]", "soa-mb"))
v.nbody_init(42)
for rep in range(3):
    ms = _time(lambda: v.nbody_update(1), reps=10, warm=3)
    t = {}
    nbody_distributed("soa-mb", n, 10, mode=1, timing=t)
    print(f"view {ms:.3f} ms   distributed update {t['update_ms']:.3f} ms  step {t['step_ms']:.3f} ms", flush=True)
