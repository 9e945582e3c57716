"""Exact n-body kernel shapes (LAMB_NB_EXACT_SHAPE) at 128K and at a 16K shard."""
import os
import subprocess
import sys

if len(sys.argv) > 1:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench_suite import R32, _time
    from paper_2302_08251_b200 import lamina as L
    n = 128 * 1024
    v = L.View(L.Layout(R32, f"i64:[{n}]", "soa-mb"))
    v.nbody_init(42)
    full = min(_time(lambda: v.nbody_update(0), reps=5, warm=2) for _ in range(2))
    part = _time(lambda: v.nbody_update(0, 0, n // 2), reps=5, warm=2)
    print(f"shape={os.environ.get('LAMB_NB_EXACT_SHAPE', '0')}: 128K {full:.3f} ms ({n * n / full / 1e9:.3f}e12/s), "
          f"64K shard {part:.3f} ms", flush=True)
else:
    for sh in ("0", "1", "2", "0"):
        subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, LAMB_NB_EXACT_SHAPE=sh), check=True)
