"""Fast n-body variants (LAMB_NB_ALT = MUFU-balanced pairs of every 8): update time at 128K
and the error after 5 steps vs exact mode."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1:
    sys.path.insert(0, ROOT)
    import numpy as np
    from bench_suite import R32, _time
    from paper_2302_08251_b200 import lamina as L
    n = 128 * 1024
    v = L.View(L.Layout(R32, f"i64:[{n}]", "soa-mb"))
    v.nbody_init(42)
    ms = min(_time(lambda: v.nbody_update(1), reps=7, warm=3) for _ in range(3))
    a = L.View(L.Layout(R32, f"i64:[{n}]", "soa-mb"))
    b = L.View(L.Layout(R32, f"i64:[{n}]", "soa-mb"))
    a.nbody_init(42)
    b.nbody_init(42)
    for _ in range(5):
        a.nbody_step(1)
        b.nbody_step(0)
    pa = [x.view(np.float32).astype(np.float64) for x in a.download_all()]
    pb = [x.view(np.float32).astype(np.float64) for x in b.download_all()]
    perr = max((np.abs(x - y) / np.maximum(1, np.abs(y))).max() for x, y in zip(pa[:3], pb[:3]))
    verr = max((np.abs(x - y) / np.maximum(1e-3, np.abs(y))).max() for x, y in zip(pa[3:6], pb[3:6]))
    ips = n * n / (ms * 1e-3)
    print(f"ALT={os.environ.get('LAMB_NB_ALT', '0')}: {ms:.3f} ms  {ips / 1e12:.3f}e12 inter/s  "
          f"{ips * 20 / 1e12 / 72.19:.4f} of 72.19 TF  pos rel err {perr:.2e}  vel rel err {verr:.2e}", flush=True)
else:
    for alt in sys.argv[2:] if len(sys.argv) > 2 else ("0", "1", "8", "1", "8"):
        subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, LAMB_NB_ALT=alt), check=True)
