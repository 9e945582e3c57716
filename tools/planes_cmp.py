"""C5-shaped copies (records -> byte planes) with and without the source slice (LAMB_PLANES_SSTAGE)."""
import os, subprocess, sys
if len(sys.argv) > 1:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench_suite import _time, _fill, R32, R64
    from paper_2302_08251_b200 import lamina as L
    from bench import peaks
    PEAK = peaks()[0]
    n = 1 << 26
    for schema, a, b, w in [(R64, "aos-packed", "changetype:f64=f32:bytesplit:soa-mb", 1), (R64, "aos-packed", "bytesplit:soa-mb", 0),
                            (R32, "aos-packed", "bytesplit:soa-mb", 0), (R64, "changetype:f64=f32:bytesplit:soa-mb", "aos-packed", 0),
                            (R64, "bytesplit:soa-mb", "aos-packed", 0), (R32, "bytesplit:soa-mb", "aos-packed", 0)]:
        la, lb = L.Layout(schema, f"i32:[{n}]", a), L.Layout(schema, f"i32:[{n}]", b, wrap=w)
        s, d = L.View(la), L.View(lb)
        _fill(L, s, 1)
        ms = _time(lambda: L.copy_view(s, d), reps=5, warm=2)
        byt = sum(la.blob_sizes) + sum(lb.blob_sizes)
        print(f"stage={os.environ.get('LAMB_PLANES_SSTAGE', '1')} {schema[:12]} {a} -> {b} wrap={w}: {byt / ms / 1e6:.0f} GB/s {byt / ms / 1e6 / PEAK:.3f}", flush=True)
        del s, d
else:
    for st in ("1",):
        subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, LAMB_PLANES_SSTAGE=st), check=True)
