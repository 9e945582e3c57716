"""Generated (NVRTC) pair kernels vs the fixed engines: identical blobs and GB/s, LAMB_JIT=1 vs 0.

GB/s counts source + destination blob bytes.  The fixed engines are parity-tested against the
oracle (tests/test_gpu_copy.py); this compares the generated kernel's blobs with theirs byte for
byte, destination pre-filled so padding bytes are checked too."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from bench_suite import _time, _fill, R32, R64
from paper_2302_08251_b200 import lamina as L
from bench import peaks

PEAK = peaks()[0]
MIXED = "Record{a:f64,b:u16,c:i8,d:f32}"
MIX2 = "Record{a:i8,b:u16,c:i32,d:u64,e:f32,f:f64,h:Record{x:i16,y:f32[3]}}"
MIXB = "Record{a:i8,b:u16,c:i32,d:u64,e:f32,f:f64,g:bool,h:Record{x:i16,y:f32[3]}}"  # tests/conftest.py MIXED
DUMP = os.path.abspath("gpurun_out/jit_src.cu")
PAIRS = [
    (MIXED, "aos-packed", "soa-mb"), (MIXED, "soa-mb", "aos-packed"), (MIXED, "aos-packed", "soa-sb"),
    (MIXED, "aosoa:8", "aos-aligned"), (MIXED, "aos-aligned", "aos-packed"), (MIXED, "aos-packed", "aosoa:16"),
    (MIXED, "aosoa:32", "aos-packed"), (MIX2, "aos-packed", "soa-mb"), (MIX2, "soa-mb", "aos-aligned"),
    (R32, "aos-packed", "aosoa:3"), (R32, "aosoa:3", "aos-packed"), (R32, "soa-mb", "aosoa:3"),
    (R32, "aosoa:6", "soa-sb"), (R32, "aosoa:32", "aosoa:3"), (R64, "aos-packed", "aosoa:3"),
    (R64, "aosoa:3", "soa-mb"), ("Record{a:u16,b:u8}", "aos-packed", "soa-mb"),
    ("Record{a:u16,b:u8}", "aos-aligned", "soa-mb"),
    (MIXB, "aos-packed", "soa-mb"), (MIXB, "soa-mb", "aos-packed"), (MIXB, "aos-packed", "aos-aligned"),
    (MIXB, "aosoa:8", "soa-mb"),
    (MIXED, "aos-packed", "bytesplit:soa-sb"), (MIXED, "aos-packed", "bytesplit:soa-mb"),
    (MIXED, "bytesplit:soa-mb", "aos-packed"), (MIXB, "aos-packed", "bytesplit:soa-mb"),
    (R64, "aosoa:8", "bytesplit:aosoa:32"),
]


def run(schema, a, b, n, jit, reps, stage=True):
    os.environ["LAMB_JIT"] = "1" if jit else "0"
    os.environ["LAMB_JIT_STAGE"] = "a" if stage else "1"
    la, lb = L.Layout(schema, f"i32:[{n}]", a), L.Layout(schema, f"i32:[{n}]", b)
    s, d = L.View(la), L.View(lb)
    _fill(L, s, 1)
    rng = np.random.default_rng(7)
    d.upload_all([rng.integers(0, 256, sz, dtype=np.uint8) for sz in lb.blob_sizes])
    before = os.path.getsize(DUMP) if os.path.exists(DUMP) else 0
    L.copy_view(s, d)
    d.sync()
    took = (os.path.getsize(DUMP) if os.path.exists(DUMP) else 0) > before
    out = [x.copy() for x in d.download_all()]
    ms = _time(lambda: L.copy_view(s, d), reps=reps, warm=1) if reps else 0.0
    byt = sum(la.blob_sizes) + sum(lb.blob_sizes)
    del s, d
    return out, (byt / ms / 1e6 if ms else 0.0), took


def main():
    os.makedirs("gpurun_out", exist_ok=True)
    os.environ["LAMB_JIT_DUMP"] = DUMP
    os.environ["LAMB_JIT_LOG"] = "1"
    big = int(os.environ.get("JIT_N", 1 << 26))
    bad = 0
    for schema, a, b in PAIRS:
        for n in (100003, big):
            reps = 3 if n == big else 0
            t0 = time.time()
            o1, g1, took = run(schema, a, b, n, True, reps)
            c1 = time.time() - t0
            o0, g0, _ = run(schema, a, b, n, False, reps)
            o2, g2, _ = run(schema, a, b, n, True, reps, stage=False)
            same = all(len(o) == len(o0) and all(np.array_equal(x, y) for x, y in zip(o, o0)) for o in (o1, o2))
            bad += not same
            tag = f"{schema[:20]:20} {a:>12} -> {b:<12} n={n:<9}"
            if reps:
                print(f"{tag} jit={'Y' if took else 'n'} same={same} jit {g1:6.0f} GB/s ({g1 / PEAK:.2f}) "
                      f"both-staged {g2 / PEAK:.2f} fixed {g0:6.0f} GB/s ({g0 / PEAK:.2f})  first-call {c1:.2f}s", flush=True)
            else:
                print(f"{tag} jit={'Y' if took else 'n'} same={same}", flush=True)
    print("jit_pairs:", "OK" if not bad else f"{bad} MISMATCHES")


if __name__ == "__main__":
    main()
