"""Profiling driver: a few copyView calls of one layout pair on the GPU (for ncu)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default="aos-packed")
    ap.add_argument("--dst", default="soa-mb")
    ap.add_argument("--schema", default=R32)
    ap.add_argument("--n", type=int, default=1 << 26)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--dst-wrap", type=int, default=0)
    ap.add_argument("--gran", type=int, default=64)
    a = ap.parse_args()
    import torch
    from paper_2302_08251_b200 import lamina as L
    ext = f"i32:[{a.n}]"
    s = L.View(L.Layout(a.schema, ext, a.src))
    d = L.View(L.Layout(a.schema, ext, a.dst, wrap=a.dst_wrap, granularity=a.gran))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.reps)]
    for r in range(a.reps):
        ev[2 * r].record()
        L.copy_view(s, d)
        ev[2 * r + 1].record()
    torch.cuda.synchronize()
    ms = [ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(a.reps)]
    nbytes = sum(s.layout.blob_sizes) + sum(d.layout.blob_sizes)
    print(f"{a.src} -> {a.dst}: " + " ".join(f"{m:.3f}ms" for m in ms) +
          f"  best {nbytes / min(ms) / 1e6:.1f} GB/s (blob bytes {nbytes})")


if __name__ == "__main__":
    main()
