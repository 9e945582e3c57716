"""Tile-engine tuning sweep on the GPU: stage size x pipeline depth x warps per CTA."""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"


def main():
    import torch
    from paper_2302_08251_b200 import lamina as L
    n = 1 << 26
    ext = f"i32:[{n}]"
    pairs = [("aos-packed", "soa-mb"), ("soa-mb", "aos-packed"), ("aosoa:8", "aosoa:32"), ("soa-sb", "aosoa:8")]
    views = {}
    for a in {x for p in pairs for x in p}:
        views[a] = (L.View(L.Layout(R32, ext, a)), L.View(L.Layout(R32, ext, a)))
    grid = list(itertools.product([12, 24, 36, 48], [2, 3, 4], [256, 512]))
    if len(sys.argv) > 1:
        grid = [tuple(float(x) for x in g.split(",")) for g in sys.argv[1:]]
    res = []
    for kb, st, th in grid:
        os.environ["LAMB_TILE_KB"] = str(kb)
        os.environ["LAMB_TILE_STAGES"] = str(int(st))
        os.environ["LAMB_TILE_THREADS"] = str(int(th))
        row = {"kb": kb, "stages": st, "threads": th}
        for a, b in pairs:
            s, d = views[a][0], views[b][1]
            L.copy_view(s, d)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
            for r in range(4):
                ev[2 * r].record()
                L.copy_view(s, d)
                ev[2 * r + 1].record()
            torch.cuda.synchronize()
            ms = min(ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(4))
            row[f"{a}->{b}"] = round(56 * n / ms / 1e6, 1)
        res.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
