"""Tile-engine tuning sweep on the GPU over the LAMB_TILE_* knobs (host planner reads them per call)."""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"
KNOBS = ["LAMB_TILE_KB", "LAMB_TILE_STAGES", "LAMB_TILE_THREADS", "LAMB_TILE_STG", "LAMB_TILE_DSTAGES",
         "LAMB_TILE_LMODE", "LAMB_TILE_CHUNK"]


def main():
    import torch
    from paper_2302_08251_b200 import lamina as L
    n = 1 << 26
    ext = f"i32:[{n}]"
    pairs = [("aos-packed", "soa-mb"), ("soa-mb", "aos-packed"), ("aosoa:8", "aosoa:32"), ("soa-sb", "aosoa:8")]
    views = {}
    for a in {x for p in pairs for x in p}:
        views[a] = (L.View(L.Layout(R32, ext, a)), L.View(L.Layout(R32, ext, a)))
    grid = [(kb, st, th, 1, 2, 1, 0) for kb, st, th in itertools.product([12, 24, 36, 48], [2, 3, 4], [256, 512])]
    grid += [(kb, st, 256, 1, 2, 0, ch) for kb, st, ch in itertools.product([24, 36], [2, 4], [1024, 4096])]
    if len(sys.argv) > 1:
        grid = [tuple(float(x) for x in g.split(",")) for g in sys.argv[1:]]
    for cfg in grid:
        for k, v in zip(KNOBS, cfg):
            os.environ[k] = str(v)
        row = dict(zip(["kb", "stages", "threads", "stg", "dstages", "lmode", "chunk"], cfg))
        for a, b in pairs:
            s, d = views[a][0], views[b][1]
            L.copy_view(s, d)
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            for r in range(3):
                ev[2 * r].record()
                L.copy_view(s, d)
                ev[2 * r + 1].record()
            torch.cuda.synchronize()
            ms = min(ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(3))
            row[f"{a}->{b}"] = round(56 * n / ms / 1e6, 1)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
