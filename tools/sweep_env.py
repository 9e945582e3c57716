"""GPU sweep over arbitrary LAMB_* env settings: args are 'VAR=v,VAR=v' configs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"
LAYS = ["aos-packed", "soa-sb", "soa-mb", "aosoa:8", "aosoa:32"]


def main():
    import torch
    from paper_2302_08251_b200 import lamina as L
    n = 1 << 26
    ext = f"i32:[{n}]"
    pairs = [(a, b) for a in LAYS for b in LAYS if a != b]
    if os.environ.get("SWEEP_PAIRS") == "4":
        pairs = [("aos-packed", "soa-mb"), ("soa-mb", "aos-packed"), ("aosoa:8", "aosoa:32"), ("soa-sb", "aosoa:8")]
    views = {a: (L.View(L.Layout(R32, ext, a)), L.View(L.Layout(R32, ext, a))) for a in LAYS}
    base = dict(os.environ)
    for cfg in sys.argv[1:]:
        os.environ.clear()
        os.environ.update(base)
        for kv in cfg.split(","):
            if kv:
                k, v = kv.split("=")
                os.environ[k] = v
        row = {"cfg": cfg}
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
        vals = [v for k, v in row.items() if "->" in k]
        row["min"], row["mean"] = min(vals), round(sum(vals) / len(vals), 1)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
