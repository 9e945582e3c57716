"""Host-pipeline diagnostics: one layout pair through lam_copy_host vs the raw link."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2302_08251_b200 import lamina as L
from bench import R32, pcie_bandwidth

n = int(os.environ.get("N", 1 << 26))
from bench import C2_LAYOUTS
pairs = [(a, b) for a in C2_LAYOUTS for b in C2_LAYOUTS] if os.environ.get("ALL") else \
    [("aos-packed", "soa-mb"), ("soa-mb", "aos-packed"), ("aos-packed", "aos-packed")]
lays = {}
for a, b in pairs:
    for x in (a, b):
        lays.setdefault(x, L.Layout(R32, f"i32:[{n}]", x))
def blobs(lay, fill):
    out = []
    for s in lay.blob_sizes:
        t = torch.empty(s, dtype=torch.uint8, pin_memory=True)
        t.fill_(fill)
        out.append(t.numpy())
    return out
for a, b in pairs:
    src, dst = blobs(lays[a], 3), blobs(lays[b], 0)
    L.copy_view_host(lays[a], src, lays[b], dst)
    t0 = time.perf_counter()
    for _ in range(3):
        L.copy_view_host(lays[a], src, lays[b], dst)
    dt = (time.perf_counter() - t0) / 3
    tot = sum(lays[a].blob_sizes) + sum(lays[b].blob_sizes)
    print(os.environ.get("LAMB_PIPE_MB", "192"), a, b, f"{dt*1e3:.1f} ms", f"{tot/dt/1e9:.1f} GB/s link traffic", flush=True)
if os.environ.get("LINK"):
    print(pcie_bandwidth(0))
