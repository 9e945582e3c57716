"""Profiling driver: C3 pack/unpack at 2^28 values (for ncu -k regex:k_pack32|k_unpack32)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench_suite import _fill  # noqa: E402
from paper_2302_08251_b200 import lamina as L  # noqa: E402

bits = os.environ.get("PACK_LAYOUT", "bitpack-int:3")
schema = "Record{v:f32}" if "float" in bits else "Record{v:u32}"
n = 1 << 28
src = L.View(L.Layout(schema, f"i32:[{n}]", "soa-mb"))
_fill(L, src, 3)
pk = L.View(L.Layout(schema, f"i32:[{n}]", bits))
back = L.View(L.Layout(schema, f"i32:[{n}]", "soa-mb"))
for _ in range(2):
    L.copy_view(src, pk)
    L.copy_view(pk, back)
torch.cuda.synchronize()
