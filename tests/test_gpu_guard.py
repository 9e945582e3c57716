"""Out-of-bounds write check without a sanitizer (compute-sanitizer is closed on the GPU pool:
profiles/r02/compute_sanitizer_refused.log): every destination blob is followed (and preceded)
by a guard band of a known byte pattern in the same allocation; after the copy the guards must
be intact.  Covers every kernel family at sizes with ragged tails (stray writes inside a blob
show up as parity failures in test_gpu_copy / test_gpu_scale instead)."""
import numpy as np
import pytest

from conftest import MIXED, R32, R64

pytestmark = pytest.mark.gpu

GUARD = 4096
PAIRS = [
    (R32, "aos-packed", "soa-mb"), (R32, "soa-mb", "aos-packed"), (R32, "aosoa:8", "aosoa:32"),
    (R32, "aos-packed", "aosoa:3"), (R32, "aos-packed", "bytesplit:soa-mb"), (R32, "bytesplit:soa-mb", "aos-packed"),
    (R32, "aos-packed", "changetype:f32=f64:soa-mb"), (R32, "aos-packed", "split:Pos:soa-mb:aos-packed"),
    (R32, "soa-mb", "bitpack-float:8,10"), (R32, "bitpack-float:5,10", "soa-mb"), (R32, "aos-packed", "bitpack-float:5,10"),
    (R64, "aos-packed", "changetype:f64=f32:bytesplit:soa-mb"), (R64, "changetype:f64=f32:bytesplit:soa-mb", "aos-packed"),
    (MIXED, "aos-packed", "soa-mb"), (MIXED, "soa-sb", "aos-aligned"),
    ("Record{v:u32,w:i32}", "soa-mb", "bitpack-int:7"), ("Record{v:u32,w:i32}", "bitpack-int:13", "soa-mb"),
    # record-side one-pass packing (k_rec_pack / k_rec_unpack)
    (R32, "bitpack-float:8,10", "aos-packed"), (R32, "bitpack-float:5,10", "aosoa:8"), (R32, "aosoa:16", "bitpack-float:8,10"),
    ("Record{v:u32,w:i32}", "bitpack-int:7", "aos-packed"), ("Record{v:u32,w:i32}", "aosoa:4", "bitpack-int:29"),
    # round 2: packv (1/2/8-byte leaves, fields wider than 32 bits), compile-time f32 formats
    ("Record{v:u16,w:i16}", "soa-mb", "bitpack-int:5"), ("Record{v:u16,w:i16}", "bitpack-int:11", "soa-mb"),
    ("Record{a:i8,b:u8}", "soa-mb", "bitpack-int:3"), ("Record{a:i8,b:u8}", "bitpack-int:7", "aosoa:32"),
    ("Record{v:u64,w:i64}", "soa-mb", "bitpack-int:47"), ("Record{v:u64,w:i64}", "bitpack-int:33", "soa-mb"),
    (R64, "soa-mb", "bitpack-float:11,52"), (R64, "bitpack-float:5,10", "soa-mb"),
    (R32, "soa-mb", "bitpack-float:4,3"), (R32, "bitpack-float:4,3", "soa-mb"),
    (R32, "soa-mb", "bitpack-float:11,30"), (R32, "bitpack-float:11,30", "soa-mb"),
]


@pytest.mark.parametrize("n", [37, 4099, 1_000_003])
@pytest.mark.parametrize("schema,a,b", PAIRS)
def test_copy_writes_stay_inside_blobs(schema, a, b, n):
    import torch
    from paper_2302_08251_b200 import lamina as L
    ext = f"i32:[{n}]"
    la, lb = L.Layout(schema, ext, a), L.Layout(schema, ext, b)
    src = L.View(la)
    bufs, ptrs = [], []
    for s in lb.blob_sizes:
        t = torch.full((s + 2 * GUARD,), 0xA5, dtype=torch.uint8, device="cuda")
        bufs.append(t)
        ptrs.append(t.data_ptr() + GUARD)  # 16-byte aligned: GUARD is a multiple of 256
    dst = L.View(lb, blobs=ptrs, blob_bytes=list(lb.blob_sizes))
    L.copy_view(src, dst)
    torch.cuda.synchronize()
    for k, t in enumerate(bufs):
        h = t.cpu().numpy()
        assert (h[:GUARD] == 0xA5).all(), f"blob {k}: write before the blob"
        assert (h[GUARD + lb.blob_sizes[k]:] == 0xA5).all(), f"blob {k}: write past the blob"
