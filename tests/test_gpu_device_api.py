"""The public device API (include/lamina_b200_device.cuh) from user kernels
(paper_2302_08251_b200/examples/device_view_demo.cu -> _lib/liblamina_b200_demo.so):
View::load/store semantics through any mapping, instrumentation counts, the direct physical
accessor and the compile-time-extent shared-memory record tile, checked against the oracle."""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import R32, ROOT, random_values
from oracle import lamina_oracle as O

pytestmark = pytest.mark.gpu

DEMO = os.path.join(ROOT, "paper_2302_08251_b200", "_lib", "liblamina_b200_demo.so")


def demo():
    L = C.CDLL(DEMO)
    L.lam_demo_scale.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_float, C.c_void_p]
    L.lam_demo_phys_add.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_float, C.c_void_p]
    L.lam_demo_tile_copy7.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
    return L


def finite_r32(rng, n):
    vals = rng.standard_normal((n, 7)).astype(np.float32).view(np.uint32).astype(np.uint64)
    return vals


@pytest.mark.parametrize("layout", ["aos-packed", "soa-mb", "aosoa:8", "bitpack-float:8,23",
                                    "changetype:f32=f64:soa-sb", "bytesplit:aosoa:4", "split:Pos:soa-mb:aos-packed"])
def test_user_kernel_load_store_any_mapping(layout):
    import torch
    from paper_2302_08251_b200 import lamina as L
    n = 1000
    rng = np.random.default_rng(5)
    vals = finite_r32(rng, n)
    ext = f"i32:[{n}]"
    m = O.make(R32, ext, layout, wrap=1)
    blobs = O.zero_blobs(m)
    O.write_all(m, blobs, vals)
    v = L.View(L.Layout(R32, ext, layout, wrap=L.WRAP_FIELD_ACCESS_COUNT))
    v.upload_all(blobs)
    v.reset_counters()
    assert demo().lam_demo_scale(v.device_plan, n, 6, 2.0, None) == 0
    torch.cuda.synchronize()
    # oracle: Mass *= 2 in f32 through the mapping
    got = O.read_all(m, v.download_all())
    want = O.read_all(m, blobs).copy()
    mass = want[:, 6].astype(np.uint32).view(np.float32) * np.float32(2.0)
    want[:, 6] = mass.view(np.uint32).astype(np.uint64)
    assert np.array_equal(got, want)
    r, w = v.counters()
    assert r.tolist() == [0] * 6 + [n] and w.tolist() == [0] * 6 + [n]


@pytest.mark.parametrize("layout", ["aos-packed", "soa-sb", "aosoa:3", "aos-aligned"])
def test_user_kernel_physical_accessor(layout):
    import torch
    from paper_2302_08251_b200 import lamina as L
    n = 777
    vals = finite_r32(np.random.default_rng(6), n)
    ext = f"i32:[{n}]"
    m = O.make(R32, ext, layout)
    blobs = O.zero_blobs(m)
    O.write_all(m, blobs, vals)
    v = L.View(L.Layout(R32, ext, layout))
    v.upload_all(blobs)
    assert demo().lam_demo_phys_add(v.device_plan, n, 1, 1.5, None) == 0
    torch.cuda.synchronize()
    want = vals.copy()
    want[:, 1] = (want[:, 1].astype(np.uint32).view(np.float32) + np.float32(1.5)).view(np.uint32)
    assert np.array_equal(O.read_all(m, v.download_all()), want)


@pytest.mark.parametrize("a,b", [("aos-packed", "aosoa:8"), ("soa-mb", "bitpack-float:8,23"),
                                 ("aosoa:32", "bytesplit:soa-mb")])
def test_user_kernel_smem_record_tile(a, b):
    import torch
    from paper_2302_08251_b200 import lamina as L
    n = 1234
    vals = random_values(np.random.default_rng(7), [8] * 7, n)
    ext = f"i32:[{n}]"
    ms, md = O.make(R32, ext, a), O.make(R32, ext, b)
    sb = O.zero_blobs(ms)
    O.write_all(ms, sb, vals)
    s, d = L.View(L.Layout(R32, ext, a)), L.View(L.Layout(R32, ext, b))
    s.upload_all(sb)
    assert demo().lam_demo_tile_copy7(s.device_plan, d.device_plan, n, None) == 0
    torch.cuda.synchronize()
    db = O.zero_blobs(md)
    O.copy_view(ms, sb, md, db)
    for x, y in zip(d.download_all(), db):
        assert np.array_equal(x, y)
