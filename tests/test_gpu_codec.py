"""Exhaustive minifloat codec check on the GPU (SURVEY §7 "floatEncode parity").

Every one of the 2^32 f32 bit patterns is packed to e8m10, e5m10 and eight other (E, M)
formats through the fast path (register pack kernel: TF32/half encoders for e8m10/e5m10, the
32-bit float_encode_f32 / float_decode_f32 for the rest) and through the generic interpreter
(integer-exact floatEncode restatement, bitpack.cpp:96-163); the packed streams must be
identical, and so must the unpacked values.  A 2M-value random subset is compared with
the reference library itself (oracle/_ref).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CHUNK = 1 << 28


def _pair(fmt, n):
    from paper_2302_08251_b200 import lamina as L
    src = L.Layout("Record{v:f32}", f"i32:[{n}]", "soa-mb")
    dst = L.Layout("Record{v:f32}", f"i32:[{n}]", f"bitpack-float:{fmt}")
    return L, src, dst


@pytest.mark.parametrize("fmt", ["8,10", "5,10", "4,3", "5,2", "8,7", "6,9", "8,23", "3,0", "2,5", "11,20"])
def test_all_f32_patterns_fast_equals_generic(fmt):
    import torch
    L, ls, ld = _pair(fmt, CHUNK)
    words = ld.blob_size(0) // 4
    vals = torch.empty(CHUNK, dtype=torch.int64, device="cuda")
    fast = torch.empty(words, dtype=torch.int32, device="cuda")
    gen = torch.empty(words, dtype=torch.int32, device="cuda")
    back_f = torch.empty(CHUNK, dtype=torch.int32, device="cuda")
    back_g = torch.empty(CHUNK, dtype=torch.int32, device="cuda")
    v32 = torch.empty(CHUNK, dtype=torch.int32, device="cuda")
    vs = L.View(ls, blobs=[v32.data_ptr()], blob_bytes=[v32.numel() * 4])
    vf = L.View(ld, blobs=[fast.data_ptr()], blob_bytes=[fast.numel() * 4])
    vg = L.View(ld, blobs=[gen.data_ptr()], blob_bytes=[gen.numel() * 4])
    bf = L.View(ls, blobs=[back_f.data_ptr()], blob_bytes=[back_f.numel() * 4])
    bg = L.View(ls, blobs=[back_g.data_ptr()], blob_bytes=[back_g.numel() * 4])
    for c in range((1 << 32) // CHUNK):
        torch.arange(c * CHUNK, (c + 1) * CHUNK, dtype=torch.int64, device="cuda", out=vals)
        v32.copy_((vals - (vals >= 2**31).to(torch.int64) * 2**32).to(torch.int32))
        os.environ.pop("LAMB_FORCE_GENERIC", None)
        L.copy_view(vs, vf)
        L.copy_view(vf, bf)
        os.environ["LAMB_FORCE_GENERIC"] = "1"
        L.copy_view(vs, vg)
        L.copy_view(vg, bg)
        os.environ.pop("LAMB_FORCE_GENERIC", None)
        torch.cuda.synchronize()
        assert torch.equal(fast, gen), f"chunk {c}: packed streams differ"
        assert torch.equal(back_f, back_g), f"chunk {c}: decoded values differ"


@pytest.mark.parametrize("fmt", ["8,10", "5,10", "4,3", "11,20"])
def test_random_subset_against_reference(fmt, ref):
    from oracle import lamina_oracle as O
    L, ls, ld = _pair(fmt, 1 << 21)
    rng = np.random.default_rng(99)
    bits = rng.integers(0, 2**32, 1 << 21, dtype=np.uint64).astype(np.uint32)
    src = L.View(ls)
    dst = L.View(ld)
    src.upload(0, bits.view(np.uint8))
    L.copy_view(src, dst)
    packed = dst.download(0)
    e, m = map(int, fmt.split(","))
    w = 1 + e + m
    got = O.read_bits(packed, np.arange(bits.size, dtype=np.uint64) * np.uint64(w), w)
    want = ref.float_encode_f32(bits, e, m)
    assert np.array_equal(got, want)


def test_fast_sqrt_rcp_equal_ieee_over_exact_nbody_range(tmp_path):
    """The exact n-body's MUFU + Newton 1/sqrt equals __frcp_rn(__fsqrt_rn(x)) on every float of
    its fast-path range (sqrt over [2^-40, 2^40], rcp over [2^-20, 2^20]), exhaustively."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = os.path.join(root, "tools", "scratch", "sqrt_rcp.cu")
    exe = tmp_path / "sqrt_rcp"
    subprocess.run(["nvcc", "-std=c++20", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", str(exe), src],
                   check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300).stdout
    assert out.count("mismatches") == 2 and out.count(": 0\n") == 2, out
