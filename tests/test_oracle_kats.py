"""Pins the numpy oracle (oracle/lamina_oracle.py) to the reference's own known-answer
tests.  Each test cites the reference test it restates (paths under /root/reference/proj).
CPU only."""
import math

import numpy as np
import pytest

from conftest import R32
from oracle import lamina_oracle as O

U = np.uint64
PARTICLE64 = "Record{Pos:Record{x:f64,y:f64,z:f64},Vel:Record{x:f64,y:f64,z:f64},Mass:f64}"
PARTICLE = "Record{Pos:Record{x:f64,y:f64,z:f64},Mass:f32}"  # test_mappings.cpp:17-20


def d2b(x):
    return int(np.float64(x).view(U))


def enc(x, e, m):
    return int(O.float_encode(np.array([d2b(x)], U), e, m)[0])


def dec(p, e, m):
    return float(O.float_decode(np.array([p], U), e, m).view(np.float64)[0])


# ---- tests/unit/test_bitpack.cpp ----------------------------------------------------------
def test_bit_fields_straddle_bytes():  # test_bitpack.cpp:18-46 (seed differs; same oracle idea)
    rng = np.random.default_rng(11)
    data = np.zeros(64, np.uint8)
    bits = np.zeros(512, bool)
    for _ in range(500):
        w = int(rng.integers(1, 65))
        off = int(rng.integers(0, 512 - w))
        v = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        O.write_bits(data, np.array([off], U), w, np.array([v], U))
        for k in range(w):
            bits[off + k] = (v >> k) & 1
        exp = sum(int(bits[off + k]) << k for k in range(w))
        assert int(O.read_bits(data, np.array([off], U), w)[0]) == exp
    assert np.array_equal(np.packbits(bits, bitorder="little"), data)


def test_minifloat_anchors():  # test_bitpack.cpp:73-92
    assert enc(1.0, 5, 10) == 0x3C00
    assert enc(0.0, 5, 10) == 0x0000
    assert enc(-0.0, 5, 10) == 0x8000
    assert enc(math.inf, 5, 10) == 0x7C00
    assert enc(-math.inf, 5, 10) == 0xFC00
    assert enc(65504.0, 5, 10) == 0x7BFF
    assert enc(65520.0, 5, 10) == 0x7C00
    assert enc(-65520.0, 5, 10) == 0xFC00
    assert enc(1e300, 5, 10) == 0x7C00
    assert enc(65519.999, 5, 10) == 0x7BFF
    assert enc(math.ldexp(1.0, -24), 5, 10) == 0x0001
    assert enc(math.ldexp(1.0, -26), 5, 10) == 0x0000
    assert dec(0x3C00, 5, 10) == 1.0
    assert dec(0x7BFF, 5, 10) == 65504.0


def test_nan_sign():  # test_bitpack.cpp:94-103
    plus = enc(math.nan, 5, 10)
    assert (plus >> 10) & 0x1F == 0x1F and plus & 0x3FF and not plus & 0x8000
    minus = int(O.float_encode(np.array([0xFFF8000000000000], U), 5, 10)[0])
    assert minus & 0x8000 and minus & 0x3FF
    assert math.isnan(dec(plus, 5, 10))


def test_binary16_equivalence():  # test_bitpack.cpp:105-128: every binary16 decode, random encodes
    p = np.arange(65536, dtype=U)
    d = O.float_decode(p, 5, 10).view(np.float64)
    h = p.astype(np.uint16).view(np.float16).astype(np.float64)
    nan = np.isnan(h)
    assert np.array_equal(np.isnan(d), nan)
    assert np.array_equal(d[~nan].view(U), h[~nan].view(U))
    rng = np.random.default_rng(5)
    e = rng.integers(-32, 32, 10000)
    v = (1.0 + rng.random(10000)) * np.exp2(e.astype(float)) * np.where(rng.random(10000) < 0.5, -1, 1)
    got = O.float_encode(v.view(U), 5, 10)
    ref16 = v.astype(np.float16).view(np.uint16).astype(U)  # IEEE RNE binary16
    assert np.array_equal(got, ref16)


def test_e8m23_is_binary32():  # test_bitpack.cpp:130-142
    rng = np.random.default_rng(17)
    b32 = rng.integers(0, 2**32, 10000, dtype=U)
    f = b32.astype(np.uint32).view(np.float32)
    keep = ~np.isnan(f)
    d = f[keep].astype(np.float64).view(U)
    assert np.array_equal(O.float_encode(d, 8, 23), b32[keep])
    assert np.array_equal(O.float_decode(b32[keep], 8, 23), d)


def test_monotone():  # test_bitpack.cpp:144-165
    rng = np.random.default_rng(23)
    v = np.sort((1.0 + rng.random(2000)) * np.exp2(rng.integers(-28, 20, 2000).astype(float)))
    for e in range(2, 9):
        for m in (1, 4, 10):
            out = O.float_encode(v.view(U), e, m)
            assert np.all(np.diff(out.astype(np.int64)) >= 0)


def test_pack_int_kats():  # test_bitpack.cpp:48-71
    m = O.BitpackInt(O.Schema.parse("Record{v:i64}"), 1, 4)
    blob = [np.zeros(4, np.uint8)]
    m.write(blob, 0, np.array([np.int64(-3).view(U)]))
    assert int(O.read_bits(blob[0], np.array([0], U), 4)[0]) == 0b1101
    assert int(m.read(blob, 0)[0].view(np.int64)) == -3
    for b in range(1, 13):
        p = np.arange(1 << b, dtype=U)
        mm = O.BitpackInt(O.Schema.parse("Record{v:u64}"), p.size, b)
        bl = [np.zeros(mm.blob_sizes()[0], np.uint8)]
        mm.write(bl, 0, p | U(1 << 40))
        assert np.array_equal(mm.read(bl, 0), p)


# ---- tests/unit/test_computed.cpp -----------------------------------------------------------
def test_bitpack_streams_and_sizes():  # test_computed.cpp:32-42, 106-113
    s = O.Schema.parse("Record{v:u16}")
    assert O.BitpackInt(s, 10, 3).name() == "bitpack-int:3"
    assert O.BitpackInt(s, 5, 7).blob_sizes() == [8]
    f = O.BitpackFloat(O.Schema.parse("Record{x:f64}"), 5, 5, 10)
    assert f.blob_sizes() == [((5 * 16 + 31) // 32) * 4]


def test_signed_bitpack_sign_extends():  # test_computed.cpp:63-74
    m = O.BitpackInt(O.Schema.parse("Record{v:i32}"), 16, 4)
    bl = [np.zeros(m.blob_sizes()[0], np.uint8)]
    vals = np.arange(-8, 8, dtype=np.int64)
    m.write(bl, 0, vals.astype(np.int32).view(np.uint32).astype(U))
    assert np.array_equal(m.read(bl, 0).astype(np.uint32).view(np.int32), vals)
    m2 = O.BitpackInt(O.Schema.parse("Record{v:i32}"), 1, 4)
    b2 = [np.zeros(4, np.uint8)]
    m2.write(b2, 0, np.array([9], U))
    assert int(m2.read(b2, 0)[0].astype(np.uint32).view(np.int32)) == -7


def test_changetype_kats():  # test_computed.cpp:115-145
    m = O.make("Record{x:f64}", "i64:[4]", "changetype:f64=f32")
    bl = O.zero_blobs(m)
    m.write(bl, 0, np.full(4, d2b(0.1), U))
    assert m.read(bl, 0)[0].view(np.float64) == 0.10000000149011612
    m = O.make("Record{v:i64}", "i64:[4]", "changetype:i64=i32")
    bl = O.zero_blobs(m)
    m.write(bl, 0, np.array([7, (1 << 32) + 5, 0, 0], U))
    assert list(m.read(bl, 0)[:2]) == [7, 5]
    with pytest.raises(ValueError, match="unsupported type change"):
        O.make("Record{v:i32}", "i64:[2]", "changetype:i32=u32")
    with pytest.raises(ValueError, match="unsupported type change"):
        O.make("Record{v:i32}", "i64:[2]", "changetype:i32=f32")


def test_bytesplit_planes():  # test_computed.cpp:171-193
    m = O.make("Record{v:u32}", "i64:[3]", "bytesplit:soa-mb")
    assert len(m.blob_sizes()) == 4
    bl = O.zero_blobs(m)
    m.write(bl, 0, np.array([1, 2, 3], U))
    assert list(bl[0]) == [1, 2, 3]
    assert all(not b.any() for b in bl[1:])
    assert list(m.read(bl, 0)) == [1, 2, 3]


def test_bytesplit_nan_payload():  # test_computed.cpp:218-225
    m = O.make("Record{x:f64}", "i64:[1]", "bytesplit:aos-packed")
    bl = O.zero_blobs(m)
    m.write(bl, 0, np.array([0x7FF800DEADBEEF01], U))
    assert int(m.read(bl, 0)[0]) == 0x7FF800DEADBEEF01


def test_null_mapping():  # test_computed.cpp:227-247
    m = O.make("Record{v:i32,x:f64,b:bool}", "i64:[5]", "null")
    assert m.blob_sizes() == []
    m.write([], 0, np.full(5, 42, U))
    assert not m.read([], 0).any()


# ---- tests/unit/test_mappings.cpp -------------------------------------------------------------
def test_offsets():  # test_mappings.cpp:55-122
    s = O.Schema.parse(PARTICLE)
    m = O.AoS(s, 10, False)
    assert m.blob_sizes() == [280] and int(m.offsets(3)[1][2]) == 80
    m = O.AoS(s, 10, True)
    assert m.rec == 32 and m.blob_sizes() == [320] and int(m.offsets(0)[1][1]) == 32
    s2 = O.Schema.parse("Record{x:f64,y:f64}")
    m = O.SoA(s2, 100, True)
    assert m.blob_sizes() == [800, 800] and m.offsets(1)[0] == 1 and int(m.offsets(1)[1][5]) == 40
    m = O.SoA(s2, 100, False)
    assert m.blob_sizes() == [1600] and m.base[1] == 800 and int(m.offsets(1)[1][5]) == 840
    m = O.AoSoA(s, 10, 4)
    assert m.block == 112 and m.blob_sizes() == [336] and int(m.offsets(1)[1][5]) == 152
    a, b = O.AoSoA(s, 13, 1), O.AoS(s, 13, False)
    for f in range(len(s.leaves)):
        assert np.array_equal(a.offsets(f)[1], b.offsets(f)[1])


@pytest.mark.parametrize("layout", ["aos-packed", "aos-aligned", "soa-sb", "soa-mb", "aosoa:3", "aosoa:8"])
def test_disjoint_and_total(layout):  # test_mappings.cpp:27-52
    m = O.make("Record{a:u8,b:f64,c:Record{d:i16,e:f32[2]}}", "i32:[11]", layout)
    cover = [np.zeros(s, np.int32) for s in m.blob_sizes()]
    for f, l in enumerate(m.schema.leaves):
        nr, off = m.offsets(f)
        for k in range(l.size):
            np.add.at(cover[nr], (off + U(k)).astype(np.int64), 1)
    assert max(c.max() for c in cover) == 1
    if layout in ("aos-packed", "soa-sb", "soa-mb") or layout == "aosoa:1":
        assert all(c.min() == 1 for c in cover)


# ---- tests/unit/test_view.cpp -----------------------------------------------------------------
def test_copy_across_layouts_roundtrip():  # test_view.cpp:211-237
    rng = np.random.default_rng(90)
    vals = rng.integers(0, 2**32, (6, 7), dtype=U)
    src = O.make(R32, "i64:[6]", "aos-packed")
    sb = O.zero_blobs(src)
    O.write_all(src, sb, vals)
    for name in ["soa-mb", "aosoa:4", "bytesplit:soa-sb", "split:Pos:soa-mb:aos-packed"]:
        dst = O.make(R32, "i64:[6]", name)
        db = O.zero_blobs(dst)
        O.copy_view(src, sb, dst, db)
        assert np.array_equal(O.read_all(dst, db), O.read_all(src, sb))
        back = O.make(R32, "i64:[6]", "aos-packed")
        bb = O.zero_blobs(back)
        O.copy_view(dst, db, back, bb)
        assert np.array_equal(bb[0], sb[0])


def test_copy_projection():  # test_view.cpp:239-253
    src = O.make("Record{x:f64}", "i64:[3]", "aos-packed")
    sb = O.zero_blobs(src)
    src.write(sb, 0, np.array([0.1, -2.0, 1e30]).view(U))
    dst = O.make("Record{x:f64}", "i64:[3]", "changetype:f64=f32")
    db = O.zero_blobs(dst)
    O.copy_view(src, sb, dst, db)
    got = dst.read(db, 0).view(np.float64)
    assert got[0] == 0.10000000149011612 and got[1] == -2.0 and got[2] == float(np.float32(1e30))


def test_copy_rejects_mismatch():  # test_view.cpp:255-263
    a = O.make(R32, "i64:[4]", "aos-packed")
    b = O.make(R32, "i64:[5]", "aos-packed")
    with pytest.raises(ValueError, match="incompatible views"):
        O.copy_view(a, O.zero_blobs(a), b, O.zero_blobs(b))


# ---- tests/unit/test_instrument.cpp ------------------------------------------------------------
def test_write_counters():  # test_instrument.cpp:54-70
    m = O.make("Record{a:f32,b:f32,c:i32,d:u8}", "i64:[10]", "field-access-count(aos-packed)")
    bl = O.zero_blobs(m)
    O.write_all(m, bl, np.ones((10, 4), U))
    assert list(m.writes) == [10] * 4 and list(m.reads) == [0] * 4


def test_heatmap_blocks():  # test_instrument.cpp:72-93
    m = O.make("Record{a:f32,b:f32}", "i64:[1]", "heatmap:1(aos-packed)")
    m.read(O.zero_blobs(m), 1)
    assert list(m.blocks[0]) == [0, 0, 0, 0, 1, 1, 1, 1]
    m = O.make("Record{a:f32,b:f32}", "i64:[1]", "heatmap:64(aos-packed)")
    m.read(O.zero_blobs(m), 1)
    assert list(m.blocks[0]) == [1]


def test_heatmap_crib_sheet():  # SURVEY §9 (probe of instrument.cpp:163-176 under copyView, N=64)
    rng = np.random.default_rng(1)
    vals = rng.integers(0, 2**32, (64, 7), dtype=U)
    src = O.make(R32, "i64:[64]", "soa-mb")
    sb = O.zero_blobs(src)
    O.write_all(src, sb, vals)
    for lay, g, total in [("aosoa:8", 1, 1792), ("aos-packed", 64, 448),
                          ("changetype:f32=f32:bytesplit:soa-mb", 1, 1792),
                          ("changetype:f32=f32:bytesplit:soa-mb", 64, 1792)]:
        dst = O.make(R32, "i64:[64]", f"heatmap:{g}({lay})")
        O.copy_view(src, sb, dst, O.zero_blobs(dst))
        assert sum(int(b.sum()) for b in dst.blocks) == total
    dst = O.make("Record{v:u32}", "i64:[64]", "heatmap:1(bitpack-int:3)")
    s1 = O.make("Record{v:u32}", "i64:[64]", "soa-mb")
    O.copy_view(s1, O.zero_blobs(s1), dst, O.zero_blobs(dst))
    assert int(dst.blocks[0].sum()) == 80 and list(dst.blocks[0][:8]) == [3, 4, 3, 3, 4, 3, 3, 4]


# ---- tests/unit/test_kernel.cpp + acceptance.cpp (n-body) --------------------------------------
def test_two_body_kat():  # test_kernel.cpp:64-88 (double precision)
    pos = np.array([[-1.0, 0, 0], [1.0, 0, 0]])
    vel = np.zeros((2, 3))
    mass = np.array([3.0, 3.0])
    v = O.nbody_update(pos, vel, mass, np.float64)
    dx = -2.0
    d2 = 0.01 + dx * dx + 0.0 + 0.0
    expected = dx * (3.0 * (1.0 / math.sqrt(d2 * d2 * d2)) * 0.0001)
    assert v[0, 0] == expected and v[1, 0] == -expected and v[0, 1] == 0.0
    p = O.nbody_move(pos, v, np.float64)
    assert p[0, 0] == -1.0 + expected * 0.0001


def test_self_interaction_zero():  # test_kernel.cpp:90-100
    v = O.nbody_update(np.array([[0.5, 0, 0]]), np.zeros((1, 3)), np.array([100.0]), np.float64)
    assert not v.any()


def test_readme_nbody_checksum():  # proj/README.md:224-228 (aosoa:8, n=64, 2 steps, seed 1, f64)
    _, _, _, cs = O.nbody_run(64, 2, seed=1, dtype=np.float64)
    assert repr(cs) == "94.327718848139796" or cs == 94.327718848139796


def test_mt19937_64_first_output():  # std::mt19937_64 default-seed known answer (5489 -> 14514284786278117030)
    assert O.MT19937_64(5489)() == 14514284786278117030
