"""GPU parity: lam_copy (sm_100a kernels, through the C ABI) vs the oracle on the same inputs.

Bit-exact on every blob byte (including bytes the copy must not write: padding,
AoSoA tail lanes, bit-stream tails) and on FieldAccessCount / Heatmap counters.
"""
import json
import os

import numpy as np
import pytest

from conftest import MIXED, R32, R64, ROOT, leaf_types, random_values
from oracle import lamina_oracle as O

pytestmark = pytest.mark.gpu

LAYOUTS_R32 = ["aos-packed", "aos-aligned", "soa-sb", "soa-mb", "aosoa:8", "aosoa:32", "aosoa:3",
               "bytesplit:soa-mb", "bytesplit:aos-packed", "changetype:f32=f64:soa-mb", "split:Pos:soa-mb:aos-packed",
               "bitpack-float:5,10", "bitpack-float:8,10", "bitpack-float:11,30", "null", "one"]
LAYOUTS_MIXED = ["aos-packed", "aos-aligned", "soa-sb", "soa-mb", "aosoa:4", "bytesplit:soa-sb",
                 "changetype:f64=f32,i8=i64,u16=u8:aosoa:2", "split:h:bytesplit:soa-mb:aos-aligned",
                 "changetype:h.y=f64:bytesplit:aosoa:3"]


def lm():
    from paper_2302_08251_b200 import lamina
    return lamina


def run_pair(schema, n, a, b, vals, src_wrap=0, dst_wrap=0, gran=3, dst_prefill=None):
    L = lm()
    ext = f"i32:[{n}]"
    ms = O.make(schema, ext, a, wrap=src_wrap, gran=gran)
    md = O.make(schema, ext, b, wrap=dst_wrap, gran=gran)
    sb = O.zero_blobs(ms)
    O.write_all(ms, sb, vals)
    if O._fac_of(ms) is not None:
        O._fac_of(ms).writes[:] = 0
    if O._heat_of(ms) is not None:
        for x in O._heat_of(ms).blocks:
            x[:] = 0
    db = O.zero_blobs(md) if dst_prefill is None else [x.copy() for x in dst_prefill]
    gs = L.View(L.Layout(schema, ext, a, wrap=src_wrap, granularity=gran))
    gd = L.View(L.Layout(schema, ext, b, wrap=dst_wrap, granularity=gran))
    gs.upload_all(sb)
    gd.upload_all(db)
    O.copy_view(ms, sb, md, db)
    L.copy_view(gs, gd)
    got = gd.download_all()
    for nr, (x, y) in enumerate(zip(got, db)):
        assert np.array_equal(x, y), f"{a} -> {b} blob {nr}: {np.flatnonzero(x != y)[:8]}"
    for m, v in ((ms, gs), (md, gd)):
        fac = O._fac_of(m)
        if fac is not None:
            r, w = v.counters()
            assert np.array_equal(r, fac.reads) and np.array_equal(w, fac.writes)
        h = O._heat_of(m)
        if h is not None:
            for nr, blk in enumerate(h.blocks):
                assert np.array_equal(v.heatmap(nr), blk), f"heatmap blob {nr}"


@pytest.mark.parametrize("n", [1, 37, 1000, 4099])
@pytest.mark.parametrize("a", LAYOUTS_R32)
def test_copy_matrix_r32(a, n):
    rng = np.random.default_rng(n)
    vals = random_values(rng, [8] * 7, n)
    for b in LAYOUTS_R32:
        if "one" in (a, b) and n != 1:
            continue
        run_pair(R32, n, a, b, vals)


@pytest.mark.parametrize("n", [1, 53, 777])
@pytest.mark.parametrize("a", LAYOUTS_MIXED)
def test_copy_matrix_mixed(a, n):
    rng = np.random.default_rng(100 + n)
    types = [l.type for l in O.Schema.parse(MIXED).leaves]
    vals = random_values(rng, types, n)
    for b in LAYOUTS_MIXED:
        run_pair(MIXED, n, a, b, vals)


@pytest.mark.parametrize("b", [3, 7, 11, 12, 16, 24, 31, 32])
def test_bitpack_int_roundtrip(b):
    schema = "Record{v:u32,w:i32}"
    n = 5003
    rng = np.random.default_rng(b)
    vals = random_values(rng, [6, 2], n)
    run_pair(schema, n, "soa-mb", f"bitpack-int:{b}", vals)
    run_pair(schema, n, "aos-packed", f"bitpack-int:{b}", vals)
    # unpack: from a packed view back to physical
    packed = O.make(schema, f"i32:[{n}]", f"bitpack-int:{b}")
    pb = O.zero_blobs(packed)
    O.write_all(packed, pb, vals)
    back = O.read_all(packed, pb)
    run_pair(schema, n, f"bitpack-int:{b}", "soa-mb", back)


@pytest.mark.parametrize("wrap", [1, 2, 3])
@pytest.mark.parametrize("gran", [1, 5, 64])
def test_instrumented_copy(wrap, gran):
    rng = np.random.default_rng(7)
    n = 300
    vals = random_values(rng, [8] * 7, n)
    for a, b in [("aos-packed", "soa-mb"), ("soa-mb", "aosoa:8"), ("aos-packed", "bytesplit:soa-mb"),
                 ("aos-packed", "bitpack-float:5,10"), ("aosoa:8", "aosoa:8")]:
        run_pair(R32, n, a, b, vals, dst_wrap=wrap, gran=gran)
        run_pair(R32, n, a, b, vals, src_wrap=wrap, gran=gran)


def test_c5_layout_r64():
    """Config 5 shape: aos-packed f64 -> FieldAccessCount(changetype:f64=f32:bytesplit:soa-mb)."""
    rng = np.random.default_rng(5)
    n = 10007
    vals = random_values(rng, [9] * 7, n)
    run_pair(R64, n, "aos-packed", "changetype:f64=f32:bytesplit:soa-mb", vals, dst_wrap=1)
    run_pair(R64, n, "aos-packed", "bytesplit:changetype:f64=f32", vals, dst_wrap=1)


@pytest.mark.parametrize("a,b,wrap", [
    ("changetype:f64=f32:bytesplit:soa-mb", "aos-packed", 1),   # planes -> f64 records (f32 -> f64 read)
    ("aos-packed", "bytesplit:soa-mb", 0),                      # f64 records -> 8 planes per leaf
    ("bytesplit:soa-mb", "aos-packed", 2),                      # 8 planes -> records, heatmap on dst
])
def test_record_plane_kernels_r64(a, b, wrap):
    """planes.cu both directions at a size with a non-multiple-of-4 tail."""
    rng = np.random.default_rng(15)
    n = 4099
    vals = random_values(rng, [9] * 7, n)
    run_pair(R64, n, a, b, vals, src_wrap=wrap if wrap == 1 else 0, dst_wrap=wrap if wrap == 2 else 0)


def test_untouched_bytes_survive():
    """Bytes copyView never writes keep their prior content (padding, tails)."""
    rng = np.random.default_rng(9)
    n = 13
    vals = random_values(rng, [l.type for l in O.Schema.parse(MIXED).leaves], n)
    for b in ["aos-aligned", "aosoa:4", "bitpack-int:3"]:
        schema = MIXED if b != "bitpack-int:3" else "Record{v:u32}"
        v = vals if b != "bitpack-int:3" else random_values(rng, [6], n)
        md = O.make(schema, f"i32:[{n}]", b)
        prefill = [rng.integers(0, 256, s, dtype=np.uint8) for s in md.blob_sizes()]
        run_pair(schema, n, "soa-mb", b, v, dst_prefill=prefill)


def test_errors_match_reference():
    L = lm()
    a = L.View(L.Layout(R32, "i32:[4]", "aos-packed"))
    b = L.View(L.Layout(R32, "i32:[5]", "aos-packed"))
    with pytest.raises(L.InvalidArgument, match="incompatible views"):
        L.copy_view(a, b)
    c = L.View(L.Layout("Record{x:f64}", "i32:[4]", "aos-packed"))
    with pytest.raises(L.InvalidArgument):
        L.copy_view(a, c)


@pytest.mark.parametrize("a,b", [("aos-packed", "soa-mb"), ("soa-mb", "aosoa:32"), ("aosoa:8", "bytesplit:soa-mb"),
                                 ("soa-mb", "bitpack-float:8,10"), ("aos-aligned", "soa-sb")])
def test_copy_host_pipeline(a, b):
    """lam_copy_host: host blobs in, host blobs out, chunked through the GPU."""
    L = lm()
    rng = np.random.default_rng(11)
    n = 3_000_001
    ext = f"i32:[{n}]"
    vals = random_values(rng, [8] * 7, n)
    ms, md = O.make(R32, ext, a), O.make(R32, ext, b, wrap=1)
    sb = O.zero_blobs(ms)
    O.write_all(ms, sb, vals)
    db = O.zero_blobs(md)
    O.copy_view(ms, sb, md, db)
    got = [np.zeros_like(x) for x in db]
    _, dc = L.copy_view_host(L.Layout(R32, ext, a), sb, L.Layout(R32, ext, b, wrap=1), got)
    for nr, (x, y) in enumerate(zip(got, db)):
        assert np.array_equal(x, y), f"blob {nr}"
    assert np.array_equal(dc, O.counters(md))


def test_copy_range_shards_concatenate():
    """Sharded copies over disjoint ranges == one whole copy (multi-GPU decomposition)."""
    L = lm()
    rng = np.random.default_rng(12)
    n = 100_003
    ext = f"i32:[{n}]"
    vals = random_values(rng, [8] * 7, n)
    for a, b in [("aos-packed", "aosoa:32"), ("soa-mb", "bitpack-float:5,10"), ("aosoa:8", "soa-sb")]:
        ms, md = O.make(R32, ext, a), O.make(R32, ext, b)
        sb = O.zero_blobs(ms)
        O.write_all(ms, sb, vals)
        db = O.zero_blobs(md)
        O.copy_view(ms, sb, md, db)
        ls, ld = L.Layout(R32, ext, a), L.Layout(R32, ext, b)
        gs, gd = L.View(ls), L.View(ld)
        gs.upload_all(sb)
        unit = np.lcm(ls.shard_unit, ld.shard_unit)
        cuts = [0] + [int(k * n // 4 // unit * unit) for k in range(1, 4)] + [n]
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            L.copy_view_range(gs, gd, lo, hi)
        for x, y in zip(gd.download_all(), db):
            assert np.array_equal(x, y)
        with pytest.raises(L.InvalidArgument):
            L.copy_view_range(gs, gd, 1, n)


# ---- view dump / restore vs the reference's writeViewDump files (view_io.cpp) ------------------
DUMP_DIR = os.path.join(ROOT, "tests", "golden", "view_dump")


def _dump_cases():
    with open(os.path.join(DUMP_DIR, "index.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _dump_cases(), ids=lambda c: c["name"])
def test_restore_and_redump_reference_files(case, tmp_path):
    L = lm()
    stem = os.path.join(DUMP_DIR, case["name"])
    v = L.read_view_dump(stem)
    with open(stem + ".meta") as f:
        assert v.layout.dump_meta() == f.read()
    got = v.download_all()
    for nr, blob in enumerate(got):
        with open(f"{stem}.blob{nr}.bin", "rb") as f:
            assert blob.tobytes() == f.read(), f"blob {nr}"
    # values read through the restored device view equal the oracle's reading of the same bytes
    m = O.make(case["schema"], case["extents"], case["layout"], dyn=case["dyn"])
    want = O.read_all(m, [np.frombuffer(b.tobytes(), np.uint8).copy() for b in got])
    out = tmp_path / "again"
    L.write_view_dump(v, str(out))
    with open(stem + ".meta") as f, open(f"{out}.meta") as g:
        assert g.read() == f.read()
    for nr in range(len(got)):
        with open(f"{stem}.blob{nr}.bin", "rb") as f, open(f"{out}.blob{nr}.bin", "rb") as g:
            assert g.read() == f.read()
    # a copy out of the restored view into aos-packed round-trips the values
    dst = L.View(L.Layout(case["schema"], case["extents"], "aos-packed", dyn=case["dyn"]))
    L.copy_view(v, dst)
    md = O.make(case["schema"], case["extents"], "aos-packed", dyn=case["dyn"])
    assert np.array_equal(O.read_all(md, dst.download_all()), want)


@pytest.mark.parametrize("ext,dyn", [("u16:[4,dyn,5]", [7]), ("i16:[3,3,3]", []), ("u64:[dyn]", [1234]),
                                      ("u32:[11,dyn]", [9])])
@pytest.mark.parametrize("a,b", [("aos-packed", "soa-mb"), ("soa-sb", "aosoa:4"), ("aos-aligned", "bytesplit:soa-mb"),
                                 ("soa-mb", "changetype:f64=f32,i8=i64:aosoa:2")])
def test_copy_multidim_extents(ext, dyn, a, b):
    """Row-major linear index over multi-dimensional, dynamic and small-index-type extents
    (extents.cpp:94-103): the copy sees the same element order as the reference."""
    L = lm()
    rng = np.random.default_rng(3)
    ms = O.make(MIXED, ext, a, dyn=dyn)
    md = O.make(MIXED, ext, b, dyn=dyn)
    n = ms.n
    types = [l.type for l in O.Schema.parse(MIXED).leaves]
    vals = random_values(rng, types, n)
    sb = O.zero_blobs(ms)
    O.write_all(ms, sb, vals)
    db = O.zero_blobs(md)
    O.copy_view(ms, sb, md, db)
    gs = L.View(L.Layout(MIXED, ext, a, dyn=dyn))
    gd = L.View(L.Layout(MIXED, ext, b, dyn=dyn))
    gs.upload_all(sb)
    L.copy_view(gs, gd)
    for x, y in zip(gd.download_all(), db):
        assert np.array_equal(x, y)


def test_copy_sharded_pairs():
    """lam_copy_sharded: several (src, dst) pairs in flight at once (one GPU here)."""
    L = lm()
    n = 50_001
    ext = f"i32:[{n}]"
    rng = np.random.default_rng(21)
    vals = random_values(rng, [8] * 7, n)
    pairs, want = [], []
    for a, b in [("aos-packed", "soa-mb"), ("soa-sb", "aosoa:8"), ("aosoa:32", "bytesplit:soa-mb")]:
        ms, md = O.make(R32, ext, a), O.make(R32, ext, b)
        sb = O.zero_blobs(ms)
        O.write_all(ms, sb, vals)
        db = O.zero_blobs(md)
        O.copy_view(ms, sb, md, db)
        gs, gd = L.View(L.Layout(R32, ext, a)), L.View(L.Layout(R32, ext, b))
        gs.upload_all(sb)
        pairs.append((gs, gd))
        want.append(db)
    L.copy_sharded(pairs)
    for (_, gd), db in zip(pairs, want):
        for x, y in zip(gd.download_all(), db):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("wrap", [2, 3])
def test_copy_host_pipeline_heatmap(wrap):
    """lam_copy_host with a Heatmap (and FieldAccessCount) destination: chunked counters sum."""
    L = lm()
    rng = np.random.default_rng(13)
    n = 2_000_003
    ext = f"i32:[{n}]"
    vals = random_values(rng, [8] * 7, n)
    ms, md = O.make(R32, ext, "aos-packed"), O.make(R32, ext, "soa-mb", wrap=wrap, gran=64)
    sb = O.zero_blobs(ms)
    O.write_all(ms, sb, vals)
    db = O.zero_blobs(md)
    O.copy_view(ms, sb, md, db)
    got = [np.zeros_like(x) for x in db]
    _, dc = L.copy_view_host(L.Layout(R32, ext, "aos-packed"), sb, L.Layout(R32, ext, "soa-mb", wrap=wrap, granularity=64),
                             got)
    for x, y in zip(got, db):
        assert np.array_equal(x, y)
    assert np.array_equal(dc, O.counters(md))


@pytest.mark.parametrize("rec", ["aos-packed", "aosoa:4", "aosoa:8", "aosoa:16"])
@pytest.mark.parametrize("n", [3239, 70001])
def test_record_side_bitpack_one_pass(rec, n):
    """pack.cu k_rec_pack / k_rec_unpack: a record-contiguous side (AoS, AoSoA<L>, L | 32) against
    bit streams, several 1024-record CTAs, a partial CTA and a generic tail, both directions,
    signed/unsigned ints and the three float codecs, FieldAccessCount on either side."""
    rng = np.random.default_rng(n)
    cases = [("Record{v:u32,w:i32,x:i32}", [6, 2, 2], f"bitpack-int:{b}") for b in (3, 12, 31)]
    cases += [(R32, [8] * 7, f"bitpack-float:{f}") for f in ("8,10", "5,10", "4,3")]
    for schema, types, packed in cases:
        vals = random_values(rng, types, n)
        run_pair(schema, n, rec, packed, vals, dst_wrap=1 if "5,10" in packed else 0)
        pm = O.make(schema, f"i32:[{n}]", packed)
        pb = O.zero_blobs(pm)
        O.write_all(pm, pb, vals)
        back = O.read_all(pm, pb)
        run_pair(schema, n, packed, rec, back, src_wrap=1 if "8,10" in packed else 0)


def test_acceptance_criterion_10_relocatable_state(ref):
    """acceptance.cpp:772-790 through the C ABI: a static-extent aos-packed view of 16 particles
    is trivially relocatable with stateBytes == blobBytes == 16 * 28; a dyn-extent one is not
    and carries one i64 slot of runtime state (view.cpp:145-162)."""
    L = lm()
    fixed = L.View(L.Layout(R32, "i32:[16]", "aos-packed"))
    assert fixed.is_trivially_relocatable() and fixed.state_bytes() == fixed.blob_bytes() == 16 * 28
    dyn = L.View(L.Layout(R32, "i64:[dyn]", "aos-packed", dyn=(16,)))
    assert not dyn.is_trivially_relocatable() and dyn.state_bytes() == dyn.blob_bytes() + 8
    for text, wrap, dv, ext in (("soa-mb", 1, (), "i32:[16]"), ("aosoa:4", 2, (), "i32:[16]"),
                                ("bitpack-float:5,10", 0, (9,), "i64:[dyn]")):
        v = L.View(L.Layout(R32, ext, text, dyn=dv, wrap=wrap, granularity=5))
        _, _, tr, sb, bb = ref.state_info(R32, ext, text, dv, wrap, 5)
        assert (v.is_trivially_relocatable(), v.state_bytes(), v.blob_bytes()) == (tr, sb, bb)


# ---- edge cases the reference's own tests pin -------------------------------------------------
def test_bitpack_int16_equals_soa_u16():
    """acceptance.cpp:389-404: bitpack-int:16 over u16 leaves is byte-identical to soa-mb u16
    (the packed blob is the soa blob padded to whole 32-bit words)."""
    L = lm()
    schema, n = "Record{v:u16,w:u16}", 4099
    rng = np.random.default_rng(16)
    vals = random_values(rng, [5, 5], n)
    run_pair(schema, n, "aos-packed", "bitpack-int:16", vals)
    soa = L.View(L.Layout(schema, f"i32:[{n}]", "soa-mb"))
    ms = O.make(schema, f"i32:[{n}]", "soa-mb")
    sb = O.zero_blobs(ms)
    O.write_all(ms, sb, vals)
    soa.upload_all(sb)
    pk = L.View(L.Layout(schema, f"i32:[{n}]", "bitpack-int:16"))
    L.copy_view(soa, pk)
    for nr, blob in enumerate(pk.download_all()):
        assert blob.nbytes == (n * 16 + 31) // 32 * 4
        assert np.array_equal(blob[: 2 * n], sb[nr]) and not blob[2 * n:].any()


@pytest.mark.parametrize("schema,bits", [("Record{a:i8,b:u8}", 3), ("Record{a:i8,b:u8}", 8),
                                         ("Record{a:i16,b:u16}", 11), ("Record{v:u64}", 33),
                                         ("Record{v:u64,w:i64}", 47), ("Record{v:i64}", 64),
                                         ("Record{a:i8,b:u64,c:i16}", 5)])
@pytest.mark.parametrize("n", [1189, 4099])  # 1189: one full warp of 32-value groups plus 5 lanes
def test_bitpack_int_other_widths(schema, bits, n):
    """BitpackIntSoA on 8/16/64-bit leaves (computed.cpp:59-67,101-122): pack truncates to the
    low b bits, unpack zero/sign-extends; 1 <= b <= 8 * leaf size.  soa-mb and aosoa:32 take the
    packv kernels (partial warps included), the others the general engines."""
    rng = np.random.default_rng(bits)
    vals = random_values(rng, leaf_types(schema), n)
    for phys in ("soa-mb", "aosoa:32", "aos-packed", "aosoa:8"):
        run_pair(schema, n, phys, f"bitpack-int:{bits}", vals)
    packed = O.make(schema, f"i32:[{n}]", f"bitpack-int:{bits}")
    pb = O.zero_blobs(packed)
    O.write_all(packed, pb, vals)
    back = O.read_all(packed, pb)
    for phys in ("soa-mb", "aosoa:32", "aos-packed"):
        run_pair(schema, n, f"bitpack-int:{bits}", phys, back)


@pytest.mark.parametrize("fmt", ["11,52", "8,23", "5,10", "8,10", "4,3", "15,40"])
def test_bitpack_float_f64_leaves(fmt):
    """BitpackFloatSoA on f64 leaves (computed.cpp:133-222; bitpack.cpp:96-188): e11m52 is
    binary64 itself, the rest round through floatEncode(double)."""
    n = 4099
    rng = np.random.default_rng(52)
    vals = random_values(rng, [9] * 7, n)
    for phys in ("aos-packed", "soa-mb", "aosoa:32"):
        run_pair(R64, n, phys, f"bitpack-float:{fmt}", vals)
    packed = O.make(R64, f"i32:[{n}]", f"bitpack-float:{fmt}")
    pb = O.zero_blobs(packed)
    O.write_all(packed, pb, vals)
    run_pair(R64, n, f"bitpack-float:{fmt}", "soa-mb", O.read_all(packed, pb))


BOOLREC = "Record{a:bool,b:u8,c:bool,d:f32,e:bool}"


@pytest.mark.parametrize("generic", [False, True], ids=["specialised", "generic"])
@pytest.mark.parametrize("a,b", [("aos-packed", "soa-mb"), ("soa-mb", "aosoa:4"), ("aos-aligned", "soa-sb"),
                                 ("aos-packed", "bytesplit:soa-mb"), ("aosoa:3", "aos-packed"),
                                 ("soa-sb", "changetype:f32=f64:aos-packed")])
def test_bool_bytes_canonicalise_on_read(a, b, generic, monkeypatch):
    """ScalarValue::fromStorageBits(Bool) = bits != 0 (scalar.hpp:259-261): a bool byte 0x02..0xFF
    in the source is written as 0x01 by every fieldwise copy path."""
    L = lm()
    n = 1031
    ext = f"i32:[{n}]"
    if generic:
        monkeypatch.setenv("LAMB_FORCE_GENERIC", "1")
    ms, md = O.make(BOOLREC, ext, a), O.make(BOOLREC, ext, b)
    rng = np.random.default_rng(2)
    sb = [rng.integers(0, 256, x.size, dtype=np.uint8) for x in O.zero_blobs(ms)]
    assert any((x > 1).any() for x in sb)
    db = O.zero_blobs(md)
    O.copy_view(ms, sb, md, db)
    gs, gd = L.View(L.Layout(BOOLREC, ext, a)), L.View(L.Layout(BOOLREC, ext, b))
    gs.upload_all(sb)
    L.copy_view(gs, gd)
    for nr, (x, y) in enumerate(zip(gd.download_all(), db)):
        assert np.array_equal(x, y), f"{a} -> {b} blob {nr}: {np.flatnonzero(x != y)[:8]}"
    vals = O.read_all(md, db)
    assert set(np.unique(vals[:, [0, 2, 4]])) <= {0, 1}


@pytest.mark.parametrize("fmt", ["4,3", "5,2", "8,7", "6,9", "3,0", "11,30", "11,52", "8,23"])
@pytest.mark.parametrize("phys", ["soa-mb", "aosoa:32"])
def test_bitpack_float_f32_formats(fmt, phys):
    """f32 leaves through the compile-time-width k_pack32 (E <= 8, M <= 23: FMT 3) and, for fields
    wider than 32 bits, k_packv<4> -- both directions, ragged size, specials included."""
    n = 1189
    rng = np.random.default_rng(int(fmt.replace(",", "")))
    vals = random_values(rng, [8] * 7, n)
    run_pair(R32, n, phys, f"bitpack-float:{fmt}", vals)
    packed = O.make(R32, f"i32:[{n}]", f"bitpack-float:{fmt}")
    pb = O.zero_blobs(packed)
    O.write_all(packed, pb, vals)
    run_pair(R32, n, f"bitpack-float:{fmt}", phys, O.read_all(packed, pb))


@pytest.mark.parametrize("fmt", ["4,3", "5,2", "3,4", "8,7", "6,9", "2,1"])
@pytest.mark.parametrize("rec", ["aos-packed", "aosoa:8", "aosoa:4"])
def test_bitpack_float_record_side_formats(fmt, rec):
    """Record side <-> minifloat bit streams in one pass (k_rec_pack / k_rec_unpack with the
    branch-free f32 codec, compile-time W for 8 and 16 bits), both directions, specials included."""
    n = 2053
    rng = np.random.default_rng(int(fmt.replace(",", "")) + len(rec))
    vals = random_values(rng, [8] * 7, n)
    run_pair(R32, n, rec, f"bitpack-float:{fmt}", vals)
    packed = O.make(R32, f"i32:[{n}]", f"bitpack-float:{fmt}")
    pb = O.zero_blobs(packed)
    O.write_all(packed, pb, vals)
    run_pair(R32, n, f"bitpack-float:{fmt}", rec, O.read_all(packed, pb))


@pytest.mark.parametrize("schema,a,b", [
    ("Record{v:u32,w:i32}", "bitpack-int:11", "bitpack-int:7"),
    ("Record{v:u32,w:i32}", "bitpack-int:5", "bitpack-int:29"),
    ("Record{v:u32,w:i32}", "bitpack-int:13", "bitpack-int:13"),
    (R32, "bitpack-float:4,3", "bitpack-float:5,10"),
    (R32, "bitpack-float:8,10", "bitpack-float:4,3"),
    (R32, "bitpack-float:5,2", "bitpack-float:5,2"),
    (R32, "bitpack-float:6,9", "bitpack-float:8,23"),
    (R32, "bitpack-float:4,3", "bitpack-float:4,3"), (R32, "bitpack-float:8,10", "bitpack-float:8,10"),
    (R32, "bitpack-float:5,10", "bitpack-float:5,10"),
])
@pytest.mark.parametrize("n", [1000, 70001])
def test_bitpack_to_bitpack(schema, a, b, n):
    """Bit stream -> bit stream in one pass (k_repack32): decode / sign-extend each source field,
    encode / truncate into the destination field, tail bits untouched."""
    rng = np.random.default_rng(n + len(a) + len(b))
    types = [l.type for l in O.Schema.parse(schema).leaves]
    vals = random_values(rng, types, n)
    src = O.make(schema, f"i32:[{n}]", a)
    sb = O.zero_blobs(src)
    O.write_all(src, sb, vals)
    run_pair(schema, n, a, b, O.read_all(src, sb))
