"""GPU parity of the generated (NVRTC) pair kernels (csrc/jit.cpp) against the oracle.

The generated path serves physical pairs of records with mixed leaf sizes (and padded
destinations) that no fixed kernel covers.  Every case checks every blob byte against the
oracle's copyView, destination pre-filled with random bytes so padding must survive, and
FieldAccessCount counters; LAMB_JIT_DUMP proves the generated kernel actually ran.
"""
import os

import numpy as np
import pytest

from conftest import MIXED, random_values
from oracle import lamina_oracle as O
from test_gpu_copy import run_pair

pytestmark = pytest.mark.gpu

MIX4 = "Record{a:f64,b:u16,c:i8,d:f32}"
MIX8 = "Record{a:i8,b:u16,c:i32,d:u64,e:f32,f:f64,h:Record{x:i16,y:f32[3]}}"
TINY = "Record{a:u16,b:u8}"
BYTES3 = "Record{a:u8,b:i8,c:u8}"

PAIRS = [
    (MIX4, "aos-packed", "soa-mb"), (MIX4, "soa-mb", "aos-packed"), (MIX4, "aos-packed", "soa-sb"),
    (MIX4, "aosoa:8", "aos-aligned"), (MIX4, "aos-aligned", "aos-packed"), (MIX4, "aos-packed", "aosoa:16"),
    (MIX4, "aosoa:32", "aos-packed"), (MIX4, "soa-sb", "aosoa:32"),
    (MIX8, "aos-packed", "soa-mb"), (MIX8, "aosoa:16", "aos-packed"),
    (TINY, "aos-packed", "soa-mb"), (TINY, "aos-aligned", "soa-mb"), (TINY, "soa-sb", "aos-aligned"),
    (BYTES3, "aos-packed", "soa-mb"), (BYTES3, "soa-mb", "aos-packed"),
    # byte planes (Bytesplit): every value byte is its own term
    (MIX4, "aos-packed", "bytesplit:soa-mb"), (MIX4, "bytesplit:soa-mb", "aos-aligned"),
    (MIX4, "aosoa:16", "bytesplit:aosoa:32"), (MIX8, "bytesplit:soa-mb", "aos-packed"),
]


def _dump_size(path):
    return os.path.getsize(path) if os.path.exists(path) else 0


@pytest.mark.parametrize("n", [4099, 65536, 100003])
@pytest.mark.parametrize("schema,a,b", PAIRS)
def test_jit_pair_matches_oracle(schema, a, b, n, tmp_path, monkeypatch):
    dump = str(tmp_path / "jit.cu")
    monkeypatch.setenv("LAMB_JIT_DUMP", dump)
    rng = np.random.default_rng(n + len(a) * 7 + len(b))
    types = [l.type for l in O.Schema.parse(schema).leaves]
    vals = random_values(rng, types, n)
    md = O.make(schema, f"i32:[{n}]", b)
    prefill = [rng.integers(0, 256, x.size, dtype=np.uint8) for x in O.zero_blobs(md)]
    run_pair(schema, n, a, b, vals, dst_prefill=prefill)
    if "soa-sb" not in (a, b):  # soa-sb leaf bases are 16-byte aligned only for some n
        assert _dump_size(dump) > 0, "the generated kernel did not run for this pair"


@pytest.mark.parametrize("wrap", [1, 3])
def test_jit_pair_counters(wrap, tmp_path, monkeypatch):
    """FieldAccessCount and Heatmap wrappers around a generated-kernel pair."""
    dump = str(tmp_path / "jit.cu")
    monkeypatch.setenv("LAMB_JIT_DUMP", dump)
    n = 5003
    rng = np.random.default_rng(wrap)
    types = [l.type for l in O.Schema.parse(MIX4).leaves]
    vals = random_values(rng, types, n)
    run_pair(MIX4, n, "aos-packed", "soa-mb", vals, src_wrap=wrap, dst_wrap=wrap, gran=5)
    assert _dump_size(dump) > 0


def test_jit_range_copies(tmp_path, monkeypatch):
    """copy_view_range over consecutive ranges (begin > 0, ragged ends) equals one whole copy."""
    from paper_2302_08251_b200 import lamina as L
    dump = str(tmp_path / "jit.cu")
    monkeypatch.setenv("LAMB_JIT_DUMP", dump)
    n = 70001
    ext = f"i32:[{n}]"
    rng = np.random.default_rng(11)
    types = [l.type for l in O.Schema.parse(MIX4).leaves]
    vals = random_values(rng, types, n)
    ms, md = O.make(MIX4, ext, "aos-packed"), O.make(MIX4, ext, "soa-mb")
    sb, db = O.zero_blobs(ms), O.zero_blobs(md)
    O.write_all(ms, sb, vals)
    O.copy_view(ms, sb, md, db)
    gs, gd = L.View(L.Layout(MIX4, ext, "aos-packed")), L.View(L.Layout(MIX4, ext, "soa-mb"))
    gs.upload_all(sb)
    cuts = [0, 16, 4096, 4112, 33344, 65536, n]  # multiples of the shard unit (16)
    for lo, hi in zip(cuts, cuts[1:]):
        L.copy_view_range(gs, gd, lo, hi)
    for x, y in zip(gd.download_all(), db):
        assert np.array_equal(x, y)
    assert _dump_size(dump) > 0


def test_jit_disabled_gives_same_bytes(monkeypatch):
    """LAMB_JIT=0 (warp-tile engine) and the generated kernel write identical blobs."""
    from paper_2302_08251_b200 import lamina as L
    n = 40000
    ext = f"i32:[{n}]"
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("LAMB_JIT", flag)
        s, d = L.View(L.Layout(MIX8, ext, "aos-packed")), L.View(L.Layout(MIX8, ext, "aosoa:8"))
        s.upload_all([np.random.default_rng(5).integers(0, 256, x, dtype=np.uint8) for x in s.layout.blob_sizes])
        L.copy_view(s, d)
        outs.append([x.copy() for x in d.download_all()])
    for x, y in zip(*outs):
        assert np.array_equal(x, y)


BOOLREC = "Record{a:bool,b:u8,c:bool,d:f32,e:bool}"


@pytest.mark.parametrize("schema,a,b", [
    (BOOLREC, "aos-packed", "soa-mb"), (BOOLREC, "soa-mb", "aos-aligned"), (BOOLREC, "aosoa:16", "aos-packed"),
    (MIXED, "aos-packed", "soa-mb"), (MIXED, "soa-mb", "aos-packed"), (MIXED, "aosoa:8", "aos-packed"),
    (MIXED, "aos-packed", "bytesplit:soa-mb"), (BOOLREC, "bytesplit:soa-mb", "aos-aligned"),
    # more than 64 plan streams (42 byte planes per side)
    (MIXED, "bytesplit:soa-mb", "bytesplit:soa-mb"), (MIXED, "bytesplit:soa-mb", "bytesplit:aosoa:16"),
])
def test_jit_bool_bytes_canonicalise(schema, a, b, tmp_path, monkeypatch):
    """Source blobs of random bytes (bool bytes 0x02..0xFF included): the generated kernel writes
    every bool as 0x01 / 0x00 like ScalarValue::fromStorageBits(Bool) (scalar.hpp:259-261)."""
    from paper_2302_08251_b200 import lamina as L
    dump = str(tmp_path / "jit.cu")
    monkeypatch.setenv("LAMB_JIT_DUMP", dump)
    n = 4103
    ext = f"i32:[{n}]"
    ms, md = O.make(schema, ext, a), O.make(schema, ext, b)
    rng = np.random.default_rng(3)
    sb = [rng.integers(0, 256, x.size, dtype=np.uint8) for x in O.zero_blobs(ms)]
    db = [rng.integers(0, 256, x.size, dtype=np.uint8) for x in O.zero_blobs(md)]
    gs, gd = L.View(L.Layout(schema, ext, a)), L.View(L.Layout(schema, ext, b))
    gs.upload_all(sb)
    gd.upload_all(db)
    O.copy_view(ms, sb, md, db)
    L.copy_view(gs, gd)
    for nr, (x, y) in enumerate(zip(gd.download_all(), db)):
        assert np.array_equal(x, y), f"{a} -> {b} blob {nr}: {np.flatnonzero(x != y)[:8]}"
    assert _dump_size(dump) > 0


@pytest.mark.parametrize("schema,a,b", [
    (MIX4, "aos-packed", "changetype:f64=f32:soa-mb"), (MIX4, "changetype:f64=f32:aosoa:8", "aos-aligned"),
    (MIX4, "soa-mb", "changetype:f32=f64,u16=u32,i8=i64:aos-packed"),
    (MIXED, "aos-packed", "changetype:f64=f32,i8=i64,u16=u8:aosoa:2"),
    (MIXED, "changetype:f64=f32,i8=i64,u16=u8:aosoa:2", "soa-mb"),
    (MIXED, "aosoa:8", "changetype:h.y=f64:bytesplit:soa-mb"),
    ("Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}", "aosoa:3", "changetype:f32=f64:soa-mb"),
])
def test_jit_conversions_raw_bytes(schema, a, b, tmp_path, monkeypatch):
    """ChangeType conversions in the generated kernel (f32 <-> f64 with NaN payloads, integer
    sign extension and truncation) on source blobs of random bytes, against the oracle."""
    from paper_2302_08251_b200 import lamina as L
    dump = str(tmp_path / "jit.cu")
    monkeypatch.setenv("LAMB_JIT_DUMP", dump)
    n = 4111
    ext = f"i32:[{n}]"
    ms, md = O.make(schema, ext, a), O.make(schema, ext, b)
    rng = np.random.default_rng(17)
    sb = [rng.integers(0, 256, x.size, dtype=np.uint8) for x in O.zero_blobs(ms)]
    db = [rng.integers(0, 256, x.size, dtype=np.uint8) for x in O.zero_blobs(md)]
    gs, gd = L.View(L.Layout(schema, ext, a)), L.View(L.Layout(schema, ext, b))
    gs.upload_all(sb)
    gd.upload_all(db)
    O.copy_view(ms, sb, md, db)
    L.copy_view(gs, gd)
    for nr, (x, y) in enumerate(zip(gd.download_all(), db)):
        assert np.array_equal(x, y), f"{a} -> {b} blob {nr}: {np.flatnonzero(x != y)[:8]}"


@pytest.mark.parametrize("a,b", [("aos-packed", "soa-mb"), ("soa-mb", "aos-aligned"), ("aosoa:8", "bytesplit:soa-mb")])
def test_jit_host_pipeline(a, b, tmp_path, monkeypatch):
    """lam_copy_host (host blobs chunked through the GPU, chunk views with shifted bases) on pairs
    the generated kernels serve, with a FieldAccessCount destination."""
    from paper_2302_08251_b200 import lamina as L
    dump = str(tmp_path / "jit.cu")
    monkeypatch.setenv("LAMB_JIT_DUMP", dump)
    n = 3_000_017
    ext = f"i32:[{n}]"
    rng = np.random.default_rng(23)
    types = [l.type for l in O.Schema.parse(MIX4).leaves]
    vals = random_values(rng, types, n)
    ms, md = O.make(MIX4, ext, a), O.make(MIX4, ext, b, wrap=1)
    sb = O.zero_blobs(ms)
    O.write_all(ms, sb, vals)
    db = O.zero_blobs(md)
    O.copy_view(ms, sb, md, db)
    got = [np.zeros_like(x) for x in db]
    _, dc = L.copy_view_host(L.Layout(MIX4, ext, a), sb, L.Layout(MIX4, ext, b, wrap=1), got)
    for nr, (x, y) in enumerate(zip(got, db)):
        assert np.array_equal(x, y), f"blob {nr}"
    assert np.array_equal(dc, O.counters(md))
    assert _dump_size(dump) > 0


@pytest.mark.parametrize("a,b", [("aosoa:16", "aos-packed"), ("soa-mb", "aosoa:32"), ("aosoa:32", "bytesplit:soa-mb"),
                                 ("aosoa:16", "aosoa:32")])
def test_jit_half_spans(a, b, tmp_path, monkeypatch):
    """8-byte spans (1-byte leaves at G = 8, in SoA blobs and inside AoSoA blocks) against the
    oracle, random bytes in both views (bool canonicalisation, untouched padding)."""
    from paper_2302_08251_b200 import lamina as L
    dump = str(tmp_path / "jit.cu")
    monkeypatch.setenv("LAMB_JIT_DUMP", dump)
    n = 9001
    ext = f"i32:[{n}]"
    ms, md = O.make(MIXED, ext, a), O.make(MIXED, ext, b)
    rng = np.random.default_rng(29)
    sb = [rng.integers(0, 256, x.size, dtype=np.uint8) for x in O.zero_blobs(ms)]
    db = [rng.integers(0, 256, x.size, dtype=np.uint8) for x in O.zero_blobs(md)]
    gs, gd = L.View(L.Layout(MIXED, ext, a)), L.View(L.Layout(MIXED, ext, b))
    gs.upload_all(sb)
    gd.upload_all(db)
    O.copy_view(ms, sb, md, db)
    L.copy_view(gs, gd)
    for nr, (x, y) in enumerate(zip(gd.download_all(), db)):
        assert np.array_equal(x, y), f"{a} -> {b} blob {nr}: {np.flatnonzero(x != y)[:8]}"
    assert _dump_size(dump) > 0
