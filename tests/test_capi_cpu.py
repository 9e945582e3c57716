"""C ABI on the CPU (no GPU needed): the library loads, exports every symbol the header
declares, and its host-side lowering agrees with the oracle / reference on names, blob
sizes, leaf tables, physical offsets and error behaviour.  No device calls here."""
import os
import re

import numpy as np
import pytest

from conftest import MIXED, R32, ROOT
from oracle import lamina_oracle as O

LAYOUTS = ["aos-packed", "aos-aligned", "soa-sb", "soa-mb", "aosoa:8", "aosoa:3", "bytesplit:soa-mb",
           "bytesplit:aos-packed", "changetype:f32=f64:soa-mb", "split:Pos:soa-mb:aos-packed", "null",
           "bitpack-float:5,10", "bitpack-float:8,10", "changetype:Pos.x=f64:aosoa:2",
           "split:Pos,Mass:aosoa:4:bytesplit:soa-sb", "field-access-count(soa-mb)", "heatmap:64(aos-packed)",
           "heatmap:3(field-access-count(bytesplit:aosoa:2))"]


def lib():
    from paper_2302_08251_b200 import _lib
    return _lib.lib()


def test_library_exports_every_header_symbol():
    L = lib()
    hdr = open(os.path.join(ROOT, "include", "lamina_b200.h")).read()
    names = set(re.findall(r"\b(lam_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) > 30
    missing = [n for n in sorted(names) if not hasattr(L, n)]
    assert not missing, missing
    from paper_2302_08251_b200 import _lib
    assert set(_lib.EXPORTED) <= names


@pytest.mark.parametrize("schema", [R32, MIXED])
@pytest.mark.parametrize("layout", LAYOUTS)
def test_layout_metadata_matches_oracle(schema, layout):
    from paper_2302_08251_b200 import lamina as L
    for n in (1, 7, 1000):
        ext = f"i32:[{n}]"
        try:
            m = O.make(schema, ext, layout)
        except Exception as e:
            with pytest.raises(L.LaminaError):
                L.Layout(schema, ext, layout)
            return
        g = L.Layout(schema, ext, layout)
        assert g.name == m.name()
        assert g.blob_sizes == m.blob_sizes()
        assert g.element_count == n
        s = O.Schema.parse(schema)
        assert g.leaf_count == len(s.leaves)
        for f, l in enumerate(s.leaves):
            assert g.leaf(f) == (l.type, l.size, l.offset_packed)
            assert g.leaf_path(f) == l.path
            assert g.is_computed(f) == m.is_computed(f)
            if isinstance(m, O.Physical):
                nr, off = m.offsets(f)
                for i in {0, n // 2, n - 1}:
                    assert g.physical_offset(i, f) == (nr, int(off[i]))
        assert g.is_fully_physical == m.is_fully_physical()
        assert g.has_mutable_state == m.has_mutable_state()
        assert g.shard_unit >= 1
        if isinstance(m, O.Heatmap):
            assert [g.heatmap_blocks(k) for k in range(g.blob_count)] == [b.size for b in m.blocks]


def test_layout_metadata_matches_reference(ref):
    from paper_2302_08251_b200 import lamina as L
    for schema in (R32, MIXED, "Record{v:u32,w:i32}"):
        for layout in LAYOUTS + ["bitpack-int:7", "bitpack-int:33", "aosoa:0", "changetype:i32=f32", "bogus"]:
            if layout.startswith(("field-access", "heatmap")):
                continue
            try:
                r = ref.layout_info(schema, "i64:[77]", layout)
            except ref.RefError as e:
                with pytest.raises(L.LaminaError) as ei:
                    L.Layout(schema, "i64:[77]", layout)
                assert str(ei.value) == str(e), (layout, str(ei.value), str(e))
                continue
            g = L.Layout(schema, "i64:[77]", layout)
            assert (g.name, g.blob_sizes) == (r["name"], r["blob_sizes"])


def test_error_types_mirror_reference():
    from paper_2302_08251_b200 import lamina as L
    with pytest.raises(L.InvalidArgument, match="unknown layout"):
        L.Layout(R32, "i32:[4]", "nope")
    with pytest.raises(L.InvalidArgument, match="lane count must be >= 1"):
        L.Layout(R32, "i32:[4]", "aosoa:0")
    with pytest.raises(L.InvalidArgument, match="bitpack-int requires integer leaves"):
        L.Layout(R32, "i32:[4]", "bitpack-int:3")
    with pytest.raises(L.InvalidArgument, match="unsupported type change"):
        L.Layout("Record{v:i32}", "i32:[4]", "changetype:i32=u32")
    with pytest.raises(L.IndexTypeOverflow, match="index type overflow"):
        L.Layout(R32, "i16:[40000]", "aos-packed")
    with pytest.raises(L.InvalidArgument, match="one mapping requires a unit array extent"):
        L.Layout(R32, "i32:[2]", "one")
    g = L.Layout(R32, "i32:[4]", "bytesplit:soa-mb")
    with pytest.raises(L.LogicError, match="computed leaf has no physical offset"):
        g.physical_offset(0, 0)
    with pytest.raises(L.OutOfRange, match="index out of range"):
        L.Layout(R32, "i32:[4]", "aos-packed").physical_offset(4, 0)


def test_dynamic_extents():
    from paper_2302_08251_b200 import lamina as L
    g = L.Layout(R32, "i64:[3,dyn]", "aosoa:4", dyn=[5])
    assert g.element_count == 15 and g.extents == "i64:[3,dyn]"
    with pytest.raises(L.InvalidArgument, match="arity error"):
        L.Layout(R32, "i64:[3,dyn]", "aos-packed")


def test_golden_fixtures_present():
    idx = os.path.join(ROOT, "tests", "golden", "index.json")
    assert os.path.exists(idx)


# ---- view dump sidecar (core/src/view_io.cpp), fixtures written by the reference ---------------
DUMP_DIR = os.path.join(ROOT, "tests", "golden", "view_dump")


def _dump_cases():
    import json
    with open(os.path.join(DUMP_DIR, "index.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _dump_cases(), ids=lambda c: c["name"])
def test_dump_meta_matches_reference_sidecar(case):
    from paper_2302_08251_b200 import lamina as L
    lay = L.Layout(case["schema"], case["extents"], case["layout"], dyn=case["dyn"])
    with open(os.path.join(DUMP_DIR, case["name"] + ".meta")) as f:
        assert lay.dump_meta() == f.read()


def _damaged_dump(tmp_path, edit_meta=None, truncate=None, drop_blob=False):
    """A copy of the io_soamb fixture, damaged like test_view_io.cpp:95-140."""
    import shutil
    stem = tmp_path / "dump"
    for nr in range(4):
        shutil.copy(os.path.join(DUMP_DIR, f"io_soamb.blob{nr}.bin"), f"{stem}.blob{nr}.bin")
    with open(os.path.join(DUMP_DIR, "io_soamb.meta")) as f:
        meta = f.read()
    if edit_meta:
        meta = edit_meta(meta)
    with open(f"{stem}.meta", "w") as f:
        f.write(meta)
    if truncate is not None:
        os.truncate(f"{stem}.blob0.bin", truncate)
    if drop_blob:
        os.remove(f"{stem}.blob0.bin")
    return str(stem)


@pytest.mark.parametrize("damage,msg", [
    (dict(truncate=8), "truncated"),
    (dict(drop_blob=True), "cannot read"),
    (dict(edit_meta=lambda m: m.replace("blob0-size=48", "blob0-size=16")), "blob size mismatch"),
    (dict(edit_meta=lambda m: m.replace("blobs=4", "blobs=3")), "blob count mismatch"),
    (dict(edit_meta=lambda m: "schema=Record{x:f64}\n"), "missing field"),
    (dict(edit_meta=lambda m: m + "garbage\n"), "malformed sidecar line"),
])
def test_restore_rejects_damaged_dumps(tmp_path, damage, msg):
    """readViewDump's checks run before any device allocation, so they are testable here."""
    from paper_2302_08251_b200 import lamina as L
    stem = _damaged_dump(tmp_path, **damage)
    with pytest.raises(L.ReferenceRuntimeError, match=msg):
        L.read_view_dump(stem)


def test_restore_missing_dump(tmp_path):
    from paper_2302_08251_b200 import lamina as L
    with pytest.raises(L.ReferenceRuntimeError, match="cannot read"):
        L.read_view_dump(str(tmp_path / "absent"))


# ---- Mapping::contiguousRun vs the compiled reference ---------------------------------------
@pytest.mark.parametrize("layout", ["aos-packed", "soa-sb", "soa-mb", "aosoa:8", "aosoa:3", "split:Pos:soa-mb:aos-packed",
                                    "changetype:f32=f64:soa-mb", "changetype:f32=f32:aosoa:4", "bytesplit:soa-mb",
                                    "bitpack-float:8,23", "soa-mb+fac", "aos-packed+heat", "null"])
@pytest.mark.parametrize("schema", ["R32", "ONE"])
def test_contiguous_run_matches_reference(layout, schema, ref):
    from paper_2302_08251_b200 import lamina as L
    sch = R32 if schema == "R32" else "Record{v:f32}"
    ext = "i32:[37]"
    wrap = 1 if layout.endswith("+fac") else (2 if layout.endswith("+heat") else 0)
    layout = layout.split("+")[0]
    if schema == "ONE" and "Pos" in layout:
        pytest.skip("split selects a field of R32")
    lay = L.Layout(sch, ext, layout, wrap=wrap, granularity=8)
    nl = lay.leaf_count
    for linear in (0, 1, 5, 7, 8, 30, 36):
        for f in range(nl):
            for n in (0, 1, 2, 3, 8, 37 - linear):
                want = ref.contiguous_run(sch, ext, layout, linear, f, n, wrap=wrap, gran=8)
                assert lay.contiguous_run(linear, f, n) == want, (layout, linear, f, n)


@pytest.mark.parametrize("extents,dyn", [("i32:[16]", ()), ("i64:[dyn]", (16,)), ("u16:[4,dyn]", (5,)),
                                         ("i64:[dyn,dyn]", (3, 7))])
@pytest.mark.parametrize("layout,wrap", [("aos-packed", 0), ("soa-mb", 0), ("aosoa:4", 0), ("bitpack-float:5,10", 0),
                                         ("split:Pos:soa-mb:aos-packed", 0), ("changetype:f32=f64:bytesplit:soa-sb", 0),
                                         ("soa-sb", 1), ("aos-packed", 2), ("aosoa:2", 3)])
def test_state_accounting_matches_reference(ref, extents, dyn, layout, wrap):
    """isFullyStatic / runtimeStateBytes of the lowered layout equal the reference's
    (extents.hpp:127-143, mapping.hpp:145-148, wrappers instrument.cpp:79-82,197-200)."""
    from paper_2302_08251_b200 import lamina as L
    fs, rs, _, _, _ = ref.state_info(R32, extents, layout, dyn, wrap, 5)
    lay = L.Layout(R32, extents, layout, dyn=dyn, wrap=wrap, granularity=5)
    assert (lay.is_fully_static, lay.runtime_state_bytes) == (fs, rs)
