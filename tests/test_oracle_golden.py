"""The oracle reproduces the golden fixtures produced by the reference itself
(tests/golden/make_golden.py -> oracle/_ref).  CPU only; needs no /root/reference."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT
from oracle import lamina_oracle as O

GOLD = os.path.join(ROOT, "tests", "golden")
INDEX = json.load(open(os.path.join(GOLD, "index.json")))
COPIES = [c for c in INDEX if c["file"].startswith("copy_")]
NBODY = [c for c in INDEX if c["file"].startswith("nbody_")]


@pytest.mark.parametrize("case", COPIES, ids=[c["file"] for c in COPIES])
def test_copy_fixture(case):
    z = np.load(os.path.join(GOLD, case["file"]))
    ext = f"i32:[{case['n']}]"
    ms = O.make(case["schema"], ext, case["src"])
    md = O.make(case["schema"], ext, case["dst"], wrap=case["dst_wrap"], gran=case["gran"])
    sb = O.zero_blobs(ms)
    O.write_all(ms, sb, z["values"])
    for nr, b in enumerate(sb):
        assert np.array_equal(b, z[f"src{nr}"]), "View::write image differs"
    db = O.zero_blobs(md)
    O.copy_view(ms, sb, md, db)
    for nr, b in enumerate(db):
        assert np.array_equal(b, z[f"dst{nr}"]), f"dst blob {nr}"
    assert md.name() == case["dst_name"]
    if case["dst_wrap"] & 1:
        assert np.array_equal(np.concatenate([O._fac_of(md).reads, O._fac_of(md).writes]), z["dst_fac"])
    if case["dst_wrap"] & 2:
        assert np.array_equal(np.concatenate(O._heat_of(md).blocks), z["dst_heat"])


def test_minifloat_fixture():
    z = np.load(os.path.join(GOLD, "minifloat.npz"))
    for e, m in json.load(open(os.path.join(GOLD, "index.json")))[-len(NBODY) - 1]["formats"]:
        assert np.array_equal(O.float_encode(z["doubles"], e, m), z[f"enc_{e}_{m}"]), (e, m)
        got = O.float_decode(z[f"pat_{e}_{m}"], e, m)
        want = z[f"dec_{e}_{m}"]
        nan = np.isnan(want.view(np.float64))
        assert np.array_equal(np.isnan(got.view(np.float64)), nan)
        assert np.array_equal(got[~nan], want[~nan]), (e, m)
        assert np.array_equal(O.float_encode(O.f32_to_f64(z["f32"]), e, m), z[f"enc32_{e}_{m}"]), (e, m)


def test_convert_fixture():
    z = np.load(os.path.join(GOLD, "convert.npz"))
    assert np.array_equal(O.f64_to_f32(z["f64"]).astype(np.uint32), z["f64_to_f32"])
    assert np.array_equal(O.f32_to_f64(z["f32"].astype(np.uint64)), z["f32_to_f64"])


@pytest.mark.parametrize("case", NBODY, ids=[c["file"] for c in NBODY])
def test_nbody_fixture(case):
    z = np.load(os.path.join(GOLD, case["file"]))
    dt = np.float64 if case["f64"] else np.float32
    pos, vel, mass, cs = O.nbody_run(case["n"], case["steps"], seed=42, dtype=dt)
    assert cs == float(z["checksum"]), (cs, float(z["checksum"]))
    t = "f64" if case["f64"] else "f32"
    schema = f"Record{{Pos:Record{{x:{t},y:{t},z:{t}}},Vel:Record{{x:{t},y:{t},z:{t}}},Mass:{t}}}"
    m = O.make(schema, f"i64:[{case['n']}]", case["layout"])
    bl = O.zero_blobs(m)
    vals = np.concatenate([pos, vel, mass[:, None]], axis=1).astype(dt).view(
        np.uint64 if case["f64"] else np.uint32).astype(np.uint64)
    O.write_all(m, bl, vals)
    for k, b in enumerate(bl):
        assert np.array_equal(b, z[f"b{k}"])
