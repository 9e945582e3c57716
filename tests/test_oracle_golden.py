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


# ---- instrumented n-body reports (runner.cpp:344-436), fixtures from the reference runner ----
TRACE_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "nbody_trace")


def _trace_cases():
    with open(os.path.join(TRACE_DIR, "index.json")) as f:
        return json.load(f)


def parse_fields_csv(text):
    rows = text.strip().split("\n")[1:]
    return [(r.split(",")[0], int(r.split(",")[1]), int(r.split(",")[2])) for r in rows]


def parse_heatmap_csv(text):
    blobs = []
    for ln in text.strip().split("\n"):
        if ln.startswith("# blob"):
            blobs.append([])
        elif not ln.startswith("blockIndex"):
            blobs[-1].append(int(ln.split(",")[2]))
    return blobs


@pytest.mark.parametrize("case", _trace_cases(), ids=lambda c: c["dir"])
def test_oracle_nbody_trace_matches_reference_runner(case):
    t = O.nbody_trace(case["layout"], case["n"], case["steps"], case["f64"], case["gran"])
    d = os.path.join(TRACE_DIR, case["dir"])
    for phase in ("update", "move"):
        r, w, blocks = t[phase]
        if case["trace"]:
            with open(os.path.join(d, f"fields_{phase}.csv")) as f:
                rows = parse_fields_csv(f.read())
            assert [(x[1], x[2]) for x in rows[:7]] == list(zip(r.tolist(), w.tolist()))
            assert rows[7] == ("TOTAL", int(r.sum()), int(w.sum()))
        if case["gran"]:
            with open(os.path.join(d, f"heatmap_{phase}.csv")) as f:
                assert parse_heatmap_csv(f.read()) == [b.tolist() for b in blocks]
