"""GPU parity for the n-body kernels (tools/nbody) over every mapping.

EXACT mode must be bit-identical to the reference (same positions, same checksum text);
FAST mode (FMA + rsqrt, reassociated) must stay within a stated tolerance:
    |pos_fast - pos_ref| <= 2e-6 * max(1, |pos_ref|)   after 5 steps at n <= 4096.
"""
import json
import os

import numpy as np
import pytest

from conftest import ROOT
from oracle import lamina_oracle as O

pytestmark = pytest.mark.gpu

LAYOUTS = ["aos-packed", "aos-aligned", "soa-sb", "soa-mb", "aosoa:8", "aosoa:32", "aosoa:3", "bytesplit:soa-mb",
           "bitpack-float:8,23", "split:Pos:soa-mb:aosoa:4"]
FAST_TOL = 2e-6


def schema(t):
    return f"Record{{Pos:Record{{x:{t},y:{t},z:{t}}},Vel:Record{{x:{t},y:{t},z:{t}}},Mass:{t}}}"


def run_gpu(layout, n, steps, f64=False, mode=0, seed=42):
    from paper_2302_08251_b200 import lamina as L
    v = L.View(L.Layout(schema("f64" if f64 else "f32"), f"i64:[{n}]", layout))
    v.nbody_init(seed)
    for _ in range(steps):
        v.nbody_update(mode)
        v.nbody_move()
    return v


@pytest.mark.parametrize("layout", LAYOUTS)
def test_exact_matches_oracle(layout):
    n, steps = 512, 3
    pos, vel, mass, cs = O.nbody_run(n, steps, seed=42, dtype=np.float32)
    v = run_gpu(layout, n, steps)
    assert v.nbody_checksum() == cs
    vals = v.read_values(np.repeat(np.arange(n), 7), np.tile(np.arange(7), n)).reshape(n, 7)
    got = vals.astype(np.uint32).view(np.float32)
    assert np.array_equal(got[:, :3].view(np.uint32), pos.view(np.uint32))
    assert np.array_equal(got[:, 3:6].view(np.uint32), vel.view(np.uint32))


@pytest.mark.parametrize("case", [c for c in json.load(open(os.path.join(ROOT, "tests", "golden", "index.json")))
                                  if c["file"].startswith("nbody_")], ids=lambda c: c["file"])
def test_exact_matches_reference_fixture(case):
    z = np.load(os.path.join(ROOT, "tests", "golden", case["file"]))
    v = run_gpu(case["layout"], case["n"], case["steps"], f64=case["f64"])
    assert v.nbody_checksum() == float(z["checksum"])
    for k, b in enumerate(v.download_all()):
        assert np.array_equal(b, z[f"b{k}"])


def test_exact_f64():
    n, steps = 256, 2
    _, _, _, cs = O.nbody_run(n, steps, seed=7, dtype=np.float64)
    assert run_gpu("soa-mb", n, steps, f64=True, seed=7).nbody_checksum() == cs


@pytest.mark.parametrize("layout", ["aos-packed", "soa-mb", "aosoa:32"])
def test_fast_within_tolerance(layout):
    n, steps = 4096, 5
    pos, _, _, _ = O.nbody_run(n, steps, seed=42, dtype=np.float64)
    v = run_gpu(layout, n, steps, mode=1)
    got = v.read_values(np.repeat(np.arange(n), 3), np.tile(np.arange(3), n)).reshape(n, 3)
    got = got.astype(np.uint32).view(np.float32).astype(np.float64)
    err = np.abs(got - pos) / np.maximum(1.0, np.abs(pos))
    assert err.max() <= FAST_TOL, err.max()


def test_sharded_update_equals_whole():
    """i-range sharding (the multi-GPU decomposition) is bit-identical to one launch."""
    from paper_2302_08251_b200 import lamina as L
    n = 1000
    a = run_gpu("aosoa:8", n, 0)
    b = run_gpu("aosoa:8", n, 0)
    a.nbody_update(0)
    for lo, hi in [(0, 256), (256, 600), (600, 1000)]:
        b.nbody_update(0, lo, hi)
    for x, y in zip(a.download_all(), b.download_all()):
        assert np.array_equal(x, y)


# ---- instrumented n-body: the device runner vs the reference runner's reports ------------------
TRACE_DIR = os.path.join(ROOT, "tests", "golden", "nbody_trace")


def _trace_cases():
    with open(os.path.join(TRACE_DIR, "index.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _trace_cases(), ids=lambda c: c["dir"])
def test_instrumented_runner_matches_reference_reports(case, tmp_path, capsys):
    from paper_2302_08251_b200 import nbody
    cfg = nbody.BenchConfig(layout=case["layout"], n=case["n"], steps=case["steps"],
                            precision="f64" if case["f64"] else "f32", seed=42, trace_fields=case["trace"],
                            heatmap_granularity=case["gran"], report_dir=str(tmp_path))
    assert nbody.run_benchmark(cfg) == 0
    out = capsys.readouterr().out.strip().split("\n")
    d = os.path.join(TRACE_DIR, case["dir"])
    with open(os.path.join(d, "stdout.csv")) as f:
        want = f.read().strip().split("\n")
    # same header, same layout/phase/width, same checksum text (exact mode is bit-identical)
    assert out[0] == want[0]
    for a, b in zip(out[1:], want[1:]):
        ra, rb = a.split(","), b.split(",")
        assert ra[:3] == rb[:3] and ra[-1] == rb[-1], (a, b)
    names = (["fields_update.csv", "fields_move.csv"] if case["trace"] else []) + \
        (["heatmap_update.csv", "heatmap_move.csv"] if case["gran"] else [])
    for name in names:
        with open(os.path.join(d, name)) as f, open(tmp_path / name) as g:
            assert g.read() == f.read(), name


def test_instrumented_sharded_update_counts():
    """Counts of an update over two i-shards add up to the whole-range update."""
    from paper_2302_08251_b200 import lamina as L
    n = 96
    lay = L.Layout(schema("f32"), f"i64:[{n}]", "aosoa:8", wrap=L.WRAP_FIELD_ACCESS_COUNT | L.WRAP_HEATMAP,
                   granularity=16)
    a, b = L.View(lay), L.View(lay)
    for v in (a, b):
        v.nbody_init(42)
        v.reset_counters()
    a.nbody_update(0)
    b.nbody_update(0, 0, 40)
    b.nbody_update(0, 40, n)
    assert all(np.array_equal(x, y) for x, y in zip(a.counters(), b.counters()))
    assert np.array_equal(a.heatmap(0), b.heatmap(0))
    assert a.nbody_checksum() == b.nbody_checksum()


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("layout", ["aos-packed", "soa-mb", "aosoa:8", "bytesplit:soa-mb"])
def test_update_from_sources_equals_single_view(layout, mode):
    """The fused multi-GPU step's kernel path: j read from several views (here on one GPU)."""
    from paper_2302_08251_b200 import lamina as L
    n = 3000
    lay = L.Layout(schema("f32"), f"i64:[{n}]", layout)
    a, b, c = L.View(lay), L.View(lay), L.View(lay)
    for v in (a, b, c):
        v.nbody_init(42)
    cuts = [0, 1000, 2000, n]
    a.nbody_update(mode)
    b.nbody_update_from([(c if k % 2 else b, cuts[k], cuts[k + 1]) for k in range(3)], mode)
    if mode == 0:
        assert all(np.array_equal(x, y) for x, y in zip(a.download_all(), b.download_all()))
    else:
        # segment sums reassociate: velocities agree to FP32 rounding of their magnitude
        m = O.make(schema("f32"), f"i64:[{n}]", layout)
        fx = O.read_all(m, a.download_all()).astype(np.uint32).view(np.float32).astype(np.float64)
        fy = O.read_all(m, b.download_all()).astype(np.uint32).view(np.float32).astype(np.float64)
        assert np.max(np.abs(fx - fy)) <= 1e-5 * np.max(np.abs(fx))


def test_ipc_handle_exports():
    from paper_2302_08251_b200 import lamina as L
    v = L.View(L.Layout(schema("f32"), "i64:[64]", "soa-mb"))
    h = L.ipc_handle(v.blob_ptr(0))
    assert len(h) == 64 and any(h)


def test_nbody_step_is_update_then_move():
    from paper_2302_08251_b200 import lamina as L
    lay = L.Layout(schema("f32"), "i64:[700]", "aosoa:8")
    a, b = L.View(lay), L.View(lay)
    for v in (a, b):
        v.nbody_init(7)
    a.nbody_update(0)
    a.nbody_move()
    b.nbody_step(0)
    assert all(np.array_equal(x, y) for x, y in zip(a.download_all(), b.download_all()))


@pytest.mark.parametrize("layout", ["soa-mb", "aosoa:8"])
def test_fused_p2p_transport_two_processes(layout):
    """nbody_distributed(transport="p2p"): two processes map each other's shards with CUDA IPC
    (here on one GPU) and update through lam_nbody_update_multi; exact mode == single view."""
    import subprocess
    import sys
    env = dict(os.environ)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29541", "tools/p2p_check.py", layout, "3000",
                        "3"], cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "OK" in r.stdout, r.stdout + r.stderr[-2000:]


# ---- hand-written baselines (steps.hpp:124-230): separate kernels, no mapping -----------------
@pytest.mark.parametrize("kind", ["manual-aos", "manual-soa"])
@pytest.mark.parametrize("f64", [False, True], ids=["f32", "f64"])
def test_manual_baseline_checksum_equals_library(kind, f64):
    """acceptance.cpp:744-766: the hand-written baselines' checksum equals the library's
    (exact mode: both bit-identical to the reference)."""
    from paper_2302_08251_b200 import lamina as L
    n, steps = 1024, 5
    m = L.ManualNbody(kind, n, f64=f64, seed=42)
    for _ in range(steps):
        m.update(L.NBODY_EXACT)
        m.move()
    lib_view = run_gpu("aos-packed" if kind == "manual-aos" else "soa-mb", n, steps, f64=f64)
    _, _, _, cs = O.nbody_run(n, steps, seed=42, dtype=np.float64 if f64 else np.float32)
    assert m.checksum() == lib_view.nbody_checksum() == cs


@pytest.mark.parametrize("kind", ["manual-aos", "manual-soa"])
def test_manual_baseline_fast_within_tolerance(kind):
    from paper_2302_08251_b200 import lamina as L
    n, steps = 4096, 5
    m = L.ManualNbody(kind, n, seed=42)
    for _ in range(steps):
        m.update(L.NBODY_FAST)
        m.move()
    _, _, _, cs = O.nbody_run(n, steps, seed=42, dtype=np.float64)
    assert abs(m.checksum() - cs) <= FAST_TOL * abs(cs)


def test_manual_runner_csv(capsys):
    """runManual's CSV rows (runner.cpp:88-103) with the library layout's checksum text."""
    from paper_2302_08251_b200.nbody import BenchConfig, run_benchmark
    outs = {}
    for lay in ("manual-soa", "soa-mb"):
        assert run_benchmark(BenchConfig(layout=lay, n=512, steps=2, precision="f32")) == 0
        rows = capsys.readouterr().out.strip().splitlines()
        assert rows[0] == "layout,phase,simd_width,seconds_per_step,checksum"
        assert [r.split(",")[:3] for r in rows[1:]] == [[lay, "update", "1"], [lay, "move", "1"]]
        outs[lay] = rows[1].split(",")[-1]
    assert outs["manual-soa"] == outs["soa-mb"]
    assert run_benchmark(BenchConfig(layout="manual-aos", n=64, steps=1, simd_width=2)) == 2


@pytest.mark.parametrize("layout,mode", [("soa-mb", 0), ("aosoa:8", 0), ("aos-packed", 1)])
def test_allgather_transport_two_processes(layout, mode):
    """nbody_distributed(transport="allgather"): the positions-only exchange (one all-gather of
    12 B/particle per step, Mass once) with the real kernels in two processes (here sharing one
    GPU, gloo) equals the single-view run: bit-identical in exact mode."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29543", "tools/allgather_check.py", layout,
                        "4096", "3", str(mode)], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "OK" in r.stdout, r.stdout + r.stderr[-2000:]
