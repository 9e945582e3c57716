"""bench.py contract on a small problem: the JSON line's keys, and the multi-rank path (two ranks
sharing one GPU over gloo; the driver's scaling runs use NCCL with one GPU per rank)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "gpu_launches", "clocks", "roofline"}


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_bench_single_gpu_small():
    r = subprocess.run([sys.executable, "bench.py", "--records", str(1 << 20), "--steps", "2", "--warmup", "3",
                        "--no-e2e", "--no-cpu", "--no-extra"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["peak"] > 0


def test_bench_two_ranks_gloo():
    env = dict(os.environ, LAMB_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
                        "--records", str(1 << 20), "--steps", "2", "--warmup", "3", "--no-cpu",
                        "--c4-particles", "8192", "--c5-records", str(1 << 22)],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["e2e"]["h2d_bytes_per_step"] > 0
    # the paths that shard / communicate: n-body with the positions-only exchange, C5 sharded
    assert d["c4_strong"]["exact"]["interactions_per_s"] > 0 and d["c4_strong"]["fast"]["exchange_bytes_per_step"] > 0
    assert d["c5_sharded"]["counters_ok"] and d["c5_sharded"]["records_total"] == 1 << 22
