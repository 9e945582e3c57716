O=gpurun_out/r2bf
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 1500 python tools/sweep_pairs.py > $O/sweep.log 2>&1
