O=gpurun_out/r2bv
mkdir -p $O
timeout 2000 python -m pytest tests -m gpu -q -x --durations=5 > $O/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python bench_suite.py > $O/bench_suite.json 2> $O/bench_suite.err
timeout 900 python bench.py > $O/bench.log 2>&1
