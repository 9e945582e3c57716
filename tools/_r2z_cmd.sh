O=gpurun_out/r2z
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $O/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref.log 2>&1
