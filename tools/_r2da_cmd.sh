O=gpurun_out/r2da
mkdir -p $O
timeout 2000 python -m pytest tests -m gpu -q -x --durations=5 > $O/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 900 python bench.py --impl reference > $O/ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 1 > $O/ncu_bench.log 2>&1
