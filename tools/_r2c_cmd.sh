O=gpurun_out/r2c
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $O/pytest.log 2>&1
timeout 300 python tools/nb_shard_time.py > $O/nb_shard.log 2>&1
timeout 600 python bench_suite.py C4 > $O/c4.json 2>&1
