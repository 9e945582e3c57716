python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --warmup 3 --suite > gpurun_out/bench_suite.json 2> gpurun_out/bench_suite.err; echo rc=$?
python tools/summarize_bench.py gpurun_out/bench_suite.json
