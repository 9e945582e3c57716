python -m pytest tests/test_gpu_nbody.py tests/test_gpu_copy.py -x -q 2>&1 | tail -3
python bench.py --warmup 3 --suite > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -3 gpurun_out/bench5.err
python tools/summarize_bench.py gpurun_out/bench5.json
