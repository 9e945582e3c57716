O=gpurun_out/r2v
mkdir -p $O
timeout 900 python bench_suite.py C3 > $O/c3.json 2>&1
timeout 900 python -m pytest tests/test_gpu_copy.py tests/test_gpu_codec.py -x -q > $O/tests.log 2>&1
timeout 600 python tools/more_pairs.py > $O/more_pairs.log 2>&1
timeout 600 python tools/heat_pairs.py > $O/heat_pairs.log 2>&1
