O=gpurun_out/r2bp
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_copy.py tests/test_gpu_guard.py -q -x > $O/tests.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
LAMB_VEC_SSTAGE=0 timeout 900 python bench.py > $O/bench_nosstage.log 2>&1
