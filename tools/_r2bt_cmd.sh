O=gpurun_out/r2bt
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_copy.py tests/test_gpu_guard.py tests/test_gpu_scale.py -q -x -k "not c3 and not c4 and not c5" tests/test_gpu_bench.py > $O/tests.log 2>&1
for i in 1 2; do timeout 900 python bench.py > $O/bench_$i.log 2>&1; done
