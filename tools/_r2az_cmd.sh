O=gpurun_out/r2az
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_copy.py tests/test_gpu_guard.py -q -x > $O/tests.log 2>&1
timeout 900 python tools/trace_pairs.py > $O/trace.log 2>&1
