O=gpurun_out/r2by
mkdir -p $O
LAMB_TRACE=1 timeout 900 python -m pytest tests/test_gpu_copy.py -q -x -k "bitpack_to_bitpack" -s > $O/trace_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_copy.py tests/test_gpu_guard.py tests/test_gpu_jit.py -q -x > $O/tests.log 2>&1
timeout 1800 python tools/sweep_pairs.py > $O/sweep.log 2>&1
