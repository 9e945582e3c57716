O=gpurun_out/r2cw
mkdir -p $O
LAMB_TRACE=1 timeout 900 python -m pytest tests/test_gpu_copy.py -q -x -k "bitpack_to_bitpack" -s > $O/trace_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_copy.py tests/test_gpu_guard.py tests/test_gpu_codec.py -q -x > $O/tests.log 2>&1
timeout 900 python tools/repack_cmp.py > $O/repack.log 2>&1
