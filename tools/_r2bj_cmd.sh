O=gpurun_out/r2bj
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_copy.py tests/test_gpu_codec.py tests/test_gpu_guard.py -q -x > $O/tests.log 2>&1
timeout 600 python tools/more_pairs.py > $O/more_pairs.log 2>&1
timeout 1500 python tools/sweep_pairs.py > $O/sweep.log 2>&1
