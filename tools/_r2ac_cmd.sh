O=gpurun_out/r2ac
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_copy.py tests/test_gpu_guard.py -x -q > $O/tests.log 2>&1
timeout 600 python tools/misc_pairs.py > $O/misc_pairs.log 2>&1
