O=gpurun_out/r2cm
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_jit.py -q -x > $O/tests.log 2>&1
timeout 1800 python tools/sweep_pairs.py > $O/sweep.log 2>&1
