O=gpurun_out/r2ah
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_jit.py -q -x > $O/jit_tests.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest.log 2>&1
timeout 600 python tools/jit_pairs.py > $O/jit_pairs.log 2>&1
rm -f gpurun_out/jit_src.cu
