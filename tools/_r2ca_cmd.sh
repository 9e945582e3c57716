O=gpurun_out/r2ca
mkdir -p $O
timeout 900 python tools/repack_cmp.py > $O/repack.log 2>&1
timeout 900 python -m pytest tests/test_gpu_copy.py -q -x -k "bitpack" > $O/tests.log 2>&1; LAMB_REPACK=2 timeout 900 python -m pytest tests/test_gpu_copy.py -q -x -k "bitpack_to_bitpack" > $O/tests2.log 2>&1
