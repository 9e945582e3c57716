O=gpurun_out/r2cz
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_copy.py -q -x -k "bitpack" > $O/tests.log 2>&1
timeout 900 python tools/repack_cmp.py > $O/repack.log 2>&1
