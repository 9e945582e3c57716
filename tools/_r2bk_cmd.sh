O=gpurun_out/r2bk
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_copy.py tests/test_gpu_codec.py -q -x -k "bitpack_float or codec or patterns" > $O/tests.log 2>&1
timeout 600 python tools/more_pairs.py > $O/more_pairs.log 2>&1
LAMB_PACK_CONSTFMT=0 timeout 600 python tools/more_pairs.py > $O/more_pairs_noconst.log 2>&1
