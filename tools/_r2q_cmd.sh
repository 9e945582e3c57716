O=gpurun_out/r2q
mkdir -p $O
LAMB_NB_EXACT=1 timeout 600 python tools/nb_shard_time.py > $O/shard_split.log 2>&1
LAMB_NB_EXACT=0 timeout 600 python tools/nb_shard_time.py > $O/shard_old.log 2>&1
timeout 900 python -m pytest tests/test_gpu_nbody.py tests/test_gpu_scale.py -x -q -k "nbody or c4" > $O/nb_tests.log 2>&1
