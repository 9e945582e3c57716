O=gpurun_out/r2p
mkdir -p $O
timeout 600 python tools/nb_exact_sweep.py > $O/exact_sweep.log 2>&1
timeout 900 python -m pytest tests/test_gpu_nbody.py tests/test_gpu_scale.py -x -q -k "nbody or c4" > $O/nb_tests.log 2>&1
LAMB_NB_EXACT_SHAPE=2 timeout 900 python -m pytest tests/test_gpu_nbody.py tests/test_gpu_scale.py -x -q -k "exact" > $O/nb_tests_shape2.log 2>&1
