O=gpurun_out/r2d
mkdir -p $O
timeout 600 python tools/nb_alt_sweep.py > $O/alt.log 2>&1
timeout 600 python -m pytest tests/test_gpu_nbody.py -x -q -k "allgather or fast or manual" > $O/nb_tests.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e > $O/bench.log 2>&1
