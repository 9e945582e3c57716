O=gpurun_out/r2b
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_scale.py -x -q --durations=0 > $O/scale.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref.log 2>&1
