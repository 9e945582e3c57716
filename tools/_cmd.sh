python -m pytest tests/test_gpu_nbody.py -x -q 2>&1 | tail -15
