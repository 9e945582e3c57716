O=gpurun_out/r2k
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_copy.py -x -q > $O/copy_tests.log 2>&1
timeout 600 python tools/more_pairs.py > $O/more_pairs.log 2>&1
timeout 600 python tools/heat_pairs.py > $O/heat_pairs.log 2>&1
LAMB_HEAT_PATTERN=0 timeout 600 python tools/heat_pairs.py > $O/heat_pairs_nopattern.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --leak-check full python tools/sanitize_copies.py > $O/sanitize_memcheck.log 2>&1
timeout 1500 $CS --tool racecheck python tools/sanitize_copies.py > $O/sanitize_racecheck.log 2>&1
timeout 1200 $CS --tool synccheck python tools/sanitize_copies.py > $O/sanitize_synccheck.log 2>&1
