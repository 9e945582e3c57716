O=gpurun_out/r2cu
mkdir -p $O
LAMB_JIT=0 timeout 1800 python tools/sweep_pairs.py > $O/sweep_nojit.log 2>&1
