O=gpurun_out/r2bh
mkdir -p $O
LAMB_JIT=0 timeout 1500 python tools/sweep_pairs.py > $O/sweep_nojit.log 2>&1
