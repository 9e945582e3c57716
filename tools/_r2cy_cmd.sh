O=gpurun_out/r2cy
mkdir -p $O
timeout 1800 python tools/sweep_pairs.py > $O/sweep.log 2>&1
