O=gpurun_out/r2bl
mkdir -p $O
NB_SHAPES="0 3 4 5 6 0" timeout 900 python tools/nb_exact_sweep.py > $O/exact_sweep.log 2>&1
