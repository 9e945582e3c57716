O=gpurun_out/r2w
mkdir -p $O
timeout 900 python tools/nb_alt_sweep.py > $O/alt.log 2>&1
