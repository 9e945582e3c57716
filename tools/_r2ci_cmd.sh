O=gpurun_out/r2ci
mkdir -p $O
timeout 900 python tools/planes_cmp.py > $O/planes.log 2>&1
