set -x
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
nproc > $O/nproc.txt; free -g >> $O/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1
timeout 600 python tools/more_pairs.py > $O/more_pairs.log 2>&1
NCU="ncu --set full --clock-control none --import-source on -f"
NBODY_MODE=0 timeout 600 $NCU -k regex:k_nbody_update -c 1 -o $O/nbody_exact python tools/nbody_prof.py > $O/ncu1.log 2>&1
timeout 600 $NCU -k regex:k_warp_tile -c 1 -o $O/warp_tile_split python tools/prof_copy.py --src aos-packed --dst split:Pos:soa-mb:aos-packed --reps 1 > $O/ncu2.log 2>&1
timeout 600 $NCU -k regex:k_generic -c 1 -o $O/generic_u16 python tools/prof_copy.py --schema "Record{v:u16,w:u16}" --src soa-mb --dst bitpack-int:5 --reps 1 > $O/ncu3.log 2>&1
timeout 600 $NCU -k regex:k_nbody_fast -c 1 -o $O/nbody_fast python tools/nbody_prof.py > $O/ncu4.log 2>&1
