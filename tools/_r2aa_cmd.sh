O=gpurun_out/r2aa
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on -f"
NBODY_MODE=0 timeout 600 $NCU -k regex:k_nbody_update -c 1 -o $O/nbody_exact_r2 python tools/nbody_prof.py > $O/ncu1.log 2>&1
timeout 600 $NCU -k regex:k_vec_multi -c 1 -o $O/vec_multi_split python tools/prof_copy.py --src aos-packed --dst split:Pos:soa-mb:aos-packed --reps 1 > $O/ncu2.log 2>&1
LAMB_FORCE_GENERIC=1 timeout 600 $NCU -k regex:k_generic_copy -c 1 -o $O/generic_forced python tools/prof_copy.py --src aos-packed --dst soa-mb --n 16777216 --reps 1 > $O/ncu3.log 2>&1
timeout 600 $NCU -k regex:k_packv -c 1 -o $O/packv_u16_r2 python tools/prof_copy.py --schema "Record{v:u16,w:u16}" --src soa-mb --dst bitpack-int:5 --reps 1 > $O/ncu4.log 2>&1
timeout 600 $NCU -k regex:k_unpack32 -c 1 -o $O/unpack32_int3 python tools/prof_copy.py --schema "Record{v:u32}" --src bitpack-int:3 --dst soa-mb --n 268435456 --reps 1 > $O/ncu5.log 2>&1
for f in $O/*.ncu-rep; do b=${f%.ncu-rep}; ncu -i $f --page details --csv > ${b}_details.csv 2>/dev/null; ncu -i $f --page raw --csv > ${b}_raw.csv 2>/dev/null; rm -f $f; done
timeout 600 python tools/nb_dist_vs_view.py > $O/nb_dist_vs_view.log 2>&1
