O=gpurun_out/r2y
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -f -k regex:k_row_permute -c 1 -o $O/row_permute python tools/prof_copy.py --schema "Record{a:f64,b:u16,c:i8,d:f32}" --src aos-packed --dst soa-mb --reps 1 > $O/ncu.log 2>&1
LAMB_ROW_PERMUTE=0 timeout 600 python tools/prof_copy.py --schema "Record{a:f64,b:u16,c:i8,d:f32}" --src aos-packed --dst soa-mb --reps 4 > $O/warp_tile.log 2>&1
timeout 600 python tools/prof_copy.py --schema "Record{a:f64,b:u16,c:i8,d:f32}" --src aos-packed --dst soa-mb --reps 4 > $O/row.log 2>&1
