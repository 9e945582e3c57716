O=gpurun_out/r2ar
mkdir -p $O
R32="Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"
timeout 300 ncu --set full --clock-control none -k regex:k_pack32 -s 2 -c 1 -o $O/pk python tools/jit_one.py "$R32" soa-mb bitpack-float:4,3 > $O/ncu_pk.log 2>&1
ncu -i $O/pk.ncu-rep --page raw --csv > $O/pk_raw.csv 2>/dev/null
ncu -i $O/pk.ncu-rep --page details --csv > $O/pk_details.csv 2>/dev/null
ncu -i $O/pk.ncu-rep --page source --csv --print-source sass > $O/pk_sass.csv 2>/dev/null
rm -f $O/pk.ncu-rep
