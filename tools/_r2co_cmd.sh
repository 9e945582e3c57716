O=gpurun_out/r2co
mkdir -p $O
R64="Record{Pos:Record{x:f64,y:f64,z:f64},Vel:Record{x:f64,y:f64,z:f64},Mass:f64}"
timeout 600 ncu --set full --clock-control none -k regex:k_rec_to_planes -s 2 -c 1 -o $O/pl python tools/prof_copy.py --schema "$R64" --src aos-packed --dst changetype:f64=f32:bytesplit:soa-mb > $O/ncu_pl.log 2>&1
ncu -i $O/pl.ncu-rep --page raw --csv > $O/pl_raw.csv 2>/dev/null
ncu -i $O/pl.ncu-rep --page details --csv > $O/pl_details.csv 2>/dev/null
rm -f $O/pl.ncu-rep
