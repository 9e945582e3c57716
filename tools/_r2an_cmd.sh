O=gpurun_out/r2an
mkdir -p $O
M4="Record{a:f64,b:u16,c:i8,d:f32}"
MB="Record{a:i8,b:u16,c:i32,d:u64,e:f32,f:f64,g:bool,h:Record{x:i16,y:f32[3]}}"
i=0
for args in "$M4 aos-packed soa-mb" "$M4 soa-mb aos-packed" "$M4 aosoa:8 aos-aligned" "$MB aos-packed soa-mb" "$MB soa-mb aos-packed"; do
  i=$((i+1))
  set -- $args
  timeout 300 ncu --set full --clock-control none -k lamjit_copy -s 1 -c 1 -o $O/jit$i python tools/jit_one.py "$1" $2 $3 > $O/ncu$i.log 2>&1
  ncu -i $O/jit$i.ncu-rep --page raw --csv > $O/jit${i}_raw.csv 2>/dev/null
  ncu -i $O/jit$i.ncu-rep --page details --csv > $O/jit${i}_details.csv 2>/dev/null
  rm -f $O/jit$i.ncu-rep
done
