O=gpurun_out/r2bm
mkdir -p $O
R32="Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"
MB="Record{a:i8,b:u16,c:i32,d:u64,e:f32,f:f64,g:bool,h:Record{x:i16,y:f32[3]}}"
M4="Record{a:f64,b:u16,c:i8,d:f32}"
i=0
for args in "s|$MB|aos-packed|soa-mb" "d|$M4|soa-mb|aos-packed" "d|$R32|aos-packed|aosoa:3" "d|$R32|bytesplit:soa-mb|soa-mb" "d|$MB|aos-packed|changetype:f64=f32,i8=i64,u16=u8:aosoa:2"; do
  i=$((i+1))
  IFS='|' read -r mode sch a b <<< "$args"
  LAMB_JIT_STAGE=$mode timeout 300 ncu --set full --clock-control none -k lamjit_copy -s 2 -c 1 -o $O/j$i python tools/jit_one.py "$sch" "$a" "$b" > $O/ncu$i.log 2>&1
  ncu -i $O/j$i.ncu-rep --page raw --csv > $O/j${i}_raw.csv 2>/dev/null
  ncu -i $O/j$i.ncu-rep --page details --csv > $O/j${i}_details.csv 2>/dev/null
  rm -f $O/j$i.ncu-rep
  echo "$i $mode $a -> $b" >> $O/index.txt
done
