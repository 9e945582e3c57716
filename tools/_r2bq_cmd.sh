O=gpurun_out/r2bq
mkdir -p $O
for i in 1 2; do
timeout 900 python bench.py > $O/bench4_$i.log 2>&1
LAMB_VEC_MINB=3 timeout 900 python bench.py > $O/bench3_$i.log 2>&1
done
