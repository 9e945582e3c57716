O=gpurun_out/r2l
mkdir -p $O
( time timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 ) > $O/bench.log 2> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extra > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -f -k regex:k_vec_transpose -c 1 -o $O/vec_transpose python tools/prof_copy.py --src aos-packed --dst soa-mb --reps 1 > $O/ncu_vec.log 2>&1
