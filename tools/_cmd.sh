nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits 2>&1 | head -3
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv,noheader,nounits 2>&1 | head -2
python tools/prof_copy.py > gpurun_out/p5.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu5a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_vec_transpose -s 2 -c 1 -o gpurun_out/prof_vec python tools/prof_copy.py > gpurun_out/ncu5.log 2>&1
cat gpurun_out/p5.log; tail -2 gpurun_out/ncu5.log; wc -l gpurun_out/launches_c2.csv
