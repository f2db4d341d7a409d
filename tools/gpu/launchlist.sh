# ncu launch list of the default bench command (per-kernel durations, cold caches, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 70000 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-roofline-2048 --no-paper-config > gpurun_out/r2_ll.log 2>&1
echo rc=$? >> gpurun_out/r2_ll.log
