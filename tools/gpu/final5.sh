ncu --metrics gpu__time_duration.sum --clock-control none -c 70000 --csv --log-file gpurun_out/f5_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-roofline-2048 --no-paper-config --no-configs > gpurun_out/f5_ll.log 2>&1
python tools/launch_list.py gpurun_out/f5_launches.csv "ncu launch list (gpu__time_duration, cold, serialised) of: python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-roofline-2048 --no-paper-config --no-configs (round-2 final code)" > gpurun_out/f5_ll.txt 2>&1
rm -f gpurun_out/f5_launches.csv
