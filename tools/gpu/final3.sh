python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo rc=$? >> gpurun_out/f3_smoke.log
python bench.py > gpurun_out/f3_bench.json 2> gpurun_out/f3_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f3_ref.json 2> gpurun_out/f3_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 70000 --csv --log-file gpurun_out/f3_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-roofline-2048 --no-paper-config --no-configs > gpurun_out/f3_ll.log 2>&1
python tools/launch_list.py gpurun_out/f3_launches.csv "ncu launch list (gpu__time_duration, cold, serialised) of: python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-roofline-2048 --no-paper-config --no-configs (round-2 final code)" > gpurun_out/f3_ll.txt 2>&1
rm -f gpurun_out/f3_launches.csv
