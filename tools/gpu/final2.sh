python -m pytest tests -m gpu -q --durations=8 > gpurun_out/f2_tests.log 2>&1; echo rc=$? >> gpurun_out/f2_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1
python bench.py > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 70000 --csv --log-file gpurun_out/f2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-roofline-2048 --no-paper-config --no-configs > gpurun_out/f2_ll.log 2>&1
