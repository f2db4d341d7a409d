python -m pytest tests -m gpu -q > gpurun_out/f4_tests.log 2>&1; echo rc=$? >> gpurun_out/f4_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo rc=$? >> gpurun_out/f4_smoke.log
python bench.py > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f4_ref.json 2> gpurun_out/f4_ref.err
