python -m pytest tests -m gpu -q -k "not golden_set" --durations=10 > gpurun_out/sb_tests.log 2>&1; echo rc=$? >> gpurun_out/sb_tests.log
python bench.py > gpurun_out/sb_bench.json 2> gpurun_out/sb_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/sb_ref.json 2> gpurun_out/sb_ref.err
