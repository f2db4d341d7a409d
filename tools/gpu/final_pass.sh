# round-2 measurement pass: GPU suite, bench lines (config 2 N=1, config 3, config 4 at N=1, config 5 single GPU and
# row-strip path at world 1), reference arm, launch list of the bench command
python -m pytest tests -m gpu -q > gpurun_out/f_tests.log 2>&1; echo rc=$? >> gpurun_out/f_tests.log
python __graft_entry__.py smoke > gpurun_out/f_smoke.log 2>&1 || true
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
python bench.py --impl reference > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
python bench.py --mode config3 --steps 2 > gpurun_out/f_config3.json 2> gpurun_out/f_config3.err
python bench.py --images-per-gpu 3 --steps 2 --no-cpu-baseline --no-roofline-2048 --no-paper-config > gpurun_out/f_config4.json 2> gpurun_out/f_config4.err
python bench.py --mode config5 > gpurun_out/f_config5.json 2> gpurun_out/f_config5.err
python bench.py --mode config5 --c5-strips > gpurun_out/f_config5_strips.json 2> gpurun_out/f_config5_strips.err
