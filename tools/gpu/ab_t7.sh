python -m pytest tests/test_gpu_parity.py tests/test_fit_configs.py tests/test_strips.py -m gpu -q -x -k "not golden_set" > gpurun_out/t7_tests.log 2>&1; echo rc=$? >> gpurun_out/t7_tests.log
K="python tools/kbench.py"
for lib in exp/libsad_t70.so paper_2604_21984_b200/libsad_b200.so exp/libsad_t70.so paper_2604_21984_b200/libsad_b200.so; do
  echo "== $lib"
  $K --lib $lib --kernel propagate_warm,propagate_flood,refresh_full --reps 50
  $K --lib $lib --kernel propagate_warm,propagate_flood --reps 20 --width 2048 --height 2048 --n-sites 100000 --iters 100
  python tools/ab_fit.py $lib
done > gpurun_out/ab_t7.txt 2>&1
