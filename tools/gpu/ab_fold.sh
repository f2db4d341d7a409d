# A/B: end-of-iteration bookkeeping folded into k_adam (default) vs a separate k_advance (SAD_NO_FOLD=1)
python -m pytest tests/test_fit_configs.py tests/test_gpu_parity.py tests/test_reduction_paths.py -m gpu -q -x > gpurun_out/fold_tests.log 2>&1; echo rc=$? >> gpurun_out/fold_tests.log
for i in 1 2 3; do
  SAD_NO_FOLD=1 python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so
  python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so
done > gpurun_out/ab_fold.txt 2>&1
