python -m pytest tests/test_gpu_parity.py tests/test_reduction_paths.py tests/test_fit_configs.py tests/test_strips.py -m gpu -q -x -k "fp64 or ordered or overflow or strips or config1" > gpurun_out/oa_tests.log 2>&1; echo rc=$? >> gpurun_out/oa_tests.log
for i in 1 2; do
  FP64=1 python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so
  FP64=1 SAD_ORD_TOTALS=1 python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so
done > gpurun_out/oa.txt 2>&1
