# fp64 reference-order reduction: parity tests, the fp64 golden over all rows, the reference suite
python tools/fp64_golden_check.py > gpurun_out/ord64.txt 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_reduction_paths.py tests/test_reference_suite.py tests/test_fit_configs.py -m gpu -q -x -k "fp64 or Fp64 or reference_suite or config1 or backward or grad or reduction" > gpurun_out/ord64_tests.log 2>&1; echo rc=$? >> gpurun_out/ord64_tests.log
