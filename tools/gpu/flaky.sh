python tools/flaky_check.py tests/golden/fit_config2_s7.npz 12 > gpurun_out/flaky.txt 2>&1
echo "--- SAD_NO_FOLD=1" >> gpurun_out/flaky.txt
SAD_NO_FOLD=1 python tools/flaky_check.py tests/golden/fit_config2_s7.npz 12 >> gpurun_out/flaky.txt 2>&1
