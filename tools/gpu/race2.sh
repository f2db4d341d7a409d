python tools/flaky_check.py tests/golden/fit_config2_s7.npz 300 > gpurun_out/race_fold.txt 2>&1
SAD_NO_FOLD=1 python tools/flaky_check.py tests/golden/fit_config2_s7.npz 300 > gpurun_out/race_nofold.txt 2>&1
