python tools/garbage_check.py tests/golden/fit_config2_s7.npz 5 > gpurun_out/garbage.txt 2>&1
python tools/garbage_check.py tests/golden/fit_config2_s3.npz 3 >> gpurun_out/garbage.txt 2>&1
python tools/garbage_check.py tests/golden/fit_config2_fp64_s1.npz 2 >> gpurun_out/garbage.txt 2>&1
