python tools/race_detail.py 200 > gpurun_out/race_detail.txt 2>&1
python tools/flaky_check.py tests/golden/fit_config2_s7.npz 300 exp/libsad_adam4.so > gpurun_out/race_adam4.txt 2>&1
