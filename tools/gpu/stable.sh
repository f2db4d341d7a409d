python tools/flaky_check.py tests/golden/fit_config2_s7.npz 300 exp/libsad_stable.so > gpurun_out/stable.txt 2>&1
python tools/ab_fit.py exp/libsad_stable.so >> gpurun_out/stable.txt 2>&1
python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so >> gpurun_out/stable.txt 2>&1
