python -m pytest tests/test_gpu_parity.py tests/test_reduction_paths.py -m gpu -q -x > gpurun_out/fb3q_tests.log 2>&1; echo rc=$? >> gpurun_out/fb3q_tests.log
K="python tools/kbench.py"
$K --kernel fwd_bwd --reps 50 > gpurun_out/fb3q_kb.txt 2>&1
SAD_BWD2=1 $K --kernel fwd_bwd --reps 50 >> gpurun_out/fb3q_kb.txt 2>&1
$K --kernel fwd_bwd --reps 20 --width 2048 --height 2048 --n-sites 100000 --iters 100 >> gpurun_out/fb3q_kb.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fwdbwd3 -s 3 -c 1 -f -o gpurun_out/fb3q_768 $K --kernel fwd_bwd --reps 5 > gpurun_out/fb3q_ncu.log 2>&1
