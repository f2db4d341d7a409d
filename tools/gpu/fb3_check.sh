# new fused fwd+bwd (k_fwdbwd3): parity tests, then A/B timing against k_backward2
python -m pytest tests/test_gpu_parity.py tests/test_reduction_paths.py tests/test_fit_configs.py -m gpu -q -x -k "not golden_set" > gpurun_out/fb3_tests.log 2>&1; echo rc=$? >> gpurun_out/fb3_tests.log
K="python tools/kbench.py"
$K --kernel fwd_bwd --reps 50 > gpurun_out/fb3_kb.txt 2>&1
SAD_BWD2=1 $K --kernel fwd_bwd --reps 50 >> gpurun_out/fb3_kb.txt 2>&1
$K --kernel fwd_bwd --reps 20 --width 2048 --height 2048 --n-sites 100000 --iters 100 >> gpurun_out/fb3_kb.txt 2>&1
SAD_BWD2=1 $K --kernel fwd_bwd --reps 20 --width 2048 --height 2048 --n-sites 100000 --iters 100 >> gpurun_out/fb3_kb.txt 2>&1
python tools/fit_time.py > gpurun_out/fb3_fit.txt 2>&1
SAD_BWD2=1 python tools/fit_time.py >> gpurun_out/fb3_fit.txt 2>&1
