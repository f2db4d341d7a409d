# ncu --set full at the config-5 scale (8192^2, 2 BPP, state after 30 iterations): fwd+bwd, warm pass, render
K="python tools/kbench.py --width 8192 --height 8192 --iters 30"
$K --kernel fwd_bwd,propagate_warm,render --reps 5 > gpurun_out/r2_kb8192.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_backward2 -s 32 -c 1 -f -o gpurun_out/r2_bwd8192 $K --kernel fwd_bwd --reps 2 > gpurun_out/r2_ncu8192.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_render -c 1 -f -o gpurun_out/r2_render8192 $K --kernel render --reps 2 >> gpurun_out/r2_ncu8192.log 2>&1
