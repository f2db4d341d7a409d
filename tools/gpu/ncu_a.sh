# ncu captures of the fwd+bwd kernel at 768x512 and 2048^2 plus kernel timings (one call: <64 MiB of reports)
K="python tools/kbench.py"
$K --kernel fwd_bwd,propagate_warm,render,propagate_flood,adam,stats,refresh_full --reps 50 > gpurun_out/r2a_kb768.txt 2>&1
$K --kernel fwd_bwd,propagate_warm,render,propagate_flood,adam,stats --reps 20 --width 2048 --height 2048 --n-sites 100000 --iters 100 > gpurun_out/r2a_kb2048.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_backward2 -s 3 -c 1 -f -o gpurun_out/r2a_bwd768 $K --kernel fwd_bwd --reps 5 > gpurun_out/r2a_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_backward2 -s 3 -c 1 -f -o gpurun_out/r2a_bwd2048 $K --kernel fwd_bwd --reps 5 --width 2048 --height 2048 --n-sites 100000 --iters 100 >> gpurun_out/r2a_ncu.log 2>&1
