# ncu captures of render and the warm propagate pass at 2048^2
K="python tools/kbench.py"
ncu --set full --clock-control none --import-source on -k regex:k_render -s 3 -c 1 -f -o gpurun_out/r2b_render2048 $K --kernel render --reps 5 --width 2048 --height 2048 --n-sites 100000 --iters 100 > gpurun_out/r2b_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_prop8_queue -s 3 -c 1 -f -o gpurun_out/r2b_warm2048 $K --kernel propagate_warm --reps 5 --width 2048 --height 2048 --n-sites 100000 --iters 100 >> gpurun_out/r2b_ncu.log 2>&1
