K="python tools/kbench.py"
ncu --set full --clock-control none --import-source on -k regex:k_fwdbwd3 -s 3 -c 1 -f -o gpurun_out/fb3_768 $K --kernel fwd_bwd --reps 5 > gpurun_out/fb3_ncu.log 2>&1
