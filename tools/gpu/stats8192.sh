python tools/kbench.py --kernel stats,adam,fwd_bwd,propagate_warm,refresh_full --reps 3 --width 8192 --height 8192 --iters 30 > gpurun_out/kb8192.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stats2|k_finalize|k_tables" --csv --log-file gpurun_out/stats8192.csv python tools/kbench.py --kernel stats --reps 2 --width 8192 --height 8192 --iters 30 > /dev/null 2>&1
