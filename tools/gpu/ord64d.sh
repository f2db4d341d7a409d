python tools/fp64_golden_check.py > gpurun_out/ord64.txt 2>&1
FP64=1 python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so > gpurun_out/ab_ord.txt 2>&1
FP64=1 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 30000 -c 3000 --csv --log-file gpurun_out/ord_launches2.csv python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so 4000 > /dev/null 2>&1
python tools/launch_list.py gpurun_out/ord_launches2.csv "fp64 fit, launches 30000-33000" > gpurun_out/ord_ll2.txt 2>&1
FP64=1 ncu --set full --import-source on --clock-control none -k regex:k_backward_ord --launch-skip 3000 -c 1 -o gpurun_out/ord_bwd3 python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so 4000 > /dev/null 2>&1
