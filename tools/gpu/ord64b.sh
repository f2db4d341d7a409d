bash tools/gpu/ord64.sh
for i in 1; do
  FP64=1 python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so
done > gpurun_out/ab_ord.txt 2>&1
FP64=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/ord_launches.csv python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so 300 > /dev/null 2>&1
python tools/launch_list.py gpurun_out/ord_launches.csv "fp64 fit 300 iterations, ordered" > gpurun_out/ord_ll.txt 2>&1
