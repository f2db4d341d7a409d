for i in 1 2; do
  python tools/ab_fit.py exp/libsad_adam5.so
  python tools/ab_fit.py exp/libsad_adam6.so
done > gpurun_out/ab_adam5.txt 2>&1
FP64=1 python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so >> gpurun_out/ab_adam5.txt 2>&1
FP64=1 python tools/ab_fit.py exp/libsad_adam5.so >> gpurun_out/ab_adam5.txt 2>&1
