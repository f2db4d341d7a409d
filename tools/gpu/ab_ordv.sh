python tools/fp64_golden_check.py tests/golden/fit_config2_fp64_t1_s2.npz > gpurun_out/ordv.txt 2>&1
for v in paper_2604_21984_b200/libsad_b200.so exp/libsad_b32m2.so exp/libsad_b32m3.so; do
  FP64=1 python tools/ab_fit.py $v >> gpurun_out/ordv.txt 2>&1
done
