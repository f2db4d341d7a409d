K="python tools/kbench.py"
for lib in paper_2604_21984_b200/libsad_b200.so exp/libsad_fin0.so exp/libsad_adam4.so exp/libsad_adam6.so; do
  echo "== $lib"
  $K --lib $lib --kernel adam,adam_active,stats --reps 50
  python tools/ab_fit.py $lib
done > gpurun_out/ab_adam.txt 2>&1
