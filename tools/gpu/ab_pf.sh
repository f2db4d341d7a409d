K="python tools/kbench.py"
for lib in exp/libsad_pf0.so paper_2604_21984_b200/libsad_b200.so; do
  echo "== $lib"
  $K --lib $lib --kernel propagate_warm,propagate_flood,refresh_full --reps 50
  $K --lib $lib --kernel propagate_warm,propagate_flood --reps 20 --width 2048 --height 2048 --n-sites 100000 --iters 100
  python tools/ab_fit.py $lib
done > gpurun_out/ab_pf.txt 2>&1
