# knob sweep on the config-2 fit (same box, back to back): build-time variants and run-time env knobs
for lib in paper_2604_21984_b200/libsad_b200.so exp/libsad_pt10.so exp/libsad_pt14.so exp/libsad_sby2.so exp/libsad_sby8.so exp/libsad_qby2.so exp/libsad_qby8.so exp/libsad_pmb3.so exp/libsad_pmb5.so paper_2604_21984_b200/libsad_b200.so; do
  python tools/ab_fit.py $lib 2>/dev/null
done > gpurun_out/sweep.txt
for e in "SAD_BOX_QUEUE_STEP=2" "SAD_BOX_QUEUE_STEP=8" "SAD_GRAPH_ITERS=4" "SAD_GRAPH_ITERS=16" "SAD_NO_PDL=1"; do
  echo "$e: $(env $e python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so 2>/dev/null)"
done >> gpurun_out/sweep.txt
