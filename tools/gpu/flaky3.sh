for i in 1 2 3; do
  python -m pytest tests -m gpu -q > gpurun_out/fs_$i.log 2>&1; echo rc=$? >> gpurun_out/fs_$i.log
done
