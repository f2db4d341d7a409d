for i in 1 2 3; do
  python -m pytest tests/test_fit_configs.py -m gpu -q > gpurun_out/fl_$i.log 2>&1; echo rc=$? >> gpurun_out/fl_$i.log
done
