python -m pytest tests/test_libm_port.py tests/test_fit_configs.py tests/test_gpu_parity.py -m gpu -q -k "not golden_set" --durations=5 > gpurun_out/gc_tests.log 2>&1; echo rc=$? >> gpurun_out/gc_tests.log
python tools/topk_convergence.py > gpurun_out/gc_conv.log 2>&1; echo rc=$? >> gpurun_out/gc_conv.log
