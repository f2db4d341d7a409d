python -m pytest tests/test_gpu_parity.py tests/test_reduction_paths.py tests/test_reference_suite.py -m gpu -q -x -k "fp64 or ordered or overflow or collisions or exhaustion or backward or reference_suite" > gpurun_out/ordB_tests.log 2>&1; echo rc=$? >> gpurun_out/ordB_tests.log
python tools/fp64_golden_check.py > gpurun_out/ordB.txt 2>&1
python tools/fp64_golden_check.py tests/golden/fit_config2_fp64_t1_s2.npz >> gpurun_out/ordB.txt 2>&1
FP64=1 python tools/ab_fit.py paper_2604_21984_b200/libsad_b200.so >> gpurun_out/ordB.txt 2>&1
FP64=1 python tools/ab_fit.py exp/libsad_orddbg.so 4000 2>&1 | grep "ord clk" | tail -1 >> gpurun_out/ordB.txt
