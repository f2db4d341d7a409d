python tools/phase_fit.py > gpurun_out/phases.txt 2>&1
W=8192 H=8192 ITERS=45 python tools/phase_fit.py >> gpurun_out/phases.txt 2>&1
W=2048 H=2048 ITERS=300 python tools/phase_fit.py >> gpurun_out/phases.txt 2>&1
