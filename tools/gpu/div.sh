for t in 1079 1080 1081 1082; do python tools/divergence_dump.py gpu $t gpurun_out/gpu_$t.npz --fp64; done > gpurun_out/div.log 2>&1
