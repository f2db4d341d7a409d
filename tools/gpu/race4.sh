SAD_STOP_AT=3990 python tools/race_stop.py 250 > gpurun_out/race_stop.txt 2>&1
SAD_STOP_AT=2000 python tools/race_stop.py 150 >> gpurun_out/race_stop.txt 2>&1
