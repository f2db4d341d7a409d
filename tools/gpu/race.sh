ITERS=400 REPS=80 python tools/race_stress.py > gpurun_out/race.txt 2>&1
ITERS=4000 REPS=15 python tools/race_stress.py >> gpurun_out/race.txt 2>&1
