#!/bin/bash
# Round-2 profile set: launch list of the bench command; ncu --set full of the bench step kernel
# (k_stepw, 2^22 points), the evaluation kernels (k_evalw cyclic-10 2^21, k_dense random-20x50 2^20)
# and the trackers (k_trackw katsura-10 / cyclic-10, all paths).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking katsura-10 --no-paper-protocol \
    > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stepw -s 3 -c 1 -o gpurun_out/r02_step -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" --no-evaluation --no-paper-protocol \
    > gpurun_out/ncu_step.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_evalw -s 1 -c 1 -o gpurun_out/r02_evalw -f \
    python tools/eval_once.py cyclic-10 > gpurun_out/ncu_evalw.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dense -s 1 -c 1 -o gpurun_out/r02_dense -f \
    python tools/eval_once.py random-20x50 > gpurun_out/ncu_dense.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_trackw -s 1 -c 1 -o gpurun_out/r02_trackw_katsura -f \
    python tools/track_once.py katsura-10:10000 > gpurun_out/ncu_trk.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_trackw -s 1 -c 1 -o gpurun_out/r02_trackw_cyclic10 -f \
    python tools/track_once.py cyclic-10:1000000 >> gpurun_out/ncu_trk.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/r02_launches.csv
