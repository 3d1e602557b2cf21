# round-1 profile set: launch list of the bench command, ncu --set full of the step kernel (bench
# launch config), the evaluation kernels (DMMA, specialised), and the tracker.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --points 1048576 --no-cpu-baseline --e2e-steps 1 --tracking katsura-10 --no-evaluation > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pht -s 3 -c 1 -o gpurun_out/prof_step python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" --no-evaluation > gpurun_out/ncu_step.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dense -s 1 -c 1 -o gpurun_out/prof_eval_dense python tools/eval_once.py cyclic-10 > gpurun_out/ncu_eval.log 2>&1
PHT_SPEC=1 ncu --set full --clock-control none --import-source on -k regex:k_pht -s 1 -c 1 -o gpurun_out/prof_eval_spec python tools/eval_once.py cyclic-10 > gpurun_out/ncu_eval_spec.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dense -s 1 -c 1 -o gpurun_out/prof_eval_rand python tools/eval_once.py random-20x50 > gpurun_out/ncu_eval_rand.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_track -s 1 -c 1 -o gpurun_out/prof_track python tools/track_bench.py noon-10:10000 > gpurun_out/ncu_track.log 2>&1
