# round-1 final profile set: launch list of the bench command, ncu --set full of the step kernel
# at the bench launch configuration, and the tracker.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking katsura-10 --no-evaluation --no-paper-protocol > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_step python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" --no-evaluation --no-paper-protocol > gpurun_out/ncu_step.log 2>&1
