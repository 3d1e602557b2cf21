# Round evidence on one B200: GPU tests, smoke, default bench line, launch list of the bench command,
# ncu --set full of the step kernel at the bench launch configuration (2^22 points).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking katsura-10 --no-evaluation --no-paper-protocol > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_step python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" --no-evaluation --no-paper-protocol > gpurun_out/ncu_step.log 2>&1
