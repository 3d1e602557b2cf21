# Round check on one B200: GPU tests, smoke, bench, launch list, ncu captures (step + tracker).
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv &
CLK=$!
python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
kill $CLK
./tools/microbench > gpurun_out/microbench.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --points 1048576 --no-cpu-baseline --e2e-steps 1 --tracking katsura-10 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pht -s 3 -c 1 -o gpurun_out/prof_step python bench.py --steps 1 --warmup 3 --points 262144 --no-cpu-baseline --e2e-steps 1 --tracking "" > gpurun_out/ncu_step.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_track -s 1 -c 1 -o gpurun_out/prof_track python tools/track_bench.py noon-10:10000 > gpurun_out/ncu_track.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pht -c 1 -o gpurun_out/prof_eval python tools/eval_once.py > gpurun_out/ncu_eval.log 2>&1
