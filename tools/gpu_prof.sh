# microbenchmarks + ncu capture of the step kernel and the evaluate kernel
set -x
./tools/microbench > gpurun_out/microbench.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pht -s 3 -c 1 -o gpurun_out/prof_step_v2 python bench.py --steps 1 --warmup 3 --points 262144 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_step.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pht -c 1 -o gpurun_out/prof_eval_v2 python tools/eval_once.py > gpurun_out/ncu_eval.log 2>&1
