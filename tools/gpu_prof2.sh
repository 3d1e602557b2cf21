mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_dense -s 1 -c 1 -o gpurun_out/prof_eval_rand3 python tools/eval_once.py random-20x50 > gpurun_out/ncu_eval_rand3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dense -s 1 -c 1 -o gpurun_out/prof_eval_dense3 python tools/eval_once.py cyclic-10 > gpurun_out/ncu_eval3.log 2>&1
