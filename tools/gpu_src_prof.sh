# Source-level ncu capture of the step kernel (cyclic-10, 2^20 points): per-line stall samples.
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_step -s 1 -c 1 -o gpurun_out/prof_src python tools/step_once.py > gpurun_out/ncu_src.log 2>&1
ncu -i gpurun_out/prof_src.ncu-rep --page source --csv --print-source sass > gpurun_out/src_sass.csv 2>&1
ncu -i gpurun_out/prof_src.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_cuda.csv 2>&1
