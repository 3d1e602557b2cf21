mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py -q -x -k "step or euler or pc" > gpurun_out/sw_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sw_tests.log
PHT_STEPW=0 python tools/step_bench.py > gpurun_out/swq_tile.txt 2>&1
python tools/step_bench.py > gpurun_out/swq_w.txt 2>&1
python tools/step_bench.py >> gpurun_out/swq_w.txt 2>&1
ncu --section MemoryWorkloadAnalysis_Tables --section SpeedOfLight --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_step -s 1 -c 1 python tools/step_once.py > gpurun_out/swq_ncu.txt 2>&1
