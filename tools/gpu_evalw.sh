# pht_evaluate: DMMA path vs warp-per-group k_stepw<N, EVAL_X> vs tile k_phte; parity with the warp kernel
mkdir -p gpurun_out
PHT_DENSE=1 python tools/eval_bench.py > gpurun_out/ew_dense.txt 2>&1
PHT_DENSE=0 python tools/eval_bench.py > gpurun_out/ew_warp.txt 2>&1
PHT_DENSE=0 PHT_EVALW=0 python tools/eval_bench.py > gpurun_out/ew_tile.txt 2>&1
PHT_DENSE=0 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py -q -x > gpurun_out/ew_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ew_tests.log
