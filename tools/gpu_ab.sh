python -m pytest tests -m gpu -q -x 2>&1 | tail -12 > gpurun_out/gpu_tests.log
python tools/eval_bench.py > gpurun_out/eval_bench.json 2> gpurun_out/eval_bench.err
PHT_DENSE=1 python tools/eval_bench.py > gpurun_out/eval_bench_dense1.json 2> gpurun_out/eval_bench_dense1.err
