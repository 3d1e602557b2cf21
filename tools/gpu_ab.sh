mkdir -p gpurun_out
python tools/eval_bench.py > gpurun_out/evald.txt 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "dense or evaluate or evaluation" > gpurun_out/dense_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dense_tests.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tracking "" > gpurun_out/ab_bench.json 2> gpurun_out/ab_bench.err
