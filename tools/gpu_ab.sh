set -x
python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/gpu_tests.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_lib.json 2>gpurun_out/bench_lib.err
