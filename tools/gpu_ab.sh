mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-evaluation > gpurun_out/ab_bench.json 2> gpurun_out/ab_bench.err
